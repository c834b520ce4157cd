"""bench.py's host-side measurement logic (CPU): the roofline selection of
SURVEY.md §8(d), nearest-rank percentiles (telemetry/metrics.py:33-37) and the
per-workload algorithmic counts it divides by."""
import importlib.util
import json

import pytest

from conftest import ROOT
from paper_2510_19689_b200 import workloads as W


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


PEAKS = {"hbm_gbs": 6536.4, "bf16_tflops": 1648.0}


def test_roofline_binding_roof(bench):
    c = W.algorithmic_counts(W.WORKLOADS["hr"])
    # bf16 on HR: HBM-bound (1000 B/row vs 106 kFLOP/row)
    r = bench.roofline("bf16", c, 65536, 0.040, PEAKS)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    t_roof = 65536 * 1000 / (6536.4e9)
    assert abs(r["frac"] - t_roof / 40e-6) < 1e-9
    assert r["tensor"]["passes"] == 1
    # 3xTF32: three passes of the flops against the TF32 peak -> tensor-bound
    r3 = bench.roofline("tf32x3", c, 65536, 0.064, PEAKS)
    assert r3["tensor"]["passes"] == 3
    assert r3["bound"] == "tensor" and r3["unit"] == "TFLOP/s"
    assert r3["frac"] == pytest.approx(r3["tensor"]["frac"])
    # fp32 CUDA cores: no tensor roof
    rf = bench.roofline("fp32", c, 65536, 2.0, PEAKS)
    assert rf["bound"] == "hbm" and rf["tensor"] is None


def test_nearest_rank(bench):
    vals = list(range(1, 101))
    assert bench.nearest_rank(vals, 50) == 50
    assert bench.nearest_rank(vals, 99) == 99
    assert bench.nearest_rank([3.0], 99) == 3.0
    assert bench.nearest_rank([], 50) is None


def test_committed_bench_lines_are_consistent():
    """Every committed bench line carries the contract keys, and its value and
    roofline fraction agree with its own timing."""
    lines = sorted((ROOT / "profiles").glob("bench_r1c_*.json"))
    assert lines
    for p in lines:
        d = json.loads(p.read_text())
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                  "higher_is_better", "scaling", "dtype", "config", "roofline", "e2e",
                  "gpu_launches", "clocks"):
            assert k in d, (p.name, k)
        rows = d["config"]["rows_per_rank"]
        assert d["value"] == pytest.approx(rows * d["n_gpus"] / (d["ms_per_step"] / 1e3), rel=1e-6)
        r = d["roofline"]
        assert 0.0 < r["frac"] < 1.0 and r["bound"] in ("hbm", "tensor")
        assert d["warmup"] >= 3 and not d["clocks"]["reasons"]


def test_l2_plan_rotates_past_l2_or_flushes(bench):
    for name, rows in [("hr", 65536), ("bls", 262144), ("wide", 262144), ("adult", 4096), ("hr_latency", 1024)]:
        per_set = rows * W.algorithmic_counts(W.WORKLOADS[name])["bytes_per_row"]
        nsets, flush = bench.l2_plan(per_set)
        assert 2 <= nsets <= 8
        if flush:
            assert nsets * per_set < 2 * bench.L2_BYTES
        else:
            assert nsets * per_set >= 2 * bench.L2_BYTES      # every step streams from HBM
        assert flush == (name in ("adult", "hr_latency"))


def test_rank_row_plans(bench):
    """Weak scaling gives every rank its own full batch; --shard (default for BLS,
    wide and hr8) splits the config's batch into contiguous shards."""
    a = bench.parse(["--config", "bls"])
    w = W.WORKLOADS["bls"]
    plans = [bench.plan_rows(w, a, r, 4) for r in range(4)]
    assert [p[0] for p in plans] == [65536] * 4 and [p[1] for p in plans] == [0, 65536, 131072, 196608]
    assert all(p[2] for p in plans)
    a = bench.parse(["--config", "hr"])
    rows, start, sh = bench.plan_rows(W.WORKLOADS["hr"], a, 3, 8)
    assert (rows, start, sh) == (65536, 3 * 65536, False)
    a = bench.parse(["--config", "hr8"])
    assert bench.plan_rows(W.WORKLOADS["hr8"], a, 7, 8) == (8192, 7 * 8192, True)
    a = bench.parse(["--config", "bls", "--no-shard"])
    assert bench.plan_rows(w, a, 1, 2) == (262144, 262144, False)
    a = bench.parse(["--config", "hr8", "--rows", "1000"])          # explicit rows: weak
    assert bench.plan_rows(W.WORKLOADS["hr8"], a, 1, 2) == (1000, 1000, False)


def test_both_arms_print_the_same_config(bench):
    for cfg in ("hr", "bls", "hr8"):
        a = bench.parse(["--config", cfg])
        w = W.WORKLOADS[cfg]
        rows, _, sh = bench.plan_rows(w, a, 0, 2)
        c = bench.bench_config(w, a, rows, 2, sh)
        assert c == bench.bench_config(w, bench.parse(["--config", cfg, "--impl", "reference"]), rows, 2, sh)
        assert "precision" not in c and c["rows_per_rank"] == rows


def test_chunked_stream_plan(bench):
    bpr = W.algorithmic_counts(W.WORKLOADS["wide"])["bytes_per_row"]
    ch, n = bench.chunk_plan(1 << 24, bpr)
    assert ch % 128 == 0 and ch * bpr <= bench.MAX_CHUNK_BYTES and ch * n >= 1 << 24 and ch * (n - 1) < 1 << 24
    assert bench.chunk_plan(65536, 1000) == (65536, 1)


def test_self_launch_command(bench):
    cmd = bench.launch_cmd(4, ["--config", "bls"], 29999)
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-2:] == ["--config", "bls"]


def test_two_rank_launch_and_reduction_gloo():
    """`bench.py --gpus 2` with WORLD_SIZE unset re-launches itself under
    torch.distributed.run (2 ranks, gloo for --dry-run): rank 0 prints n_gpus 2,
    the shard plan, the max of the per-rank times and the sum of their rows."""
    import os
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "bls", "--dry-run"],
                       capture_output=True, text=True, timeout=240, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["rows_per_rank"] == 131072 and d["rows_all_ranks"] == 262144
    assert d["max_ms"] == 2.0 and d["shards"] == [[0, 131072], [131072, 131072]]
    assert d["step_max_ms"] == [6.0, 6.0, 1.0]      # per-step latency: the slowest rank per step
    assert d["scaling"] == "strong"
