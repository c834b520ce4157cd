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
