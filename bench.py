#!/usr/bin/env python
"""Benchmark: TabNet predict+explain rows/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config hr]
                    [--precision bf16] [--shard | --no-shard] [--inflight Q]
                    [--impl ours|reference]

One "step" = one fused forward of the workload's batch with inputs resident in
HBM (HR: 65,536 rows, BASELINE.json configs[1]).  ``--gpus N`` runs one process
per GPU: launched under torchrun by the driver, or re-launched through
``torch.distributed.run`` by this script when WORLD_SIZE is unset.  Rows are
independent (reference network.py:11-14), so the ranks never exchange data:

* weak scaling (HR, Adult, the latency sweep): every rank runs its own batch;
* strong scaling (``--shard``, the default for BLS, wide and ``hr8``): the
  config's batch is split into contiguous row shards, rank r taking
  ``shard_bounds(batch, N)[r]`` (BASELINE.json configs[2] and the north star's
  65,536-row batch on 8 GPUs).

Timing is CUDA events on the launching stream, max over ranks; rank 0 prints
ONE JSON line.  ``--inflight Q`` (and the ``steady_state`` sub-object) keeps Q
independent batches of the rank's rows in flight on Q streams per step: what a
GPU serving a stream of 8,192-row requests sustains.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port under oracle/, bitwise equal to the reference's apply) on the
host's cores with a process pool, on the same config/metric.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2510_19689_b200 import workloads as W  # noqa: E402
from paper_2510_19689_b200.sharding import shard_bounds  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
METRIC = "TabNet inferences/sec (predict+explain)"
MAX_CHUNK_BYTES = 3 << 30      # a launch's outputs stay below this: bigger shards stream in chunks


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="hr", choices=sorted(W.WORKLOADS))
    ap.add_argument("--rows", type=int, default=0,
                    help="rows per rank (weak scaling; default: the config's batch, or its shard)")
    ap.add_argument("--shard", dest="shard", action="store_true", default=None,
                    help="split the config's batch over the ranks (strong scaling)")
    ap.add_argument("--no-shard", dest="shard", action="store_false")
    ap.add_argument("--inflight", type=int, default=0,
                    help="steady-state batches in flight per GPU (default 8 when a rank's batch "
                         "is below 65,536 rows, else 0 = not reported)")
    ap.add_argument("--precision", default="bf16",
                    choices=["bf16", "tf32", "tf32x3", "fp32"],
                    help="FC contraction arithmetic (bf16: the production mode; tf32x3: the "
                         "fp32-faithful exactness mode)")
    ap.add_argument("--regime", default="trained", choices=["trained", "init"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-share", action="store_true",
                    help="skip the north-star share sub-object (HR: 8,192-row batches, one GPU's share of 65,536 on 8)")
    ap.add_argument("--no-parity-mode", action="store_true",
                    help="skip the tf32x3 (parity mode) timing sub-object")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch each timed step from Python instead of replaying a CUDA graph")
    ap.add_argument("--latency-sweep", action="store_true",
                    help="also report p50/p99 device+e2e latency for batches 1..1024 (config 3)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the ranks (gloo), print the row plan and the cross-rank reduction, "
                         "touch no GPU")
    return ap.parse_args(argv)


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_cmd(n: int, argv: list[str], port: int) -> list[str]:
    """The torchrun command that runs this script on n ranks (one per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]


def shard_mode(w: W.Workload, a) -> bool:
    if a.rows:
        return False
    return w.shard if a.shard is None else a.shard


def plan_rows(w: W.Workload, a, rank: int, world: int) -> tuple[int, int, bool]:
    """(rows this rank processes per step, its first row in the workload's input
    stream, sharded?).  Weak scaling gives every rank a full batch of its own
    rows; sharding splits the config's batch into contiguous blocks."""
    if shard_mode(w, a):
        lo, hi = shard_bounds(w.batch, world)[rank]
        return hi - lo, lo, True
    rows = a.rows or w.batch
    return rows, rank * rows, False


def reduce_over_ranks(total_ms: float, rows: int, world: int, dist, device) -> tuple[float, float]:
    """(max over ranks of the timed device milliseconds, rows of all ranks)."""
    import torch
    t = torch.tensor([total_ms, float(rows)], dtype=torch.float64, device=device)
    if world == 1:
        return total_ms, float(rows)
    tmax, tsum = t.clone(), t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return float(tmax[0].item()), float(tsum[1].item())


def max_over_ranks_list(vals: list, world: int, dist, device) -> list:
    """Elementwise max over ranks (each step's batch latency at N GPUs is its
    slowest shard's)."""
    if world == 1:
        return list(vals)
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def run_dry(a) -> None:
    """The rank/row plan and the max/sum reduction of run_ours, over gloo on
    CPU (tests/test_bench_logic.py runs it under the self-launch)."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    w = W.WORKLOADS[a.config]
    rows, start, sharded = plan_rows(w, a, rank, world)
    fake_ms = 1.0 + rank                      # a made-up per-rank time: the max must win
    ms, total = reduce_over_ranks(fake_ms, rows, world, dist, torch.device("cpu"))
    # per-step latencies: each step's slowest rank (rank r is slow on step r)
    steps = max_over_ranks_list([1.0 + (5.0 if i == rank else 0.0) for i in range(3)], world, dist,
                                torch.device("cpu"))
    starts = [None] * world
    if world > 1:
        dist.all_gather_object(starts, (start, rows))
    else:
        starts = [(start, rows)]
    if rank == 0:
        print(json.dumps({"n_gpus": world, "rows_per_rank": rows, "rows_all_ranks": total,
                          "max_ms": ms, "step_max_ms": steps, "shards": starts,
                          "scaling": "strong" if sharded else "weak",
                          "config": bench_config(w, a, rows, world, sharded)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_config(w: W.Workload, a, rows: int, world: int, sharded: bool) -> dict:
    """The workload description both arms print (identical for the same flags)."""
    return {"workload": w.description, "batch": w.batch if sharded else rows, "rows_per_rank": rows,
            "regime": a.regime,
            "head": "regression (identity head on logit column 0 of the 2-class reference model)"
            if w.regression else "softmax classifier",
            "outputs": ("output value, masks (S,B,F), importance" if w.regression else
                        "logits, probabilities, masks (S,B,F), importance, class"),
            "parallelism": (f"row-shard x{world} of one batch (strong scaling, no collective)" if sharded
                            else f"independent batch per rank x{world} (weak scaling, no collective)")}


def nearest_rank(vals, q):
    """Nearest-rank percentile (reference telemetry/metrics.py:33-37)."""
    s = sorted(vals)
    if not s:
        return None
    k = max(1, int(np.ceil(q / 100.0 * len(s))))
    return s[k - 1]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- cpu arm
REF_DIR = ROOT / "baseline" / "_ref"      # the unmodified reference (tools/install_reference.sh)


def reference_kind() -> str:
    """"reference": the unmodified tabserve package is installed in baseline/_ref
    and its own TabNetModel.apply is timed; "port": the oracle restatement
    (bitwise equal to it, tests/test_oracle.py) stands in."""
    return "reference" if (REF_DIR / "tabserve" / "model" / "network.py").exists() else "port"


def _oracle_worker(args):
    name, regime, start, rows = args
    w = W.WORKLOADS[name]
    m = W.make_model(name, regime)
    x = W.make_inputs(w, rows, start=start).astype(np.float64)
    if reference_kind() == "reference":
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        from tabserve.model.config import ModelConfig as RefConfig
        from tabserve.model.network import TabNetModel as RefModel
        c = m.config
        ref = RefModel(config=RefConfig(feature_count=c.feature_count, n_classes=c.n_classes, n_d=c.n_d,
                                        n_a=c.n_a, n_steps=c.n_steps, gamma=c.gamma),
                       params=m.params, norm_mean=m.norm_mean, norm_var=m.norm_var,
                       model_version=m.model_version)
        t0 = time.perf_counter()
        ref.apply(x)                                 # network.py:195-267, the reference's own code
        return time.perf_counter() - t0
    from oracle import tabnet_oracle as O
    t0 = time.perf_counter()
    O.apply_model(m, x)
    return time.perf_counter() - t0


class CpuReference:
    """The reference algorithm on host cores: the unmodified tabserve
    TabNetModel.apply from baseline/_ref (else oracle/tabnet_oracle.py, bitwise
    equal to it) over a fork pool of contiguous row shards (its einsum path is
    single-threaded)."""

    def __init__(self, name: str, regime: str, rows_per_step: int, procs: int | None = None):
        import multiprocessing as mp
        self.procs = procs or max(1, len(os.sched_getaffinity(0)))
        self.name, self.regime = name, regime
        self.rows = rows_per_step
        self.pool = mp.get_context("fork").Pool(self.procs)

    def step(self) -> float:
        bounds = np.linspace(0, self.rows, self.procs + 1).astype(int)
        jobs = [(self.name, self.regime, int(a), int(b - a)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        # the shards run concurrently: a step lasts as long as its slowest shard
        return max(self.pool.map(_oracle_worker, jobs))

    def close(self):
        self.pool.close()
        self.pool.join()


REF_SRC = {"reference": "tabserve TabNetModel.apply (unmodified reference, baseline/_ref)",
           "port": "oracle/tabnet_oracle.py (bitwise = reference apply)"}

CPU_ROWS_PER_CORE = {"adult": 16384, "hr": 4096, "hr8": 4096, "hr_latency": 4096, "bls": 1536, "wide": 96}


def cpu_rows_per_step(w: W.Workload, procs: int) -> int:
    return int(min(w.batch, CPU_ROWS_PER_CORE[w.name] * procs))


def cpu_baseline(w: W.Workload, regime: str, steps: int = 3) -> dict:
    """The reference algorithm (oracle port) on every host core plus a 1-core
    figure, on a bounded sample of the workload (rank 0, N=1 only)."""
    procs = max(1, len(os.sched_getaffinity(0)))
    crow = cpu_rows_per_step(w, procs)
    if w.name == "wide":       # a 65,536-row subset, extrapolated
        crow = min(w.batch, 65536)
        steps = 1
    ref = CpuReference(w.name, regime, crow)
    if w.name != "wide":
        ref.step()
    ct = [ref.step() for _ in range(steps)]
    ref.close()
    one_rows = CPU_ROWS_PER_CORE[w.name]
    t1 = _oracle_worker((w.name, regime, 0, one_rows))
    extrap = crow < w.batch
    kind = reference_kind()
    return {"value": crow * steps / sum(ct), "unit": "rows/s", "cores": procs, "kind": kind,
            "cpu_model": cpu_model(), "value_1core": one_rows / t1,
            "sample": (f"{crow} rows x {steps} steps of {w.name} ({regime} weights), "
                       f"{REF_SRC[kind]} on {procs} fork-pool "
                       f"processes; 1-core figure on {one_rows} rows"
                       + ("; rows/s of this subset stand for the full batch (per-row cost is "
                          "constant beyond ~1k rows: an extrapolation)" if extrap else ""))}


def run_reference(a) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = W.WORKLOADS[a.config]
    rows, _, sharded = plan_rows(w, a, 0, world)
    procs = max(1, len(os.sched_getaffinity(0)))
    crow = cpu_rows_per_step(w, procs)
    ref = CpuReference(a.config, a.regime, crow)
    for _ in range(a.warmup):
        ref.step()
    times = [ref.step() for _ in range(a.steps)]
    ref.close()
    total = sum(times)
    value = crow * a.steps / total
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "rows/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * total / a.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(w, a, rows, world, sharded),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": procs, "kind": reference_kind(),
                         "cpu_model": cpu_model(),
                         "sample": f"{crow} rows/step of {a.config} ({a.regime} weights), "
                                   f"{REF_SRC[reference_kind()]} over {procs} fork-pool processes"
                                   + (" (a bounded subset of the batch)" if crow < rows else "")},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def profile_traffic(config: str, precision: str, rows: int):
    """DRAM read+write bytes per launch of `rows` rows from the committed ncu
    captures: the steady-state capture (tools/profile_traffic.sh: application
    replay, no cache control, inside a rotating > L2 launch sequence) scaled
    per row, else the single-launch --set full figure."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None, None
    try:
        d = json.loads(p.read_text())
        e = d.get(f"{config}/{precision}") or {}
        if "dram_bytes_per_row_steady" in e:
            return e["dram_bytes_per_row_steady"] * rows, e.get("steady_how")
        v = e.get("dram_bytes_per_launch")
        return v, ("single --set full launch (outputs left in L2: under-counts writes)" if v else None)
    except Exception:
        return None, None


def roofline(precision: str, counts: dict, rows: int, kernel_ms: float, peaks: dict) -> dict:
    """t_roof = max(bytes / HBM, flops * passes / P_mode); the
    binding roof is reported (achieved and peak in its units), the other one
    alongside.  passes = 3 for 3xTF32 (three MMAs per product), else 1."""
    hbm = peaks.get("hbm_gbs", 6650.0)
    tf32_file = ROOT / "profiles" / "measured_tf32.json"
    tf32 = json.loads(tf32_file.read_text()) if tf32_file.exists() else {}
    if precision == "bf16":
        tpk, tsrc = peaks.get("bf16_tflops", 2250.0), "MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3, burst)"
    elif precision in ("tf32", "tf32x3"):
        tpk = tf32.get("tf32_tflops", peaks.get("bf16_tflops", 2250.0) / 2)
        tsrc = ("profiles/measured_tf32.json tf32_tflops (cuBLAS fp32+allow_tf32 8192^3, burst)"
                if tf32 else "estimate: MEASURED_PEAKS bf16_tflops / 2")
    else:
        tpk, tsrc = None, "no tensor-core path (CUDA-core fp32)"
    passes = 3 if precision == "tf32x3" else 1
    t_s = kernel_ms / 1e3
    bytes_ = counts["bytes_per_row"] * rows
    flops = counts["flops_per_row"] * rows * passes
    t_hbm = bytes_ / (hbm * 1e9)
    t_ten = flops / (tpk * 1e12) if tpk else 0.0
    hbm_part = {"achieved": bytes_ / t_s / 1e9, "peak": hbm, "unit": "GB/s", "frac": t_hbm / t_s}
    ten_part = ({"achieved": flops / t_s / 1e12, "peak": tpk, "unit": "TFLOP/s", "frac": t_ten / t_s,
                 "passes": passes, "peak_source": tsrc} if tpk else None)
    bound = "tensor" if (tpk and t_ten > t_hbm) else "hbm"
    main = ten_part if bound == "tensor" else hbm_part
    return {"bound": bound, "achieved": main["achieved"], "peak": main["peak"], "unit": main["unit"],
            "frac": main["frac"], "traffic": None,
            "hbm": hbm_part, "tensor": ten_part,
            "algorithmic_bytes_per_row": counts["bytes_per_row"],
            "algorithmic_flops_per_row": counts["flops_per_row"],
            "kernel_ms_per_launch": kernel_ms,
            "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if peaks else "fallback 6650 GB/s"}


def l2_plan(per_set_bytes: int) -> tuple:
    """(rotating input/output sets, flush_mode) for a step that touches
    ``per_set_bytes``: rotate over >= 2.5x L2 with at most 8 sets; batches too
    small for that (Adult, the latency sweep) flush L2 before every timed step
    and time each step on its own instead."""
    nsets = min(8, max(2, int(np.ceil(2.5 * L2_BYTES / per_set_bytes))))
    return nsets, nsets * per_set_bytes < 2 * L2_BYTES


def chunk_plan(rows: int, bytes_per_row: int) -> tuple[int, int]:
    """(rows per launch, launches per step): a rank's step larger than
    MAX_CHUNK_BYTES of outputs (the wide config's 2^24 rows) streams through
    equal chunks (multiples of 128 rows) so its buffers stay device-resident."""
    if rows * bytes_per_row <= MAX_CHUNK_BYTES:
        return rows, 1
    ch = max(128, (MAX_CHUNK_BYTES // bytes_per_row) // 128 * 128)
    n = (rows + ch - 1) // ch
    ch = ((rows + n - 1) // n + 127) // 128 * 128      # n equal chunks (the last may be short by < 128 n)
    return ch, (rows + ch - 1) // ch


class StepRunner:
    """One rank's device-resident step: rotating input/output sets (> 2.5x L2
    in total, or an L2 flush per step when they would fit) and, for shards
    bigger than one launch, a chunked stream over them."""

    def __init__(self, model, w, rows: int, start: int, local: int, flush_ok: bool = True, flags: int = 0):
        import torch
        from paper_2510_19689_b200.device import DeviceRunner
        self.torch = torch
        self.dev = torch.device("cuda", local)
        bpr = W.algorithmic_counts(w)["bytes_per_row"]
        self.rows = rows
        self.chunk, self.nchunks = chunk_plan(rows, bpr)
        self.nsets, self.flush_mode = l2_plan(self.chunk * bpr)
        if not flush_ok:
            self.flush_mode = False
        if self.nchunks > 1:                 # streaming: rows repeat over the distinct input chunks
            self.nsets = max(2, min(self.nsets, self.nchunks))
        self.runner = DeviceRunner(model, self.chunk, device=local, flags=flags)
        self.xs = [torch.from_numpy(W.make_inputs(w, self.chunk, start=start + i * self.chunk)).to(self.dev)
                   for i in range(self.nsets)]
        self.outs = [self.runner.alloc_outputs(self.chunk) for _ in range(self.nsets)]
        self.sizes = [min(self.chunk, rows - c * self.chunk) for c in range(self.nchunks)]
        self.k = 0                            # rotating set counter

    def launch(self, stream) -> int:
        """Queue one step on ``stream``; returns the number of kernel launches."""
        for c in range(self.nchunks):
            i = self.k % self.nsets
            self.k += 1
            n = self.sizes[c]
            x = self.xs[i] if n == self.chunk else self.xs[i][:n]
            self.runner.run(x, self.outs[i] if n == self.chunk else self.runner.views(n), stream=stream)
        return self.nchunks


def capture(torch, dev, fn):
    """CUDA graph of ``fn(stream)`` captured on a side stream."""
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            fn(side)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    return g


def time_graph(torch, g, stream, reps: int = 3) -> float:
    """Best-of-reps device time (ms) of one replay, CUDA events on ``stream``."""
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def run_ours(a) -> None:
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    w = W.WORKLOADS[a.config]
    rows, start, sharded = plan_rows(w, a, rank, world)
    counts = W.algorithmic_counts(w)
    model = W.make_engine_model(a.config, a.regime, precision=a.precision, device=local)
    sr = StepRunner(model, w, rows, start, local)
    runner = sr.runner
    stream = torch.cuda.current_stream(dev)
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if sr.flush_mode else None

    for _ in range(a.warmup):
        sr.launch(stream)
    torch.cuda.synchronize()
    runner.check_finite()
    # The K timed steps are captured into ONE CUDA graph (the fused launches back
    # to back on the rotating sets), so host launch overhead (ctypes + Python,
    # tens of us per call) never leaves the GPU idle between steps.  Per-step
    # latency is measured separately with one single-step graph per set.
    use_graph = not a.no_graph
    launches_per_step = sr.nchunks
    if use_graph:
        sr.k = 0
        big = capture(torch, dev, lambda s: [sr.launch(s) for _ in range(a.steps)])
        singles = []
        for i in range(sr.nsets if sr.nchunks == 1 else 1):
            sr.k = i
            singles.append(capture(torch, dev, lambda s: sr.launch(s)))
        step_fns = [g1.replay for g1 in singles]
        for f1 in step_fns:
            f1()
        torch.cuda.synchronize()
        runner.check_finite()
    else:
        step_fns = [lambda: sr.launch(stream)]

    clocks = ClockSampler(local)
    clocks.start()
    # ~0.3 s of untimed load so the clock samples see the GPU busy
    t_load = time.perf_counter()
    while time.perf_counter() - t_load < 0.3:
        if use_graph:
            big.replay()
        else:
            for i in range(a.steps):
                step_fns[i % len(step_fns)]()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    flushed_ms = None
    if sr.flush_mode:
        # per step: write 2x L2 (torch fill), then the step between its own events;
        # the host queues the whole loop behind a device sleep so no launch gap
        # falls inside an event pair
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                 for _ in range(a.steps)]
        torch.cuda._sleep(int(2_000_000 + 60_000 * a.steps))
        for i in range(a.steps):
            flush_buf.fill_(i & 0xFF)
            pairs[i][0].record(stream)
            step_fns[i % len(step_fns)]()
            pairs[i][1].record(stream)
        torch.cuda.synchronize()
        flushed_ms = [p0.elapsed_time(p1) for p0, p1 in pairs]
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if use_graph:
            big.replay()
        else:
            for i in range(a.steps):
                step_fns[0]()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(flushed_ms) if sr.flush_mode else e0.elapsed_time(e1)
    # max over ranks of the device time; the rows of all ranks
    total_ms_max, total_rows = reduce_over_ranks(total_ms, rows, world, dist, dev)
    value = total_rows * a.steps / (total_ms_max / 1e3)
    kernel_ms = total_ms / a.steps / launches_per_step     # per launch, this rank
    runner.check_finite()
    # per-batch latency: each step on its own (single-step graph replay between events)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    torch.cuda._sleep(200_000)          # keep the GPU busy while the host queues the loop
    ev[0].record(stream)
    for i in range(a.steps):
        step_fns[i % len(step_fns)]()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    per_step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
    if sr.flush_mode:
        per_step_ms = flushed_ms        # cold-L2 per-step device times
    per_step_ms = max_over_ranks_list(per_step_ms, world, dist, dev)

    # ---- steady state: Q batches of this rank's rows in flight on Q streams
    steady = None
    q = a.inflight if a.inflight else (8 if rows < 65536 and sr.nchunks == 1 else 0)
    if q > 1 and use_graph:
        steady = steady_state(torch, dev, model, w, rows, start, local, q, counts, world, dist)

    # ---- parity mode (3xTF32, the fp32-faithful exactness mode) timed the same way
    parity = None
    if not a.no_parity_mode and a.precision != "tf32x3" and use_graph:
        parity = parity_mode(torch, dev, w, a, rows, start, local, counts, world, dist)

    # ---- the north star's per-GPU share (65,536 rows over 8 GPUs = 8,192 rows per GPU)
    share = None
    if (a.config == "hr" and rows == 65536 and world == 1 and not a.no_share and use_graph
            and a.precision == "bf16"):
        share = north_star_share(torch, dev, model, w, start, local, counts, world, dist)

    # ---- end to end through the C-ABI host call: pinned host in/out, H2D+D2H timed
    e2e = None
    if not a.no_e2e:
        e2e = end_to_end(torch, dev, model, w, sr, rank, world, dist, a)

    # ---- latency sweep (config 3) ----
    latency = None
    if a.latency_sweep and rank == 0:
        latency = latency_sweep(model, local, w.feature_count)

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(w, a.regime)

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    roof = roofline(a.precision, counts, sr.chunk, kernel_ms, peaks)
    roof["traffic"], how = profile_traffic(a.config, a.precision, sr.chunk)
    roof["traffic_source"] = f"profiles/ncu_summary.json: {how}" if how else None
    if rank == 0:
        cfg = bench_config(w, a, rows, world, sharded)
        line = {
            "metric": METRIC,
            "value": value, "unit": "rows/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": total_ms_max / a.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": {"tf32x3": "fp32 (3xTF32 tcgen05 GEMMs)", "tf32": "tf32",
                                           "bf16": "bf16", "fp32": "fp32 (CUDA-core FFMA)"}[a.precision],
            "data": "synthetic",
            "config": cfg,
            "timing": {
                "precision": a.precision,
                "l2": (f"flushed before every timed step (a {2 * L2_BYTES >> 20} MiB write; "
                       f"{sr.nsets} rotating sets would fit in L2)" if sr.flush_mode else
                       f"rotating {sr.nsets} input/output sets > 126 MiB L2"),
                "launch": "python loop" if a.no_graph else
                ("one single-step CUDA graph replay per step between its own CUDA events "
                 "(the L2 flush outside them); value = rows x K / sum of step times"
                 if sr.flush_mode else "one CUDA graph of the K steps (timed as one replay)"),
                "launches_per_step": launches_per_step,
                "rows_per_launch": sr.chunk,
                "stream": (f"{rows} rows per step as {sr.nchunks} chunked launches over {sr.nsets} "
                           "distinct device-resident input chunks" if sr.nchunks > 1 else None),
                "rows_all_ranks_per_step": total_rows,
            },
            "roofline": roof,
            "latency_ms": {"p50": nearest_rank(per_step_ms, 50), "p99": nearest_rank(per_step_ms, 99),
                           "batch": rows, "kind": "device (CUDA events around each step's single-step graph replay"
                                                  + (", L2 flushed before each" if sr.flush_mode else "")
                                                  + ("; max over ranks per step)" if world > 1 else ")")},
            "steady_state": steady,
            "parity_mode": parity,
            "north_star_share": share,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": a.steps * launches_per_step,
            "clocks": clk,
        }
        if latency is not None:
            line["latency_sweep"] = latency
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def steady_state(torch, dev, model, w, rows, start, local, q, counts, world, dist) -> dict:
    """Q independent batches of ``rows`` in flight on Q streams per step (one
    graph, K_SS steps): the sustained rows/s of a GPU serving such requests."""
    # TBN_FLAG_PACKED: each batch takes full row tiles on as few SMs as it
    # needs, so the Q batches run side by side instead of each spreading one
    # partial tile over every SM (launch geometry only; outputs are identical)
    from paper_2510_19689_b200 import _native as N
    runners = [StepRunner(model, w, rows, start + j * rows, local, flush_ok=False, flags=N.FLAG_PACKED)
               for j in range(q)]
    ks = 10

    def body(s):
        ev0 = torch.cuda.Event()
        ev0.record(s)
        subs = [torch.cuda.Stream(dev) for _ in range(q)]
        for _ in range(ks):
            joins = []
            for sr_j, sj in zip(runners, subs):
                sj.wait_event(ev0)
                sr_j.launch(sj)
                e = torch.cuda.Event()
                e.record(sj)
                joins.append(e)
            for e in joins:
                s.wait_event(e)
            ev0 = torch.cuda.Event()
            ev0.record(s)
    g = capture(torch, dev, body)
    g.replay()
    torch.cuda.synchronize()
    ms = time_graph(torch, g, torch.cuda.current_stream(dev))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total = world * q * rows * ks
    for r in runners:
        r.runner.check_finite()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    frac = counts["bytes_per_row"] * total / (ms / 1e3) / (world * peaks.get("hbm_gbs", 6650.0) * 1e9)
    return {"inflight_per_gpu": q, "rows_per_batch": rows, "value": total / (ms / 1e3), "unit": "rows/s",
            "ms_per_round": ms / ks, "hbm_frac": frac,
            "how": f"{q} streams per GPU, each launching its own {rows}-row batch per round (TBN_FLAG_PACKED), "
                   f"{ks} rounds in one CUDA graph, max over ranks"}


def north_star_share(torch, dev, model, w, start, local, counts, world, dist) -> dict:
    """One GPU's share of the north star's HR batch (65,536 rows row-sharded
    over 8 GPUs, no collective): 8,192-row batches back to back on one stream
    (each a single tile chain per SM), and 16 such batches in flight."""
    rows = 65536 // 8
    sr = StepRunner(model, w, rows, start, local, flush_ok=False)
    ks = 20
    g = capture(torch, dev, lambda s: [sr.launch(s) for _ in range(ks)])
    g.replay()
    torch.cuda.synchronize()
    ms = time_graph(torch, g, torch.cuda.current_stream(dev)) / ks
    sr.runner.check_finite()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0) * 1e9
    ss = steady_state(torch, dev, model, w, rows, start, local, 16, counts, world, dist)
    return {"rows_per_gpu": rows, "gpus": 8,
            "one_batch": {"us": ms * 1e3, "rows_per_s": rows / (ms / 1e3),
                          "hbm_frac": counts["bytes_per_row"] * rows / (ms / 1e3) / hbm,
                          "how": f"{ks} back-to-back 8,192-row batches on one stream in one CUDA graph"},
            "inflight_16": {"rows_per_s": ss["value"], "hbm_frac": ss["hbm_frac"], "how": ss["how"]}}


def parity_mode(torch, dev, w, a, rows, start, local, counts, world, dist) -> dict | None:
    """The fp32-faithful 3xTF32 mode on the same rows, timed the same way."""
    from paper_2510_19689_b200.errors import UnsupportedShapeError
    try:
        m = W.make_engine_model(a.config, a.regime, precision="tf32x3", device=local)
        m.engine(device=local)
    except UnsupportedShapeError as e:
        return {"precision": "tf32x3", "unavailable": str(e)}
    sr = StepRunner(m, w, rows, start, local, flush_ok=False)
    ks = max(5, min(20, a.steps))
    g = capture(torch, dev, lambda s: [sr.launch(s) for _ in range(ks)])
    g.replay()
    torch.cuda.synchronize()
    ms = time_graph(torch, g, torch.cuda.current_stream(dev))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    sr.runner.check_finite()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    roof = roofline("tf32x3", counts, sr.chunk, ms / ks / sr.nchunks, peaks)
    return {"precision": "tf32x3", "value": world * rows * ks / (ms_max / 1e3), "unit": "rows/s",
            "ms_per_step": ms_max / ks, "roofline_bound": roof["bound"], "roofline_frac": roof["frac"],
            "hbm_frac": roof["hbm"]["frac"],
            "kernel": ("K2 3xTF32" if w.feature_count < 64 else
                       "K3X 3xTF32 (wide)" if w.feature_count >= 512 else "K1 3xTF32")}


def end_to_end(torch, dev, model, w, sr, rank, world, dist, a) -> dict:
    """The same metric through the public C-ABI host call (pinned host buffers,
    H2D + kernel + D2H inside the timed region), plus the reference's own call
    shape (TabNetModel.apply on float64 numpy)."""
    rows = sr.chunk
    xh = torch.from_numpy(W.make_inputs(w, rows, start=rank * rows)).pin_memory()
    oh = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in sr.runner.outputs.items()}
    np_out = {k: v.numpy() for k, v in oh.items()}
    xnp = xh.numpy()
    eng = model.engine(device=int(dev.index))
    for _ in range(max(2, a.warmup // 2)):
        eng.forward_host_f32(xnp, 0, np_out)
    steps = max(5, min(a.steps, 30))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.forward_host_f32(xnp, 0, np_out)
    el = time.perf_counter() - t0
    te = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    h2d = rows * w.feature_count * 4
    d2h = sum(v.numel() * v.element_size() for v in oh.values())
    out = {"value": world * rows * steps / float(te.item()), "unit": "rows/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": 1e3 * float(te.item()) / steps,
           "rows_per_step": rows,
           "path": ("tbn_forward_host (C-ABI, pinned host fp32 buffers; " +
                    ("one zero-copy kernel: x read and outputs written over PCIe by the kernel)" if rows <= 32768
                     else "3-stream chunked H2D/kernel/D2H)"))}
    if rows <= 262144:
        # the reference's own call shape: TabNetModel.apply on float64 numpy in/out
        # (network.py:195-267), host conversions included
        x64 = xnp.astype(np.float64)
        model.apply(x64)
        ta = []
        for _ in range(3):
            t0 = time.perf_counter()
            model.apply(x64)
            ta.append(time.perf_counter() - t0)
        out["apply_f64"] = {"value": rows / min(ta), "unit": "rows/s", "ms_per_call": 1e3 * min(ta),
                            "path": "TabNetModel.apply (float64 numpy in/out, tbn_forward_host_f64)"}
    return out


def x_dev(local):
    import torch
    return torch.device("cuda", local)


LAT_REPS = 1000


def latency_sweep(model, local, f):
    """HR shape, batches 1..1024 (BASELINE config 3): nearest-rank p50/p99 of the
    device-only kernel time (L2 flushed before each call) and of the end-to-end
    host call.  SURVEY.md §8(d) run 4: every power of two 1..1,024, 1,000 timed
    reps per batch size."""
    import torch
    from paper_2510_19689_b200.device import DeviceRunner
    res = {}
    eng = model.engine(device=local)
    runner = DeviceRunner(model, 1024, device=local)
    stream = torch.cuda.current_stream()
    w = W.WORKLOADS["hr_latency"]
    flush = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=x_dev(local))
    for b in [1 << i for i in range(11)]:
        x = torch.from_numpy(W.make_inputs(w, b)).cuda()
        for _ in range(20):
            runner.run(x)
        torch.cuda.synchronize()
        dev_ms = []
        for _ in range(LAT_REPS):
            # a queued spin keeps the GPU busy while the host enqueues the events
            # and the launch, so e0 -> e1 is device time only (no host overhead)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(len(dev_ms) & 0xFF)      # cold L2 for every timed call
            torch.cuda._sleep(100_000)
            e0.record(stream)
            runner.run(x)
            e1.record(stream)
            e1.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
        xh = torch.from_numpy(W.make_inputs(w, b)).pin_memory()
        oh = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in runner.views(b).items()}
        np_out = {k: v.numpy() for k, v in oh.items()}
        e2e_ms = []
        for i in range(LAT_REPS + 20):
            t0 = time.perf_counter()
            eng.forward_host_f32(xh.numpy(), 0, np_out)
            if i >= 20:
                e2e_ms.append(1e3 * (time.perf_counter() - t0))
        res[str(b)] = {"device_p50": nearest_rank(dev_ms, 50), "device_p99": nearest_rank(dev_ms, 99),
                       "e2e_p50": nearest_rank(e2e_ms, 50), "e2e_p99": nearest_rank(e2e_ms, 99)}
    return res


def main(argv=None):
    a = parse(argv)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this script under torch.distributed.run
        cmd = launch_cmd(a.gpus, sys.argv[1:] if argv is None else list(argv), free_port())
        os.execv(sys.executable, cmd)
    _, world, _ = dist_env()
    if a.gpus != world:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if a.dry_run:
        run_dry(a)
    elif a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
