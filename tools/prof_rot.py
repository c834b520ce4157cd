"""Driver for steady-state DRAM-traffic captures (ncu --replay-mode application
--cache-control none): back-to-back fused forwards over rotating input/output
sets larger than L2, exactly as bench.py's timed graph does, so the profiled
launch sees the HBM traffic of the steady state (its inputs not in L2, the
previous launches' dirty outputs being written back).
  python tools/prof_rot.py --config hr --precision bf16 [--iters 24]"""
import argparse
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="hr")
ap.add_argument("--precision", default="bf16")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--iters", type=int, default=24)
a = ap.parse_args()
w = W.WORKLOADS[a.config]
rows = a.rows or min(w.batch, 262144)
bpr = W.algorithmic_counts(w)["bytes_per_row"]
nsets = max(2, min(8, int(np.ceil(2.5 * 126 * 2**20 / (rows * bpr)))))
m = W.make_engine_model(a.config, "trained", precision=a.precision, device=0)
r = DeviceRunner(m, rows, device=0)
xs = [torch.from_numpy(W.make_inputs(w, rows, start=i * rows)).cuda() for i in range(nsets)]
outs = [r.alloc_outputs(rows) for _ in range(nsets)]
for i in range(a.iters):
    r.run(xs[i % nsets], outs[i % nsets])
torch.cuda.synchronize()
print("done", nsets, "sets")
