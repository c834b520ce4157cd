"""Dev A/B timing of one kernel instance: device time per launch of a CUDA graph
of back-to-back forwards over rotating input/output sets (> L2), at several
batch sizes, plus a quick parity spot-check against the oracle (test-only
import).  python tools/k2_time.py [config] [precision]"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner

cfg = sys.argv[1] if len(sys.argv) > 1 else "hr"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
label = os.environ.get("LABEL", "")
w = W.WORKLOADS[cfg]
m = W.make_engine_model(cfg, "trained", precision=prec, device=0)
bpr = W.algorithmic_counts(w)["bytes_per_row"]
for rows in [int(v) for v in os.environ.get("ROWS", "128,8192,65536,262144").split(",")]:
    nsets = max(2, min(8, int(np.ceil(2.5 * 126 * 2**20 / (rows * bpr)))))
    r = DeviceRunner(m, rows, device=0)
    xs = [torch.randn(rows, w.feature_count, device="cuda", generator=torch.Generator("cuda").manual_seed(i))
          for i in range(nsets)]
    outs = [r.alloc_outputs(rows) for _ in range(nsets)]
    for i in range(3):
        r.run(xs[i % nsets], outs[i % nsets])
    torch.cuda.synchronize()
    K = 20
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(K):
                r.run(xs[i % nsets], outs[i % nsets], stream=s)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / K)
    frac = rows * bpr / (best * 1e-3) / 6536.4e9
    print(f"{label} {cfg} {prec} rows={rows:7d} t={best*1e3:9.2f} us  {rows/best/1e6:8.3f} Grows/s  hbm_frac={frac:.3f}",
          flush=True)
if os.environ.get("PARITY", "1") == "1":
    from oracle import tabnet_oracle as O   # checker only
    x = W.make_inputs(w, 2048).astype(np.float64)
    res = m.apply(x)
    ref = O.apply_model(m, x)
    mass = np.abs(ref["masks"]).sum(-1)
    merr = (np.abs(res.masks - ref["masks"]).max(-1) / np.maximum(mass, 1e-30)).max()
    cls = np.mean(np.argmax(res.probabilities, 1) == np.argmax(ref["probabilities"], 1))
    print(f"{label} parity: class-agree={cls:.4f} max|dprob|={np.abs(res.probabilities - ref['probabilities']).max():.2e} "
          f"mask-err/rowmass={merr:.3e} max|dimp|={np.abs(res.importance - ref['importance']).max():.2e}", flush=True)
