"""Minimal driver for ncu: a few fused forwards of one config (device path)."""
import argparse, sys
sys.path.insert(0, ".")
import torch
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.network import TabNetModel
from paper_2510_19689_b200.device import DeviceRunner

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="hr")
ap.add_argument("--precision", default="tf32x3")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
w = W.WORKLOADS[a.config]
rows = a.rows or w.batch
m = W.make_engine_model(a.config, "trained", precision=a.precision, device=0)
r = DeviceRunner(m, rows, device=0)
x = torch.from_numpy(W.make_inputs(w, rows)).cuda()
for _ in range(a.iters):
    r.run(x)
torch.cuda.synchronize()
print("done")
