"""A/B of the fp32 CUDA-core kernels (row-blocked vs per-row, TBN_SIMT_PER_ROW=1):
time one device forward and dump the outputs for a bitwise comparison.
    python tools/simt_ab.py <tag>    -> /tmp/simt_<tag>.npz (compare two tags in the same box session)"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner
from paper_2510_19689_b200.network import TabNetModel

tag = sys.argv[1]
res = {}
for cfg, rows in (("wide", 32768), ("bls", 65536), ("hr", 65536), ("adult", 4099)):
    m = TabNetModel.from_reference(W.make_model(cfg, "trained"), precision="fp32", device=0)
    r = DeviceRunner(m, rows, device=0)
    x = torch.from_numpy(W.make_inputs(W.WORKLOADS[cfg], rows)).cuda()
    r.run(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        out = r.run(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{tag} {cfg} rows={rows} {ms:.2f} ms  {rows / ms * 1e3:.3g} rows/s")
    for k, v in out.items():
        res[f"{cfg}_{k}"] = v.cpu().numpy()
np.savez(f"/tmp/simt_{tag}.npz", **res)
