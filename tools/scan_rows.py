"""Kernel time vs rows (device path, CUDA events) to expose per-tile latency."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.network import TabNetModel
from paper_2510_19689_b200.device import DeviceRunner
cfg = sys.argv[1] if len(sys.argv) > 1 else "hr"
for prec in sys.argv[2:] or ["tf32x3", "tf32"]:
    w = W.WORKLOADS[cfg]
    m = TabNetModel.from_reference(W.make_model(cfg, "trained"), precision=prec, device=0)
    maxr = 148 * 128 * 16
    r = DeviceRunner(m, maxr, device=0)
    x = torch.from_numpy(W.make_inputs(w, maxr)).cuda()
    for rows in [int(v) for v in __import__('os').environ.get('ROWS', '128,37888,56832,65536,151552').split(',')]:
        xs = x[:rows].contiguous()
        for _ in range(3):
            r.run(xs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            r.run(xs)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10
        print(f"{cfg} {prec} rows={rows:7d} tiles/CTA~{rows/128/148:5.2f} t={t*1e3:8.1f} us  {rows/t/1e3:8.1f} Mrows/s")
