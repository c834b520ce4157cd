"""Kernel time vs rows with launches replayed from a CUDA graph (no host
launch overhead between back-to-back forwards)."""
import os
import sys
sys.path.insert(0, ".")
import torch
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.network import TabNetModel
from paper_2510_19689_b200.device import DeviceRunner

cfg = sys.argv[1] if len(sys.argv) > 1 else "hr"
rows_list = [int(v) for v in os.environ.get("ROWS", "128,18944,37888,56832,65536,75776,151552,303104").split(",")]
G = int(os.environ.get("G", "20"))
for prec in sys.argv[2:] or ["bf16"]:
    w = W.WORKLOADS[cfg]
    m = TabNetModel.from_reference(W.make_model(cfg, "trained"), precision=prec, device=0)
    maxr = max(rows_list)
    r = DeviceRunner(m, maxr, device=0)
    x = torch.from_numpy(W.make_inputs(w, maxr)).cuda()
    for rows in rows_list:
        xs = x[:rows].contiguous()
        outs = r.views(rows)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                r.run(xs, outs, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            st = torch.cuda.current_stream()
            for _ in range(G):
                r.run(xs, outs, stream=st)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / (3 * G)
        print(f"{cfg} {prec} rows={rows:7d} tiles/CTA~{rows/128/148:5.2f} t={t*1e3:8.1f} us  {rows/t/1e3:8.1f} Mrows/s")
