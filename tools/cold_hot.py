"""Kernel time with hot vs rotating (HBM-cold) inputs/outputs, CUDA-graph replay."""
import os, sys
sys.path.insert(0, ".")
import torch
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.network import TabNetModel
from paper_2510_19689_b200.device import DeviceRunner
cfg = sys.argv[1] if len(sys.argv) > 1 else "hr"
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
w = W.WORKLOADS[cfg]
rows = w.batch
m = TabNetModel.from_reference(W.make_model(cfg, "trained"), precision=prec, device=0)
r = DeviceRunner(m, rows, device=0)
N = 6
xs = [torch.from_numpy(W.make_inputs(w, rows, start=i * rows)).cuda() for i in range(N)]
outs = [r.alloc_outputs(rows) for _ in range(N)]
def timeit(xi, oi, G=24):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        r.run(xs[0], outs[0], stream=s)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st = torch.cuda.current_stream()
        for i in range(G):
            r.run(xs[xi(i)], outs[oi(i)], stream=st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / G * 1e3
print(cfg, prec, "hot x, hot out      ", round(timeit(lambda i: 0, lambda i: 0), 1), "us")
print(cfg, prec, "rotating x, hot out ", round(timeit(lambda i: i % N, lambda i: 0), 1), "us")
print(cfg, prec, "hot x, rotating out ", round(timeit(lambda i: 0, lambda i: i % N), 1), "us")
print(cfg, prec, "rotating both       ", round(timeit(lambda i: i % N, lambda i: i % N), 1), "us")
r2 = DeviceRunner(m, rows, device=0, outputs=("logits", "probabilities", "predicted_class"))
outs2 = [r2.alloc_outputs(rows) for _ in range(N)]
r, outs = r2, outs2
print(cfg, prec, "predict-only rotating", round(timeit(lambda i: i % N, lambda i: i % N), 1), "us")
