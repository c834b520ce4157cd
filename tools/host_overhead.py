"""Where a 1-row host call's time goes: Python wrapper overhead, the raw
ctypes call with a prebuilt output struct, and the kernel's device time in the
same warm loop.  python tools/host_overhead.py"""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2510_19689_b200 import _native as N
from paper_2510_19689_b200 import workloads as W
from paper_2510_19689_b200.device import DeviceRunner

m = W.make_engine_model("hr", "trained", precision="bf16", device=0)
eng = m.engine(device=0)


def p50(fn, n=2000):
    for _ in range(100):
        fn()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t) * 1e6)
    ts.sort()
    return ts[n // 2]


x0 = np.empty((0, 35), np.float32)
o0 = {"logits": np.empty((0, 2), np.float32), "probabilities": np.empty((0, 2), np.float32),
      "masks": np.empty((5, 0, 35), np.float32), "importance": np.empty((0, 35), np.float32),
      "predicted_class": np.empty((0,), np.int32)}
print("python wrapper + ctypes, rows=0 (returns at once): %.2f us" % p50(lambda: eng.forward_host_f32(x0, 0, o0)))
for b in (1, 256):
    x = torch.from_numpy(W.make_inputs(W.WORKLOADS["hr"], b)).pin_memory().numpy()
    o = {k: torch.from_numpy(np.empty(v.shape[:-2] + (b,) + v.shape[-1:] if k == "masks" else (b,) + v.shape[1:],
                                      v.dtype)).pin_memory().numpy() for k, v in o0.items()}
    print(f"{b} rows, wrapper call p50: %.1f us" % p50(lambda: eng.forward_host_f32(x, 0, o)))
    st = N.TbnOutputs(*(N.ptr(o[k]) for k in ("logits", "probabilities", "masks", "importance", "predicted_class")))
    fh, h, xp, sref = eng._lib.tbn_forward_host, eng.handle, x.ctypes.data, C.byref(st)
    print(f"{b} rows, raw ctypes call p50: %.1f us" % p50(lambda: fh(h, xp, b, 0, sref)))
    r = DeviceRunner(m, b, device=0)
    xd = torch.from_numpy(x).cuda()
    for _ in range(20):
        r.run(xd)
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(50_000)
        e0.record()
        r.run(xd)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{b} rows, device time (warm L2) p50: %.1f us" % ts[100])
