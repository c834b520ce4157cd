import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2510_19689_b200 import workloads as W
m = W.make_engine_model("hr", "trained", precision="bf16", device=0)
eng = m.engine(device=0)
x0 = np.empty((0, 35), np.float32)
outs = {"logits": np.empty((0, 2), np.float32), "probabilities": np.empty((0, 2), np.float32),
        "masks": np.empty((5, 0, 35), np.float32), "importance": np.empty((0, 35), np.float32),
        "predicted_class": np.empty((0,), np.int32)}
for _ in range(100): eng.forward_host_f32(x0, 0, outs)
t = time.perf_counter()
for _ in range(2000): eng.forward_host_f32(x0, 0, outs)
print("python+ctypes overhead per call (rows=0): %.2f us" % ((time.perf_counter() - t) / 2000 * 1e6))
# C-level: a 1-row call timed with the device time via events on a side probe
x1 = torch.from_numpy(W.make_inputs(W.WORKLOADS["hr"], 1)).pin_memory().numpy()
o1 = {k: torch.from_numpy(np.empty(v.shape[:-2] + (1,) + v.shape[-1:] if k == "masks" else (1,) + v.shape[1:], v.dtype)).pin_memory().numpy() for k, v in outs.items()}
for _ in range(50): eng.forward_host_f32(x1, 0, o1)
ts = []
for _ in range(500):
    t = time.perf_counter(); eng.forward_host_f32(x1, 0, o1); ts.append((time.perf_counter() - t) * 1e6)
ts.sort(); print("1-row call p50 %.1f us" % ts[250])
