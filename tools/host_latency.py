import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2510_19689_b200 import workloads as W
m = W.make_engine_model("hr", "trained", precision="bf16", device=0)
eng = m.engine(device=0)
for b in (1, 16, 256):
    x = torch.from_numpy(W.make_inputs(W.WORKLOADS["hr"], b)).pin_memory().numpy()
    outs = {"logits": np.empty((b, 2), np.float32), "probabilities": np.empty((b, 2), np.float32),
            "masks": np.empty((5, b, 35), np.float32), "importance": np.empty((b, 35), np.float32),
            "predicted_class": np.empty((b,), np.int32)}
    pin = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in outs.items()}
    ts = []
    for i in range(520):
        t0 = time.perf_counter()
        eng.forward_host_f32(x, 0, pin)
        if i >= 20: ts.append((time.perf_counter() - t0) * 1e6)
    ts.sort()
    print(sys.argv[1], "batch", b, "p50 %.1f us p99 %.1f" % (ts[len(ts)//2], ts[int(len(ts)*0.99)]))
