import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_2510_19689_b200 import workloads as W
m = W.make_engine_model("hr", "trained", precision=sys.argv[1] if len(sys.argv) > 1 else "bf16", device=0)
res = {}
for rows in (1, 16, 128, 512, 2048, 8192, 32768):
    x = W.make_inputs(W.WORKLOADS["hr"], rows).astype(np.float64)
    for _ in range(5): m.apply(x)
    ts = []
    for _ in range(50):
        t0 = time.perf_counter(); m.apply(x); ts.append(time.perf_counter() - t0)
    ts.sort(); res[rows] = round(1e6 * ts[len(ts)//2], 1)
print(json.dumps(res))
