"""Wall time of the reference-facing TabNetModel.apply (float64 numpy in/out)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_19689_b200 import workloads as W
for prec in sys.argv[1:] or ["bf16", "tf32x3"]:
    m = W.make_engine_model("hr", "trained", precision=prec)
    x = W.make_inputs(W.WORKLOADS["hr"], 65536).astype(np.float64)
    m.apply(x)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); m.apply(x); ts.append(time.perf_counter() - t0)
    print(prec, "apply(65536 rows, f64 numpy) ms: min %.1f median %.1f" % (1e3 * min(ts), 1e3 * sorted(ts)[2]))
