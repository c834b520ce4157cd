"""Where do the occasional 0.3-0.7 s request latencies of the 256-row GPU
serving case come from?  Records every TabNetModel.apply call's duration inside
the unmodified InferenceService and prints the slow ones next to the request
latency tail."""
import json
import sys
import threading
import time
sys.path.insert(0, "tools")
import serving_bench as sb  # noqa: E402
import paper_2510_19689_b200 as P  # noqa: E402
from paper_2510_19689_b200 import workloads as W  # noqa: E402

gpu = P.TabNetModel.from_reference(W.make_model("hr", "trained"), precision="bf16")
calls = []
orig = gpu.apply


def timed_apply(x, **kw):
    t0 = time.perf_counter()
    r = orig(x, **kw)
    calls.append((t0, time.perf_counter() - t0, x.shape[0], threading.get_ident()))
    return r


gpu.apply = timed_apply
for i in range(6):
    calls.clear()
    r = sb.run(gpu, 256, 400, 8, 256)
    d = sorted(c[1] for c in calls)
    slow = [(round(1e3 * c[1], 1), c[2]) for c in calls if c[1] > 0.02]
    print(json.dumps({"p99_ms": round(r["p99_ms"], 1), "rows_per_s": round(r["rows_per_s"]), "apply_calls": len(calls),
                      "apply_p50_ms": round(1e3 * d[len(d) // 2], 2), "apply_max_ms": round(1e3 * d[-1], 1),
                      "slow_apply": slow[:10]}), flush=True)
