"""Where the float64 apply() call's time goes (HR @ 65,536, bf16): fresh output
allocation + first touch, the C-ABI f64 host call into pre-touched arrays, and
the whole apply().  Prints one JSON line."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_19689_b200 import workloads as W        # noqa: E402
from paper_2510_19689_b200 import _native as N          # noqa: E402


def best(fn, reps=7):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * sorted(ts)[len(ts) // 2]


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    w = W.WORKLOADS["hr"]
    model = W.make_engine_model("hr", "trained", precision="bf16", device=0)
    x = W.make_inputs(w, rows).astype(np.float64)
    eng = model.engine()
    cfg = model.config
    b, f, c, s = rows, cfg.feature_count, eng.n_out, cfg.n_steps

    def alloc():
        return dict(logits=np.empty((b, c)), probabilities=np.empty((b, c)), masks=np.empty((s, b, f)),
                    importance=np.empty((b, f)), predicted_class=np.empty(b, dtype=np.int32))

    def alloc_touch():
        o = alloc()
        for v in o.values():
            v.fill(0)
        return o

    pre = alloc_touch()

    def call(o=pre):
        t = N.TbnOutputs(*(N.ptr(o[k]) for k in ("logits", "probabilities", "masks", "importance",
                                                  "predicted_class")))
        N.check(eng._lib.tbn_forward_host_f64(eng.handle, x.ctypes.data, b, 0, C.byref(t)), "f64")

    res = {"rows": rows,
           "alloc_ms": best(alloc),
           "alloc_touch_ms": best(alloc_touch),
           "host_f64_pretouched_ms": best(call),
           "host_f64_fresh_ms": best(lambda: call(alloc())),
           "apply_ms": best(lambda: model.apply(x))}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
