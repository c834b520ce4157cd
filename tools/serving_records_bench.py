"""Host time of response building: the reference's per-row loop
(service.py:176-183) vs serving.build_records, on ForwardResult-shaped float64
arrays (host-only work; no GPU needed).
    python tools/serving_records_bench.py"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2510_19689_b200 as P
from paper_2510_19689_b200.serving import build_records

def loop(r, n):
    out = []
    for j in range(n):
        out.append({"prediction": int(np.argmax(r.probabilities[j])),
                    "probabilities": r.probabilities[j].tolist(),
                    "masks": r.masks[:, j, :].tolist(),
                    "importance": r.importance[j].tolist()})
    return out

rng = np.random.default_rng(0)
for name, (c, s, f) in {"hr": (2, 5, 35), "adult": (2, 3, 14), "wide": (10, 8, 512)}.items():
    for b in (1, 256, 1024):
        r = P.ForwardResult(logits=rng.random((b, c)), probabilities=rng.random((b, c)),
                            masks=rng.random((s, b, f)), importance=rng.random((b, f)))
        ts = {}
        for label, fn in (("loop", lambda: loop(r, b)), ("vectorized", lambda: build_records(r))):
            fn()
            reps = max(3, int(2000 / b))
            t0 = time.perf_counter()
            for _ in range(reps):
                fn()
            ts[label] = (time.perf_counter() - t0) / reps * 1e6
        assert loop(r, b) == build_records(r)
        print(f"{name:6s} batch {b:5d}: loop {ts['loop']:9.1f} us  vectorized {ts['vectorized']:9.1f} us  "
              f"x{ts['loop'] / ts['vectorized']:.2f}")
