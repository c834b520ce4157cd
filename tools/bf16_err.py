"""Full-size HR error distribution of a single-pass mode vs the oracle."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from oracle import tabnet_oracle as O
prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
m = P.TabNetModel.from_reference(W.make_model("hr", "trained"), precision=prec)
x = W.make_inputs(W.WORKLOADS["hr"], 65536).astype(np.float64)
ref = O.apply_model(m, x)
r = m.apply(x)
me = np.abs(r.masks - ref["masks"]).max(axis=2).max(axis=0)       # per row, worst step
ie = np.abs(r.importance - ref["importance"]).max(axis=1)
pe = np.abs(r.probabilities - ref["probabilities"]).max(axis=1)
for nm, e in (("mask", me), ("importance", ie), ("prob", pe)):
    print(prec, nm, "max %.3g p99.9 %.3g p99 %.3g median %.3g" % (e.max(), np.quantile(e, 0.999), np.quantile(e, 0.99), np.median(e)))
cls = np.argmax(r.probabilities, 1) != np.argmax(ref["probabilities"], 1)
ps = np.sort(ref["probabilities"], 1); gap = ps[:, -1] - ps[:, -2]
print(prec, "class flips", int(cls.sum()), "max gap among flips", float(gap[cls].max()) if cls.any() else 0.0)
