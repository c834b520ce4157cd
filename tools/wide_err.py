"""Wide (F=512) bf16 error distribution against the oracle on N rows."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from oracle import tabnet_oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
for regime in ("trained", "init"):
    m = W.make_engine_model("wide", regime, precision="bf16")
    x = W.make_inputs(W.WORKLOADS["wide"], n).astype(np.float64)
    ref = O.apply_model(m, x)
    r = m.apply(x)
    me = np.abs(r.masks - ref["masks"]).max(axis=2).max(axis=0)
    ie = np.abs(r.importance - ref["importance"]).max(axis=1)
    pe = np.abs(r.probabilities - ref["probabilities"]).max(axis=1)
    ps = np.sort(ref["probabilities"], 1); gap = ps[:, -1] - ps[:, -2]
    flips = np.argmax(r.probabilities, 1) != np.argmax(ref["probabilities"], 1)
    print(regime, "mask max %.3g p99 %.3g | imp max %.3g | prob max %.3g | class flips %d (max gap %.2g)" % (
        me.max(), np.quantile(me, 0.99), ie.max(), pe.max(), flips.sum(), gap[flips].max() if flips.any() else 0))
