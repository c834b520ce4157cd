import numpy as np, sys, time
sys.path.insert(0, '.')
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from oracle import tabnet_oracle as O
for name in ("adult", "hr", "bls"):
    for prec in ("tf32x3", "tf32", "bf16"):
        m = P.TabNetModel.from_reference(W.make_model(name, "trained"), precision=prec)
        x = W.make_inputs(W.WORKLOADS[name], 1000).astype(np.float64)
        t0 = time.time()
        r = m.apply(x)
        ref = O.apply_model(m, x)
        print(name, prec, "time %.3f" % (time.time() - t0),
              "cls_agree", np.mean(np.argmax(r.probabilities, 1) == np.argmax(ref["probabilities"], 1)),
              "dprob %.2e" % np.abs(r.probabilities - ref["probabilities"]).max(),
              "dmask %.2e" % np.abs(r.masks - ref["masks"]).max(),
              "dimp %.2e" % np.abs(r.importance - ref["importance"]).max(), flush=True)
