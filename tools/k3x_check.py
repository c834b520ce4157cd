import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W
from oracle import tabnet_oracle as O
sys.path.insert(0, "tests")
from parity import compare
prec = sys.argv[1] if len(sys.argv) > 1 else "tf32x3"
m = P.TabNetModel.from_reference(W.make_model("wide", "trained"), precision=prec, device=0)
print("kernel ok; engine", m.engine())
for rows in (160, 2000):
    x = W.make_inputs(W.WORKLOADS["wide"], rows, seed=4242).astype(np.float64)
    r = m.apply(x)
    ref = O.apply_model(m, x, diagnostics=True)
    zs, tau = ref["z_shift"], ref["tau"]
    ref["margin"] = np.abs(zs - tau[..., None]).min(axis=2) / np.maximum(np.abs(zs).max(axis=2), 1e-300)
    p = np.sort(ref["probabilities"], axis=1); ref["top2_gap"] = p[:, -1] - p[:, -2]
    got = dict(logits=r.logits, probabilities=r.probabilities, masks=r.masks, importance=r.importance)
    rep = compare(ref, got)
    print(prec, rows, "ok" if rep.ok else "FAIL", "exempt", len(rep.exempt_rows), "sup", rep.support_mismatch_rows[:5],
          "cls", rep.class_mismatch_rows[:5], "viol", rep.viol,
          {k: float(f"{v:.3g}") for k, v in rep.max_err.items() if not k.endswith("_rel")})
