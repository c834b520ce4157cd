"""Quick K3 (wide, bf16) check against the golden oracle outputs."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
sys.path.insert(0, "tests")
from conftest import load_golden
from parity import compare
import paper_2510_19689_b200 as P
for regime in ("trained", "init"):
    g = load_golden(f"wide_{regime}")
    f, nd, na, s, c = (int(v) for v in g["shape"])
    cfg = P.ModelConfig(feature_count=f, n_classes=c, n_d=nd, n_a=na, n_steps=s)
    p = P.init_parameters(cfg)
    if regime == "trained":
        for k in list(p):
            if k.endswith("_att_W"):
                p[k] = p[k] * 16.0
        p["head_W"] = p["head_W"] * 8.0
    m = P.TabNetModel(config=cfg, params=p, norm_mean=g["norm_mean"], norm_var=g["norm_var"],
                      model_version="w", precision="bf16")
    t0 = time.time()
    r = m.apply(g["x"].astype(np.float64))
    print(regime, "apply s", round(time.time() - t0, 3), flush=True)
    rep = compare(g, dict(logits=r.logits, probabilities=r.probabilities, masks=r.masks, importance=r.importance),
                  delta=0.0, gap=5e-2, rtol=1.5e-1, atol={"probabilities": 3e-2, "logits": 2e-1})
    print(regime, rep.summary()[:400])
    print("cls agree", np.mean(np.argmax(r.probabilities, 1) == np.argmax(g["probabilities"], 1)),
          "max|dprob|", np.abs(r.probabilities - g["probabilities"]).max(),
          "max|dmask|", np.abs(r.masks - g["masks"]).max(), "max|dimp|", np.abs(r.importance - g["importance"]).max())
