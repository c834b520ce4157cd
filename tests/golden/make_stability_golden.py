"""Golden vectors for the stability consumer (interpret/stability.py), produced
by the UNMODIFIED reference in the builder container:

    python tests/golden/make_stability_golden.py

Cases: per-partition mean-importance matrices (random, with all-zero and
zero-mean-but-nonzero columns, exact ties across features, few/many
partitions) through ``stability_from_batches``, and one end-to-end
``stability_score`` of the reference's own ``TabNetModel`` on the HR workload
(weights regenerated from ``init_parameters(seed=0)``, trained regime), whose
per-partition means the GPU test compares against.  Only the .npz travels.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main() -> None:
    sys.path.insert(0, str(REF))
    sys.path.insert(0, str(OUT.parent.parent))
    from tabserve.interpret.stability import stability_from_batches, stability_score
    from tabserve.model.network import TabNetModel as RefModel
    from paper_2510_19689_b200 import workloads as W

    rng = np.random.default_rng(2510)
    cases = {}
    a = rng.random((6, 9))
    cases["random"] = a
    b = rng.random((4, 7))
    b[:, 2] = 0.0                    # all zero -> stability 1
    b[:, 5] = [0.3, -0.3, 0.1, -0.1]  # mean 0, not all zero -> stability 0
    b[:, 6] = b[:, 1]                # exact tie with feature 1
    cases["zeros_ties"] = b
    cases["two_partitions"] = rng.random((2, 35))
    cases["many_partitions"] = rng.dirichlet(np.ones(64), size=40)
    out = {}
    for name, m in cases.items():
        rep = stability_from_batches(m, sample_count=123, load_mode="offline")
        out[f"{name}__in"] = m
        out[f"{name}__names"] = np.array([f.name for f in rep.features])
        out[f"{name}__mean"] = np.array([f.mean_importance for f in rep.features])
        out[f"{name}__stability"] = np.array([f.stability for f in rep.features])
        out[f"{name}__rank_variance"] = np.array(rep.rank_variance)
        out[f"{name}__csv"] = np.array(rep.to_csv())
        out[f"{name}__json"] = np.array(rep.to_json())

    # end to end on the reference model (HR shape, trained regime)
    m = W.make_model("hr", "trained", model_cls=RefModel)
    x = W.make_inputs(W.WORKLOADS["hr"], 2050, seed=77).astype(np.float64)
    parts = 8
    per = x.shape[0] // parts
    means = np.stack([m.apply(x[i * per:(i + 1) * per]).importance.mean(axis=0) for i in range(parts)])
    rep = stability_score(m, x, parts)
    out["hr__x_seed"] = np.array(77)
    out["hr__rows"] = np.array(x.shape[0])
    out["hr__partitions"] = np.array(parts)
    out["hr__means"] = means
    out["hr__names"] = np.array([f.name for f in rep.features])
    out["hr__stability"] = np.array([f.stability for f in rep.features])
    out["hr__rank_variance"] = np.array(rep.rank_variance)
    np.savez_compressed(OUT / "stability.npz", **out)
    print("wrote", OUT / "stability.npz")


if __name__ == "__main__":
    main()
