"""Generate the golden parity fixtures by running the UNMODIFIED reference.

Run in the builder container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``tabserve`` from ``/root/reference/pkg/src`` and, for every
BASELINE config shape and both weight regimes of SURVEY.md §8(d), records the
reference's ``TabNetModel.apply`` outputs on seeded float32 inputs, plus the
tie-margin diagnostics the comparator needs.  Weights are NOT stored (they are
regenerated from ``init_parameters(seed=0)``); a SHA-256 of the reference's
flattened params pins that the regeneration is bit-identical.  Also stores the
SPEC.md sparsemax/attentive_step examples and a .tbnt byte stream.

Nothing at GPU-test time reads /root/reference: only these .npz files travel.
"""
from __future__ import annotations

import hashlib
import io
import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

# (name, config_id, F, n_d, n_a, n_steps, n_classes, rows)
SHAPES = [
    ("adult", 0, 14, 8, 8, 3, 2, 512),
    ("hr", 1, 35, 16, 16, 5, 2, 512),
    ("bls", 2, 64, 32, 32, 5, 2, 256),
    ("wide", 4, 512, 64, 64, 8, 10, 24),
]


def params_digest(params: dict) -> str:
    h = hashlib.sha256()
    for k in sorted(params):
        h.update(k.encode())
        h.update(np.ascontiguousarray(params[k], dtype="<f8").tobytes())
    return h.hexdigest()


def margins(z_shift: np.ndarray, tau: np.ndarray) -> np.ndarray:
    """Per (step,row) relative sparsemax tie margin min_i|z_i - tau| / max|z|."""
    scale = np.maximum(np.abs(z_shift).max(axis=2), 1e-300)
    return np.abs(z_shift - tau[..., None]).min(axis=2) / scale


def run(ref_model_mod, sparsemax_mod, name, cid, f, nd, na, s, c, rows, regime):
    from tabserve.model import ModelConfig, TabNetModel, init_parameters
    cfg = ModelConfig(feature_count=f, n_classes=c, n_d=nd, n_a=na, n_steps=s, seed=0)
    params = init_parameters(cfg)
    if regime == "trained":
        for k in list(params):
            if k.endswith("_att_W"):
                params[k] = params[k] * 16.0
        params["head_W"] = params["head_W"] * 8.0
    rng = np.random.default_rng(7)
    mean = rng.standard_normal(f)
    var = rng.uniform(0.5, 2.0, f)
    model = TabNetModel(config=cfg, params=params, norm_mean=mean, norm_var=var,
                        model_version=f"{name}-{regime}-v1")
    x32 = np.random.default_rng(1000 + cid).standard_normal((rows, f), dtype=np.float32)
    res = model.apply(x32.astype(np.float64))

    # diagnostics: re-run the reference's own sparsemax on the reference's own z
    # (monkeypatch-free: wrap network.sparsemax to capture its inputs)
    captured = []
    orig = ref_model_mod.sparsemax

    def spy(z):
        out = orig(z)
        zz = np.asarray(z, dtype=np.float64)
        zs = zz - zz.max(axis=1, keepdims=True)
        # tau recovered exactly as sparsemax.py:33-39 computes it
        z_sorted = np.sort(zs, axis=1)[:, ::-1]
        cs = np.cumsum(z_sorted, axis=1)
        kr = np.arange(1, zs.shape[1] + 1, dtype=np.float64)
        k = np.count_nonzero(1.0 + kr * z_sorted > cs, axis=1)
        tau = (cs[np.arange(zs.shape[0]), k - 1] - 1.0) / k
        captured.append((zs, tau))
        return out

    ref_model_mod.sparsemax = spy
    try:
        res2 = model.apply(x32.astype(np.float64))
    finally:
        ref_model_mod.sparsemax = orig
    assert np.array_equal(res.masks, res2.masks)
    z_shift = np.stack([z for z, _ in captured])
    tau = np.stack([t for _, t in captured])
    p = np.sort(res.probabilities, axis=1)
    top2 = p[:, -1] - p[:, -2]
    out = dict(
        x=x32, norm_mean=mean, norm_var=var,
        logits=res.logits, probabilities=res.probabilities, masks=res.masks,
        importance=res.importance, margin=margins(z_shift, tau), tau=tau,
        top2_gap=top2,
        shape=np.array([f, nd, na, s, c], dtype=np.int64),
        gamma=np.float64(cfg.gamma),
        params_sha256=np.array(params_digest(params)),
        regime=np.array(regime),
    )
    return out, model


def fallback_case():
    """Rows where every step's decision output is zero -> importance falls back to
    mean(masks) (network.py:258-261).  Found by scanning Adult init weights with
    identity norm stats (3/65,536 rows)."""
    from tabserve.model import ModelConfig, TabNetModel, init_parameters
    cfg = ModelConfig(feature_count=14, n_classes=2, n_d=8, n_a=8, n_steps=3, seed=0)
    model = TabNetModel(config=cfg, params=init_parameters(cfg), norm_mean=np.zeros(14),
                        norm_var=np.ones(14) - 1e-8, model_version="adult-fallback")
    x = np.random.default_rng(4242).standard_normal((65536, 14), dtype=np.float32)
    res = model.apply(x.astype(np.float64))
    agg_tot = None
    # rows where importance == mean of masks (fallback fired)
    fb = np.all(res.importance == res.masks.mean(axis=0), axis=1)
    idx = np.nonzero(fb)[0]
    # keep the fallback rows and some neighbours
    keep = np.unique(np.concatenate([idx, np.arange(64)]))
    xs = x[keep]
    r = model.apply(xs.astype(np.float64))
    return dict(x=xs, norm_mean=model.norm_mean, norm_var=model.norm_var,
                logits=r.logits, probabilities=r.probabilities, masks=r.masks,
                importance=r.importance, fallback_rows=np.nonzero(
                    np.all(r.importance == r.masks.mean(axis=0), axis=1))[0],
                shape=np.array([14, 8, 8, 3, 2], dtype=np.int64), gamma=np.float64(1.3),
                params_sha256=np.array(params_digest(model.params)))


def spec_examples():
    from tabserve.model import sparsemax, project_simplex_bruteforce
    c = 0.37
    cases = {
        "sm_a": np.array([0.6, 0.4]),
        "sm_b": np.array([c, c, c]),
        "sm_c": np.array([2.0, 1.0, 0.1]),
    }
    out = {}
    for k, v in cases.items():
        out[k + "_in"] = v
        out[k + "_out"] = sparsemax(v)
    rng = np.random.default_rng(3)
    z = rng.standard_normal((1000, 5)) * 2
    out["bf_in"] = z
    out["bf_out"] = np.stack([project_simplex_bruteforce(r) for r in z])
    # random widths 1..64
    zz = rng.standard_normal((200, 64)) * 3
    out["rand64_in"] = zz
    out["rand64_out"] = sparsemax(zz)
    zt = rng.standard_normal((64, 512)) * 5
    out["rand512_in"] = zt
    out["rand512_out"] = sparsemax(zt)
    return out


def tbnt_stream():
    from tabserve.model import ModelConfig, TabNetModel, init_parameters, save_model
    cfg = ModelConfig(feature_count=14, n_classes=2, n_d=8, n_a=8, n_steps=3, seed=0)
    rng = np.random.default_rng(7)
    model = TabNetModel(config=cfg, params=init_parameters(cfg),
                        norm_mean=rng.standard_normal(14), norm_var=rng.uniform(0.5, 2.0, 14),
                        model_version="adult-tbnt-v1")
    return save_model(model)


def main():
    sys.path.insert(0, str(REF))
    import tabserve.model.network as net
    import tabserve.model.sparsemax as sm
    print("numpy", np.__version__)
    for (name, cid, f, nd, na, s, c, rows) in SHAPES:
        for regime in ("init", "trained"):
            out, _ = run(net, sm, name, cid, f, nd, na, s, c, rows, regime)
            path = OUT / f"{name}_{regime}.npz"
            np.savez_compressed(path, numpy_version=np.array(np.__version__), **out)
            print(path.name, path.stat().st_size, "bytes; min margin",
                  float(out["margin"].min()))
    np.savez_compressed(OUT / "adult_fallback.npz", **fallback_case())
    np.savez_compressed(OUT / "sparsemax_spec.npz", **spec_examples())
    (OUT / "adult.tbnt").write_bytes(tbnt_stream())
    print("done")


if __name__ == "__main__":
    main()
