"""The oracle is pinned to the reference: bitwise equal to outputs the
unmodified reference produced (tests/golden/make_golden.py)."""
import hashlib

import numpy as np
import pytest

from conftest import load_golden
from oracle import tabnet_oracle as O
from paper_2510_19689_b200 import ModelConfig, init_parameters

CASES = [f"{n}_{r}" for n in ("adult", "hr", "bls", "wide") for r in ("init", "trained")]


def params_for(g):
    f, nd, na, s, c = (int(v) for v in g["shape"])
    p = O.init_parameters(f, c, nd, na, s, seed=0)
    if str(g["regime"]) == "trained":
        for k in list(p):
            if k.endswith("_att_W"):
                p[k] = p[k] * 16.0
        p["head_W"] = p["head_W"] * 8.0
    return p, (f, nd, na, s, c)


def digest(params):
    h = hashlib.sha256()
    for k in sorted(params):
        h.update(k.encode())
        h.update(np.ascontiguousarray(params[k], dtype="<f8").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("case", CASES)
def test_oracle_bitwise_equals_reference(case):
    g = load_golden(case)
    p, (f, nd, na, s, c) = params_for(g)
    assert digest(p) == str(g["params_sha256"])
    out = O.apply(p, g["norm_mean"], g["norm_var"], n_d=nd, n_steps=s, gamma=float(g["gamma"]),
                  x=g["x"].astype(np.float64), diagnostics=True)
    for k in ("logits", "probabilities", "masks", "importance"):
        assert np.array_equal(out[k], g[k]), k
    assert np.array_equal(out["tau"], g["tau"])


@pytest.mark.parametrize("case", CASES)
def test_package_init_parameters_matches_reference(case):
    g = load_golden(case)
    f, nd, na, s, c = (int(v) for v in g["shape"])
    p = init_parameters(ModelConfig(feature_count=f, n_classes=c, n_d=nd, n_a=na, n_steps=s))
    if str(g["regime"]) == "trained":
        for k in list(p):
            if k.endswith("_att_W"):
                p[k] = p[k] * 16.0
        p["head_W"] = p["head_W"] * 8.0
    assert digest(p) == str(g["params_sha256"])


def test_oracle_fallback_rows():
    g = load_golden("adult_fallback")
    f, nd, na, s, c = (int(v) for v in g["shape"])
    p = O.init_parameters(f, c, nd, na, s, seed=0)
    assert digest(p) == str(g["params_sha256"])
    out = O.apply(p, g["norm_mean"], g["norm_var"], n_d=nd, n_steps=s, gamma=1.3,
                  x=g["x"].astype(np.float64))
    assert np.array_equal(out["importance"], g["importance"])
    assert len(g["fallback_rows"]) >= 1
    fb = g["fallback_rows"]
    assert np.array_equal(out["importance"][fb], out["masks"].mean(axis=0)[fb])


def test_sparsemax_spec_examples():
    g = load_golden("sparsemax_spec")
    for k in ("sm_a", "sm_b", "sm_c"):
        assert np.array_equal(O.sparsemax(g[k + "_in"]), g[k + "_out"])
    np.testing.assert_allclose(O.sparsemax(np.array([0.6, 0.4])), [0.6, 0.4], atol=1e-15)
    np.testing.assert_allclose(O.sparsemax(np.array([2.0, 1.0, 0.1])), [1.0, 0.0, 0.0])
    assert np.array_equal(O.sparsemax(g["rand64_in"]), g["rand64_out"])
    assert np.array_equal(O.sparsemax(g["rand512_in"]), g["rand512_out"])
    # acceptance #6: brute force agreement within 1e-8 on 5-vectors
    np.testing.assert_allclose(O.sparsemax(g["bf_in"]), g["bf_out"], atol=1e-8)


def test_sparsemax_invariants():
    rng = np.random.default_rng(11)
    for n in (1, 2, 7, 35, 64):
        z = rng.standard_normal((500, n)) * 4
        m = O.sparsemax(z)
        assert np.all(m >= 0)
        np.testing.assert_allclose(m.sum(axis=1), 1.0, atol=1e-12)
        np.testing.assert_allclose(O.sparsemax(z + 3.7), m, atol=1e-12)
    with pytest.raises(O.OracleInputError):
        O.sparsemax(np.array([1.0, np.nan]))
    with pytest.raises(O.OracleInputError):
        O.sparsemax(np.array([]))
