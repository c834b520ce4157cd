"""CPU oracle for the TabNet predict+explain hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped path (``paper_2510_19689_b200``)
runs on the GPU through ``libtabnet_b200.so`` and fails loudly without it.

It is a float64 NumPy restatement of the reference algorithm, operation for
operation, so that its outputs are *bitwise identical* to the reference's
``TabNetModel.apply`` on the same inputs (pinned by ``tests/test_oracle.py``
against ``tests/golden/*.npz``, which ``tests/golden/make_golden.py`` generated
by importing the unmodified reference from ``/root/reference``).

Reference anchors (``/root/reference/pkg/src/tabserve/``):
  * ``model/network.py:58-61``   ``_glu``
  * ``model/network.py:71-97``   ``init_parameters``
  * ``model/network.py:118-120`` ``normalize``
  * ``model/network.py:124-141`` ``_transform``
  * ``model/network.py:170-191`` ``attentive_step``
  * ``model/network.py:195-267`` ``apply``
  * ``model/sparsemax.py:13-41`` ``sparsemax``
  * ``model/sparsemax.py:60-84`` ``project_simplex_bruteforce``
The arithmetic itself is executed by NumPy (``einsum``, ``sort``, ``cumsum``,
``exp``); the reference pins ``numpy>=1.23`` unversioned
(``pkg/pyproject.toml:11``).  Goldens were produced with NumPy 2.3.5.
"""
from __future__ import annotations

import math

import numpy as np

NORM_EPS = 1e-8                      # network.py:27
RESIDUAL_SCALE = math.sqrt(0.5)      # network.py:29


class OracleInputError(ValueError):
    """Mirror of the reference's InvalidInputError for the oracle itself."""


def init_parameters(feature_count: int, n_classes: int, n_d: int, n_a: int,
                    n_steps: int, seed: int = 0) -> dict[str, np.ndarray]:
    """Seeded uniform fan-in init, same draw order as network.py:71-97."""
    rng = np.random.default_rng(seed)
    h = n_d + n_a
    f = feature_count

    def uniform(fan_in: int, shape: tuple[int, ...]) -> np.ndarray:
        bound = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-bound, bound, size=shape)

    params: dict[str, np.ndarray] = {
        "shared1_W": uniform(f, (f, 2 * h)),
        "shared1_b": np.zeros(2 * h),
        "shared2_W": uniform(h, (h, 2 * h)),
        "shared2_b": np.zeros(2 * h),
        "head_W": uniform(n_d, (n_d, n_classes)),
        "head_b": np.zeros(n_classes),
    }
    for s in range(n_steps + 1):
        params[f"step{s}_fc1_W"] = uniform(h, (h, 2 * h))
        params[f"step{s}_fc1_b"] = np.zeros(2 * h)
        params[f"step{s}_fc2_W"] = uniform(h, (h, 2 * h))
        params[f"step{s}_fc2_b"] = np.zeros(2 * h)
    for s in range(1, n_steps + 1):
        params[f"step{s}_att_W"] = uniform(n_a, (n_a, f))
        params[f"step{s}_att_b"] = np.zeros(f)
    return params


def sparsemax(logits: np.ndarray, *, return_tau: bool = False):
    """Row-wise simplex projection, sparsemax.py:13-41 step for step."""
    z = np.asarray(logits, dtype=np.float64)
    if z.size == 0:
        raise OracleInputError("sparsemax input must have length >= 1")
    if not np.all(np.isfinite(z)):
        raise OracleInputError("sparsemax input must be finite")
    squeeze = z.ndim == 1
    if squeeze:
        z = z[None, :]
    z = z - np.max(z, axis=1, keepdims=True)                       # :32
    z_sorted = np.sort(z, axis=1)[:, ::-1]                         # :33
    n = z.shape[1]
    k_range = np.arange(1, n + 1, dtype=np.float64)
    cumsum = np.cumsum(z_sorted, axis=1)                           # :36
    support = 1.0 + k_range * z_sorted > cumsum                    # :37
    k = np.count_nonzero(support, axis=1)                          # :38
    tau = (cumsum[np.arange(z.shape[0]), k - 1] - 1.0) / k         # :39
    out = np.maximum(z - tau[:, None], 0.0)                        # :40
    if return_tau:
        return (out[0] if squeeze else out), z, tau
    return out[0] if squeeze else out


def project_simplex_bruteforce(z: np.ndarray) -> np.ndarray:
    """Exhaustive-support simplex projection, sparsemax.py:60-84."""
    z = np.asarray(z, dtype=np.float64)
    n = z.size
    best = None
    best_dist = np.inf
    for mask_bits in range(1, 2 ** n):
        support = np.array([(mask_bits >> i) & 1 for i in range(n)], dtype=bool)
        k = support.sum()
        tau = (z[support].sum() - 1.0) / k
        cand = np.where(support, z - tau, 0.0)
        if np.any(cand < -1e-12):
            continue
        cand = np.maximum(cand, 0.0)
        dist = np.sum((cand - z) ** 2)
        if dist < best_dist - 1e-15:
            best_dist = dist
            best = cand
    return best


def _glu(u: np.ndarray) -> np.ndarray:
    """network.py:58-61 (linear half first, gate half second)."""
    h = u.shape[1] // 2
    sig = 1.0 / (1.0 + np.exp(-u[:, h:]))
    return u[:, :h] * sig


def _transform(p: dict, x: np.ndarray, step: int) -> np.ndarray:
    """network.py:124-141: shared1 -> shared2 -> step fc1 -> step fc2."""
    u1 = np.einsum("bf,fk->bk", x, p["shared1_W"]) + p["shared1_b"]
    g1 = _glu(u1)
    u2 = np.einsum("bh,hk->bk", g1, p["shared2_W"]) + p["shared2_b"]
    g2 = (_glu(u2) + g1) * RESIDUAL_SCALE
    u3 = np.einsum("bh,hk->bk", g2, p[f"step{step}_fc1_W"]) + p[f"step{step}_fc1_b"]
    g3 = (_glu(u3) + g2) * RESIDUAL_SCALE
    u4 = np.einsum("bh,hk->bk", g3, p[f"step{step}_fc2_W"]) + p[f"step{step}_fc2_b"]
    return (_glu(u4) + g3) * RESIDUAL_SCALE


def apply(params: dict, norm_mean: np.ndarray, norm_var: np.ndarray, *,
          n_d: int, n_steps: int, gamma: float, x: np.ndarray,
          normalized: bool = False, use_batch_stats: bool = False,
          diagnostics: bool = False) -> dict:
    """Restatement of ``TabNetModel.apply`` (network.py:195-267).

    Returns ``logits, probabilities, masks (S,B,F), importance``.  With
    ``diagnostics=True`` also the tie-margin data the parity comparator needs:
    ``z_shift (S,B,F)`` and ``tau (S,B)`` of every sparsemax call,
    ``d_pre_absmin (B,)`` = min over steps/units of |pre-ReLU decision|.
    """
    x = np.asarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[None, :]
    f = norm_mean.shape[0]
    if x.shape[1] != f:
        raise OracleInputError(f"batch width {x.shape[1]} != feature_count {f}")
    if not np.all(np.isfinite(x)):
        raise OracleInputError("features must be finite")
    if not normalized:
        if use_batch_stats:                                     # :213-216
            mean = x.mean(axis=0)
            var = x.var(axis=0)
            xn = (x - mean) / np.sqrt(var + NORM_EPS)
        else:                                                   # :118-120
            xn = (x - norm_mean) / np.sqrt(norm_var + NORM_EPS)
    else:
        xn = x
    p = params
    b = xn.shape[0]
    f0 = _transform(p, xn, 0)                                   # :226
    a = f0[:, n_d:]
    prior = np.ones((b, f))
    d_sum = np.zeros((b, n_d))
    agg = np.zeros((b, f))
    masks = np.empty((n_steps, b, f))
    zs = np.empty((n_steps, b, f)) if diagnostics else None
    taus = np.empty((n_steps, b)) if diagnostics else None
    d_absmin = np.full(b, np.inf)
    for s in range(1, n_steps + 1):                             # :232-251
        att = np.einsum("ba,af->bf", a, p[f"step{s}_att_W"]) + p[f"step{s}_att_b"]
        z = prior * att
        if diagnostics:
            m, z_shift, tau = sparsemax(z, return_tau=True)
            zs[s - 1] = z_shift
            taus[s - 1] = tau
        else:
            m = sparsemax(z)
        new_prior = prior * (gamma - m)
        xm = m * xn
        fs = _transform(p, xm, s)
        d_pre = fs[:, :n_d]
        if diagnostics:
            d_absmin = np.minimum(d_absmin, np.abs(d_pre).min(axis=1))
        d = np.maximum(d_pre, 0.0)
        d_sum = d_sum + d
        eta = d.sum(axis=1)
        agg = agg + eta[:, None] * m
        masks[s - 1] = m
        a = fs[:, n_d:]
        prior = new_prior
    logits = np.einsum("bd,dc->bc", d_sum, p["head_W"]) + p["head_b"]   # :253-256
    shifted = logits - logits.max(axis=1, keepdims=True)
    expv = np.exp(shifted)
    probs = expv / expv.sum(axis=1, keepdims=True)
    totals = agg.sum(axis=1, keepdims=True)                     # :258-261
    fallback = masks.mean(axis=0)
    importance = np.where(totals > 0.0, agg / np.where(totals > 0.0, totals, 1.0),
                          fallback)
    out = dict(logits=logits, probabilities=probs, masks=masks, importance=importance)
    if diagnostics:
        # the magnitude of the terms each logit sums (network.py:253): the
        # conditioning of d_sum @ head_W, for the comparator's logits bound
        logit_scale = np.abs(d_sum) @ np.abs(p["head_W"]) + np.abs(p["head_b"])
        out.update(z_shift=zs, tau=taus, d_pre_absmin=d_absmin,
                   agg_total=totals[:, 0], logit_scale=logit_scale)
    return out


def apply_model(model, x, **kw) -> dict:
    """Convenience: run the oracle on any object shaped like TabNetModel."""
    cfg = model.config
    return apply(model.params, np.asarray(model.norm_mean), np.asarray(model.norm_var),
                 n_d=cfg.n_d, n_steps=cfg.n_steps, gamma=cfg.gamma, x=x, **kw)
