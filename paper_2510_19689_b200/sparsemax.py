"""Sparsemax (simplex projection) — API of ``tabserve/model/sparsemax.py``.

``sparsemax`` runs on the GPU in float64 for any width (a warp-per-row
sort-free Michelot kernel, via ``tbn_sparsemax_host_f64``), the reference
helper's precision; validation and error types follow sparsemax.py:13-30.  ``project_simplex_bruteforce`` is the reference's
exhaustive-support oracle (sparsemax.py:60-84), kept for API parity; it is a
test oracle, never used by the engine.
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from .errors import InvalidInputError


def sparsemax(logits: np.ndarray) -> np.ndarray:
    z = np.asarray(logits, dtype=np.float64)
    if z.size == 0:
        raise InvalidInputError("sparsemax input must have length >= 1")
    if not np.all(np.isfinite(z)):
        raise InvalidInputError("sparsemax input must be finite")
    squeeze = z.ndim == 1
    if squeeze:
        z = z[None, :]
    if z.ndim != 2:
        raise InvalidInputError("sparsemax expects a vector or a 2-D batch")
    z = np.ascontiguousarray(z)
    out = np.empty_like(z)
    N.check(N.lib().tbn_sparsemax_host_f64(z.ctypes.data, z.shape[0], z.shape[1],
                                           out.ctypes.data), "tbn_sparsemax_host_f64")
    return out[0] if squeeze else out


def project_simplex_bruteforce(z: np.ndarray) -> np.ndarray:
    """Exact simplex projection by exhaustive support enumeration (oracle)."""
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
