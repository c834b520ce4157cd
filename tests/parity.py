"""Tie-aware parity comparator shared by the GPU tests.

A row is EXEMPT when the float64 reference's own sparsemax margin at any step,
min_i |z_i - tau| / max|z|, is below ``delta`` (default 2e-5; every fp32 / 3xTF32
support flip measured on B200 had a margin below 2.7e-6) (the support set there is decided
by rounding, not by the model), or — for the class check only — when its top-2
probability gap is below ``gap``.  On every other row: identical sparsemax
support sets at every step, identical predicted class, and values within
``|gpu - ref| <= rtol*|ref| + atol`` elementwise for probabilities,
``|gpu - ref|_c <= rtol * max(max_c |ref|, scale_c) + atol`` for logits, where
``scale_c = sum_k |d_sum_k W_kc| + |b_c|`` is the magnitude of the terms the
logit sums (the oracle's ``logit_scale``; the goldens, which predate it, use
the row's inf-norm alone),
and normwise per row (per step for masks) for the simplex-valued masks and
importance, relative to the vector's total mass:
``max_f |gpu - ref| <= rtol * sum_f |ref| + atol`` (sum_f |ref| = 1 for these
probability vectors).  Elementwise relative error is meaningless for a mask
entry sitting just above the sparsemax threshold (m_i = z_i - tau is a
difference of O(max|z|) quantities).  Elementwise and max-normalised figures
are still reported (``max_err``).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class ParityReport:
    rows: int
    exempt_rows: list = field(default_factory=list)
    support_mismatch_rows: list = field(default_factory=list)
    class_mismatch_rows: list = field(default_factory=list)
    max_err: dict = field(default_factory=dict)
    viol: dict = field(default_factory=dict)

    @property
    def ok(self) -> bool:
        return not self.support_mismatch_rows and not self.class_mismatch_rows and \
            all(v == 0 for v in self.viol.values())

    def summary(self) -> str:
        return (f"rows={self.rows} exempt={len(self.exempt_rows)} "
                f"support_mismatch={self.support_mismatch_rows[:10]} "
                f"class_mismatch={self.class_mismatch_rows[:10]} "
                f"max_err={ {k: float(f'{v:.3g}') for k, v in self.max_err.items()} } viol={self.viol}")


def compare(ref: dict, got: dict, *, delta: float = 2e-5, gap: float = 1e-6,
            rtol: float = 1e-4, atol: dict | None = None) -> ParityReport:
    atol = {"logits": 1e-6, "probabilities": 1e-6, "masks": 1e-6, "importance": 1e-6,
            **(atol or {})}
    margin = ref["margin"]                   # (S, B)
    b = margin.shape[1]
    exempt = np.any(margin < delta, axis=0)
    rep = ParityReport(rows=b, exempt_rows=np.nonzero(exempt)[0].tolist())
    keep = ~exempt
    sup_ref = ref["masks"] > 0
    sup_got = np.asarray(got["masks"]) > 0
    sup_bad = np.any(sup_ref != sup_got, axis=(0, 2)) & keep
    rep.support_mismatch_rows = np.nonzero(sup_bad)[0].tolist()
    cls_ref = np.argmax(ref["probabilities"], axis=1)
    cls_got = np.argmax(np.asarray(got["probabilities"]), axis=1)
    cls_keep = keep & (ref["top2_gap"] >= gap)
    rep.class_mismatch_rows = np.nonzero((cls_ref != cls_got) & cls_keep)[0].tolist()
    for k in ("logits", "probabilities", "importance", "masks"):
        r = np.asarray(ref[k], dtype=np.float64)
        g = np.asarray(got[k], dtype=np.float64)
        if k == "masks":
            r, g = r[:, keep], g[:, keep]
        else:
            r, g = r[keep], g[keep]
        err = np.abs(g - r)
        rep.max_err[k] = float(err.max()) if err.size else 0.0
        rep.max_err[k + "_rel"] = float((err / np.maximum(np.abs(r), 1e-30)).max()) if err.size else 0.0
        if not err.size:
            rep.viol[k] = 0
        elif k == "logits":
            # logits are unbounded and may sit near 0: relative to the row's
            # inf-norm, or (when the reference provides it) to the magnitude of
            # the terms the logit sums, |d_sum| @ |head_W| + |head_b| (the
            # conditioning of network.py:253; a logit that cancels to ~1e-2 out of
            # terms ~1 carries the terms' rounding)
            r_row = np.abs(r).max(axis=-1, keepdims=True)
            scale = r_row
            if "logit_scale" in ref:
                scale = np.maximum(r_row, np.asarray(ref["logit_scale"], np.float64)[keep])
            rep.viol[k] = int(np.count_nonzero(np.any(err > rtol * scale + atol[k], axis=-1)))
        elif k in ("masks", "importance"):
            # reported only: elementwise relative error on the support entries
            # that carry at least 1% of the row's mass
            on = np.abs(r) >= 1e-2 * np.maximum(np.abs(r).sum(axis=-1, keepdims=True), 1e-300)
            rep.max_err[k + "_support_rel"] = float((err[on] / np.abs(r[on])).max()) if on.any() else 0.0
            e_row = err.max(axis=-1)
            r_row = np.abs(r).sum(axis=-1)
            rep.max_err[k + "_rownorm_rel"] = float((e_row / np.maximum(r_row, 1e-30)).max())
            rep.max_err[k + "_rowmax_rel"] = float((e_row / np.maximum(np.abs(r).max(axis=-1), 1e-30)).max())
            rep.viol[k] = int(np.count_nonzero(e_row > rtol * r_row + atol[k]))
        else:
            rep.viol[k] = int(np.count_nonzero(err > rtol * np.abs(r) + atol[k]))
    return rep
