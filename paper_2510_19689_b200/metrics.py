"""Evaluation helpers over the GPU model: ``accuracy`` and ``roc_auc``.

Mirrors the reference's ``tabserve/model/training.py:177-202`` (callers of
``apply``, SURVEY.md §8(b)'s "callers who must not notice"); training itself is
out of scope.  Both run ``model.apply`` on the device and return the reference's
numbers bit for bit:

* ``accuracy`` is the same argmax-of-probabilities mean (training.py:177-180).
* ``roc_auc`` computes the same rank statistic, ordinal ranks of a stable
  (mergesort) argsort of ``concat(pos, neg)`` with ties replaced by their
  midranks (training.py:183-202), but in O(n log n): one pass over the sorted
  scores finds the tie runs instead of the reference's per-unique-value scan
  (O(n * n_unique): seconds at 65,536 rows).  A tie run at sorted positions
  [i, j) has midrank (i + 1 + j) / 2, which is exactly the float64 mean the
  reference takes (integer sums below 2^53, an exact quotient), so the rank
  array and its sum are identical.
"""
from __future__ import annotations

import numpy as np

from .errors import TrainingError


def _as_matrix(x) -> np.ndarray:
    return np.asarray(getattr(x, "values", x), dtype=np.float64)


def accuracy(model, x, y) -> float:
    """Share of rows whose argmax probability equals ``y`` (training.py:177-180)."""
    res = model.apply(_as_matrix(x))
    pred = np.argmax(res.probabilities, axis=1)
    return float((pred == np.asarray(y)).mean())


def midranks(v: np.ndarray) -> np.ndarray:
    """1-based ranks of ``v`` with ties at their mean rank (training.py:191-199)."""
    v = np.asarray(v, dtype=np.float64)
    n = v.size
    order = np.argsort(v, kind="mergesort")
    sv = v[order]
    # tie runs in sorted order: run k covers sorted positions [start_k, end_k)
    brk = np.flatnonzero(sv[1:] != sv[:-1]) + 1
    start = np.concatenate(([0], brk))
    end = np.concatenate((brk, [n]))
    run_rank = (start + 1 + end).astype(np.float64) / 2.0
    ranks = np.empty(n, dtype=np.float64)
    ranks[order] = np.repeat(run_rank, end - start)
    return ranks


def roc_auc(model, x, y) -> float:
    """Binary AUC via the rank statistic, ties at midranks (training.py:183-202)."""
    res = model.apply(_as_matrix(x))
    scores = res.probabilities[:, 1]
    y = np.asarray(y)
    pos = scores[y == 1]
    neg = scores[y == 0]
    if pos.size == 0 or neg.size == 0:
        raise TrainingError("AUC needs both classes present")
    ranks = midranks(np.concatenate([pos, neg]))
    r_pos = ranks[:pos.size].sum()
    return float((r_pos - pos.size * (pos.size + 1) / 2) / (pos.size * neg.size))
