"""Device preprocessing: the reference's
``PreprocessPlan.transform`` (data/preprocess.py:68-122) with its numeric tail
on the GPU, feeding the fused forward without a host float64 matrix.

Split of the work:
* host (``encode``): the per-cell lookups only Python objects allow — a raw
  cell (float, level string or None) becomes one float64 code per column:
  the value or NaN (missing) for standardize / passthrough, the mapped level or
  -1 for ordinal, the category index or -1 for one-hot (an absent level, incl.
  a missing cell whose plan has no "missing" category).  Unseen counts are
  tallied exactly as the reference does.
* device (``tbn_preprocess``, csrc/kernel_prep.cu): median imputation,
  ``(v - mean) / std`` in float64 rounded once, ordinal values, one-hot
  expansion, written as the forward's float32 input.

``apply_table`` runs codes -> preprocessing kernel -> fused forward on one
stream; the per-row results equal ``model.apply(reference_matrix)`` bit for
bit, because the device matrix equals the reference's float64 matrix rounded
to float32 (the engine's input precision) element for element.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .errors import ConfigurationError, InvalidInputError

_KINDS = {"standardize": 0, "passthrough": 1, "ordinal": 2, "onehot": 3}


def _transforms(plan):
    """ColumnTransform-like records from a reference PreprocessPlan or its to_dict()."""
    ts = plan["transforms"] if isinstance(plan, dict) else plan.transforms
    out = []
    for t in ts:
        g = (lambda k, d=None, t=t: t.get(k, d)) if isinstance(t, dict) else \
            (lambda k, d=None, t=t: getattr(t, k, d))
        out.append(dict(label=g("label"), kind=g("kind"), median=float(g("median", 0.0)),
                        mean=float(g("mean", 0.0)), std=float(g("std", 1.0)),
                        categories=tuple(g("categories", ()) or ()),
                        mapping=tuple((str(k), int(v)) for k, v in (g("mapping", ()) or ()))))
    return out


class PlanCodes:
    """The host half of a fitted plan: column descriptors and the cell -> code
    lookups (no GPU needed)."""

    def __init__(self, plan):
        self.transforms = _transforms(plan)
        if not self.transforms:
            raise ConfigurationError("preprocessing plan has no feature columns")
        names = []
        for t in self.transforms:
            if t["kind"] not in _KINDS:
                raise ConfigurationError(f"unknown transform kind {t['kind']!r}")
            if t["kind"] == "onehot":
                names.extend(f"{t['label']}={cat}" for cat in t["categories"])
            else:
                names.append(t["label"])
        self.column_names = names
        self.width = len(names)
        self._maps = [dict(t["mapping"]) if t["kind"] == "ordinal" else
                      {cat: j for j, cat in enumerate(t["categories"])} if t["kind"] == "onehot" else None
                      for t in self.transforms]

    def descriptors(self):
        cols = (N.TbnPrepColumn * len(self.transforms))()
        for c, t in zip(cols, self.transforms):
            c.kind = _KINDS[t["kind"]]
            c.width = len(t["categories"]) if t["kind"] == "onehot" else 1
            c.median, c.mean, c.std = t["median"], t["mean"], t["std"]
        return cols

    def encode(self, columns: dict, n_rows: int | None = None) -> tuple[np.ndarray, dict]:
        """Raw table columns (``RawTable.columns``: label -> list of cells) ->
        (codes (rows, ncols) float64, unseen counts) — preprocess.py:74-111's
        lookups, nothing else."""
        n = n_rows if n_rows is not None else len(columns[self.transforms[0]["label"]])
        if n == 0:
            raise InvalidInputError("no rows to transform after quarantine")
        codes = np.empty((n, len(self.transforms)), dtype=np.float64)
        unseen: dict[str, int] = {}
        for c, (t, mp) in enumerate(zip(self.transforms, self._maps)):
            raw = columns[t["label"]]
            if t["kind"] in ("standardize", "passthrough"):
                col = np.array([math.nan if v is None else float(v) for v in raw], dtype=np.float64)
                if not np.all(np.isfinite(col[~np.isnan(col)])) or \
                        np.any(np.isnan(col) != np.array([v is None for v in raw])):
                    # a present non-finite value: the reference's FeatureMatrix rejects it
                    raise InvalidInputError("feature matrix must be finite")
                codes[:, c] = col
            elif t["kind"] == "ordinal":
                col = np.array([mp.get(v, -1) if v is not None else -1 for v in raw], dtype=np.float64)
                misses = int(np.count_nonzero(col < 0))
                if misses:
                    unseen[t["label"]] = misses
                codes[:, c] = col
            else:
                col = np.array([mp.get("missing" if v is None else v, -1) for v in raw], dtype=np.float64)
                misses = int(np.count_nonzero(col < 0))
                if misses:
                    unseen[t["label"]] = misses
                codes[:, c] = col
        return codes, unseen


class DevicePreprocessor(PlanCodes):
    """A fitted plan resident on one GPU (``tbn_prep``)."""

    def __init__(self, plan, device: int | None = None):
        super().__init__(plan)
        self.device = N.env_device() if device is None else device
        self._lib = N.lib()
        h = C.c_void_p()
        N.check(self._lib.tbn_prep_create(self.descriptors(), len(self.transforms), self.device, C.byref(h)),
                "tbn_prep_create")
        self.handle = h
        assert int(self._lib.tbn_prep_width(h)) == self.width

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.tbn_prep_destroy(h)
            except Exception:
                pass

    def transform_device(self, codes, out=None, stream=None):
        """Device codes (torch float64 (rows, ncols), CUDA) -> torch float32
        (rows, width) on the same device (async on ``stream``)."""
        import torch
        assert codes.is_cuda and codes.dtype == torch.float64 and codes.is_contiguous()
        rows = codes.shape[0]
        if out is None:
            out = torch.empty((rows, self.width), dtype=torch.float32, device=codes.device)
        st = (stream or torch.cuda.current_stream(codes.device)).cuda_stream
        N.check(self._lib.tbn_preprocess(self.handle, codes.data_ptr(), rows, out.data_ptr(), st), "tbn_preprocess")
        return out

    def transform(self, columns: dict, n_rows: int | None = None) -> tuple[np.ndarray, dict]:
        """(float32 matrix (rows, width) computed on the device, unseen counts)."""
        import torch
        codes, unseen = self.encode(columns, n_rows)
        d = torch.from_numpy(codes).to(torch.device("cuda", self.device))
        out = self.transform_device(d)
        return out.cpu().numpy(), unseen


def apply_table(model, prep: DevicePreprocessor, columns: dict, n_rows: int | None = None):
    """Raw table -> ForwardResult through the device: host lookups, one H2D of
    the codes, preprocessing kernel, fused forward, D2H of the outputs."""
    import torch
    from .device import DeviceRunner
    from .network import ForwardResult
    if prep.width != model.config.feature_count:
        raise InvalidInputError(f"plan width {prep.width} != feature_count {model.config.feature_count}")
    codes, _ = prep.encode(columns, n_rows)
    dev = torch.device("cuda", prep.device)
    rows = codes.shape[0]
    runner = DeviceRunner(model, rows, device=prep.device)
    stream = torch.cuda.current_stream(dev)
    x = prep.transform_device(torch.from_numpy(codes).to(dev, non_blocking=False), stream=stream)
    out = runner.run(x, stream=stream)
    torch.cuda.synchronize(dev)
    runner.check_finite()
    o = {k: v.cpu().numpy() for k, v in out.items()}
    return ForwardResult(logits=o["logits"].astype(np.float64), probabilities=o["probabilities"].astype(np.float64),
                         masks=o["masks"].astype(np.float64), importance=o["importance"].astype(np.float64))
