"""TabNet predict + explain on B200 behind the reference's own API.

Mirrors ``tabserve/model/network.py`` (dataclasses :32-55, ``init_parameters``
:71-97, ``TabNetModel`` :100-343) so callers of the reference — the serving
worker (serving/service.py:144), stability (interpret/stability.py:108) and the
invariance check (interpret/invariance.py:34) — run unchanged.  ``apply`` is the
hot path and always runs on the GPU through libtabnet_b200.so: one fused
persistent kernel per call.  There is no CPU fallback; without a usable CUDA
device ``apply`` raises :class:`DeviceError`.

The model owns one immutable device replica of its packed weights per
(device, precision), built lazily on first use; ``params`` must not be mutated
after the first ``apply`` (use ``copy()``).
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .config import ModelConfig
from .errors import ConfigurationError, InvalidInputError, UnsupportedShapeError

_NORM_EPS = 1e-8
_RESIDUAL_SCALE = math.sqrt(0.5)
DEFAULT_PRECISION = "auto"
# "auto": the fused tcgen05 kernel in 3xTF32 (fp32-faithful) where an instance
# is compiled for the model shape, else the fp32 CUDA-core kernel.  Both are GPU
# kernels; neither is a CPU fallback.
AUTO_ORDER = ("tf32x3", "fp32")


class _Lease:
    """Buffer-protocol owner of one pooled allocation (PEP 688): numpy arrays
    made from it, and every view of those, keep it alive; when the last one is
    gone the memory goes back to the pool."""

    __slots__ = ("raw", "pool")

    def __init__(self, raw: np.ndarray, pool: "_OutputPool"):
        self.raw, self.pool = raw, pool

    def __buffer__(self, flags: int) -> memoryview:
        return memoryview(self.raw)

    def __release_buffer__(self, view: memoryview) -> None:
        view.release()

    def __del__(self):
        try:
            self.pool.give(self.raw)
        except Exception:           # interpreter shutdown
            pass


class _OutputPool:
    """Recycled float64 result buffers for ``apply``.

    A fresh numpy array is mapped on first touch: for HR @ 65,536 the 112 MB of
    float64 results cost ~3 ms of page faults (zero-filled by the kernel) per
    call, more than the GPU forward and the PCIe copies together.  Results are
    handed out as arrays over a leased buffer (``_Lease``) that returns to the
    pool only when the result and every view of it are garbage, so a result is
    never overwritten while reachable.  At most ``keep`` free buffers per size
    and ``max_free`` bytes in all are kept.
    """

    def __init__(self, keep: int = 2, max_free: int = 1 << 30, min_bytes: int = 1 << 20):
        self.keep, self.max_free, self.min_bytes = keep, max_free, min_bytes
        self._free: dict[int, list[np.ndarray]] = {}
        self._free_bytes = 0
        self._lock = threading.Lock()

    def take(self, shape: tuple, dtype=np.float64) -> np.ndarray:
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        if n < self.min_bytes:
            return np.empty(shape, dtype)
        raw = None
        with self._lock:
            lst = self._free.get(n)
            if lst:
                raw = lst.pop()
                self._free_bytes -= n
        if raw is None:
            raw = np.empty(n, np.uint8)
        return np.frombuffer(_Lease(raw, self), dtype=dtype).reshape(shape)

    def give(self, raw: np.ndarray) -> None:
        n = raw.nbytes
        with self._lock:
            lst = self._free.setdefault(n, [])
            if len(lst) < self.keep and self._free_bytes + n <= self.max_free:
                lst.append(raw)
                self._free_bytes += n


_RESULTS = _OutputPool()


@dataclass
class Explanation:
    """Per-step feature masks and their aggregate for one sample (network.py:32-37)."""

    step_masks: np.ndarray
    aggregate_importance: np.ndarray


@dataclass
class PredictionOutput:
    probabilities: np.ndarray
    predicted_class: int
    explanation: Explanation


@dataclass
class ForwardResult:
    """Batched forward outputs (network.py:47-55)."""

    logits: np.ndarray            # (B, C)
    probabilities: np.ndarray     # (B, C)
    masks: np.ndarray             # (n_steps, B, F)
    importance: np.ndarray        # (B, F)
    caches: dict = field(default_factory=dict)


def init_parameters(config: ModelConfig) -> dict[str, np.ndarray]:
    """Seeded uniform fan-in initialization, same draws as network.py:71-97."""
    rng = np.random.default_rng(config.seed)
    h = config.n_d + config.n_a
    f = config.feature_count

    def uniform(fan_in: int, shape: tuple[int, ...]) -> np.ndarray:
        bound = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-bound, bound, size=shape)

    params: dict[str, np.ndarray] = {
        "shared1_W": uniform(f, (f, 2 * h)),
        "shared1_b": np.zeros(2 * h),
        "shared2_W": uniform(h, (h, 2 * h)),
        "shared2_b": np.zeros(2 * h),
        "head_W": uniform(config.n_d, (config.n_d, config.n_classes)),
        "head_b": np.zeros(config.n_classes),
    }
    for s in range(config.n_steps + 1):
        params[f"step{s}_fc1_W"] = uniform(h, (h, 2 * h))
        params[f"step{s}_fc1_b"] = np.zeros(2 * h)
        params[f"step{s}_fc2_W"] = uniform(h, (h, 2 * h))
        params[f"step{s}_fc2_b"] = np.zeros(2 * h)
    for s in range(1, config.n_steps + 1):
        params[f"step{s}_att_W"] = uniform(config.n_a, (config.n_a, f))
        params[f"step{s}_att_b"] = np.zeros(f)
    return params


class DeviceModel:
    """Owner of one ``tbn_model*`` (packed weights resident on one GPU)."""

    def __init__(self, config: ModelConfig, params: dict, norm_mean: np.ndarray,
                 norm_var: np.ndarray, precision: str, device: int, *, regression: bool = False):
        L = N.lib()
        if precision not in N.PRECISIONS:
            raise ConfigurationError(f"unknown precision {precision!r}; one of {sorted(N.PRECISIONS)}")
        self.n_out = 1 if regression else config.n_classes
        cfg = N.TbnConfig(config.feature_count, self.n_out, config.n_d, config.n_a,
                          config.n_steps, N.CFG_REGRESSION if regression else 0, float(config.gamma))
        keys = sorted(params)
        arrays = [np.ascontiguousarray(params[k], dtype=np.float64) for k in keys]
        names = (C.c_char_p * len(keys))(*[k.encode() for k in keys])
        vals = (C.c_void_p * len(keys))(*[a.ctypes.data for a in arrays])
        sizes = (C.c_int64 * len(keys))(*[a.size for a in arrays])
        mean = np.ascontiguousarray(norm_mean, dtype=np.float64)
        var = np.ascontiguousarray(norm_var, dtype=np.float64)
        if mean.shape != (config.feature_count,) or var.shape != (config.feature_count,):
            raise ConfigurationError("normalization stats must have shape (feature_count,)")
        handle = C.c_void_p()
        N.check(L.tbn_model_create(C.byref(cfg), names, vals, sizes, len(keys),
                                   mean.ctypes.data, var.ctypes.data,
                                   N.PRECISIONS[precision], int(device), C.byref(handle)),
                "tbn_model_create")
        self.handle = handle
        self.config = config
        self.precision = precision
        self.device = device
        self._lib = L

    @classmethod
    def from_tbnt(cls, stream: bytes, precision: str, device: int, *, regression: bool = False,
                  head_column: int = 0) -> "DeviceModel":
        """The cold-start path: a .tbnt stream (reference io.py:43-57) parsed,
        CRC-checked, packed and uploaded by one native call."""
        L = N.lib()
        if precision not in N.PRECISIONS:
            raise ConfigurationError(f"unknown precision {precision!r}; one of {sorted(N.PRECISIONS)}")
        handle = C.c_void_p()
        N.check(L.tbn_model_create_from_tbnt(stream, len(stream), N.PRECISIONS[precision], int(device),
                                             N.CFG_REGRESSION if regression else 0, int(head_column),
                                             C.byref(handle)), "tbn_model_create_from_tbnt")
        self = cls.__new__(cls)
        cfg = N.TbnConfig()
        prec, dev = C.c_int32(), C.c_int32()
        N.check(L.tbn_model_info(handle, C.byref(cfg), C.byref(prec), C.byref(dev)))
        self.handle = handle
        self.n_out = cfg.n_classes
        self.config = ModelConfig(feature_count=cfg.feature_count, n_classes=max(2, cfg.n_classes),
                                  n_d=cfg.n_d, n_a=cfg.n_a, n_steps=cfg.n_steps, gamma=cfg.gamma)
        self.precision = precision
        self.device = device
        self._lib = L
        return self

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.tbn_model_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- host-buffer path (reference-facing) ----------------------------------
    def forward_host_f64(self, x: np.ndarray, flags: int, want_masks: bool = True) -> dict:
        cfg = self.config
        b, f, c, s = x.shape[0], cfg.feature_count, self.n_out, cfg.n_steps
        take = _RESULTS.take
        out = dict(logits=take((b, c)), probabilities=take((b, c)),
                   masks=take((s, b, f)) if want_masks else None,
                   importance=take((b, f)),
                   predicted_class=np.empty(b, dtype=np.int32))
        o = N.TbnOutputs(*(N.ptr(out[k]) for k in
                           ("logits", "probabilities", "masks", "importance", "predicted_class")))
        N.check(self._lib.tbn_forward_host_f64(self.handle, x.ctypes.data, b, flags, C.byref(o)),
                "tbn_forward_host_f64")
        return out

    def forward_host_f32(self, x: np.ndarray, flags: int, out: dict) -> None:
        o = N.TbnOutputs(*(N.ptr(out.get(k)) for k in
                           ("logits", "probabilities", "masks", "importance", "predicted_class")))
        N.check(self._lib.tbn_forward_host(self.handle, x.ctypes.data, x.shape[0], flags,
                                           C.byref(o)), "tbn_forward_host")

    # -- device path (torch tensors as plumbing; zero-copy) ---------------------
    def workspace_bytes(self, rows: int, flags: int = 0) -> int:
        return int(self._lib.tbn_workspace_bytes(self.handle, rows, flags))

    def forward_device(self, x_ptr: int, rows: int, flags: int, out_ptrs: dict,
                       err_ptr: int | None, ws_ptr: int, ws_bytes: int, stream_ptr: int) -> None:
        o = N.TbnOutputs(*(out_ptrs.get(k) for k in
                           ("logits", "probabilities", "masks", "importance", "predicted_class")))
        N.check(self._lib.tbn_forward(self.handle, x_ptr, rows, flags, C.byref(o), err_ptr,
                                      ws_ptr, ws_bytes, stream_ptr), "tbn_forward")


@dataclass
class TabNetModel:
    """Trained model bundle (network.py:100-114) whose ``apply`` runs on a B200."""

    config: ModelConfig
    params: dict[str, np.ndarray]
    norm_mean: np.ndarray
    norm_var: np.ndarray
    model_version: str
    precision: str = DEFAULT_PRECISION
    device: int | None = None

    def __post_init__(self) -> None:
        if not self.model_version:
            raise ConfigurationError("model_version must be non-empty")
        if np.any(np.asarray(self.norm_var) <= 0):
            raise ConfigurationError("normalization variances must be > 0")
        if self.precision not in N.PRECISIONS and self.precision != "auto":
            raise ConfigurationError(f"unknown precision {self.precision!r}")
        self._engines: dict = {}
        self._engine_lock = threading.Lock()

    # -- construction helpers ---------------------------------------------------
    @classmethod
    def from_reference(cls, model, *, precision: str = DEFAULT_PRECISION,
                       device: int | None = None) -> "TabNetModel":
        """Wrap any object shaped like the reference's TabNetModel (duck-typed:
        ``config, params, norm_mean, norm_var, model_version``)."""
        rc = model.config
        cfg = ModelConfig(feature_count=rc.feature_count, n_classes=rc.n_classes, n_d=rc.n_d,
                          n_a=rc.n_a, n_steps=rc.n_steps, lambda_sparse=rc.lambda_sparse,
                          gamma=rc.gamma, seed=rc.seed)
        return cls(config=cfg, params={k: np.asarray(v, dtype=np.float64) for k, v in model.params.items()},
                   norm_mean=np.asarray(model.norm_mean, dtype=np.float64),
                   norm_var=np.asarray(model.norm_var, dtype=np.float64),
                   model_version=model.model_version, precision=precision, device=device)

    def engine(self, device: int | None = None, precision: str | None = None) -> DeviceModel:
        dev = N.env_device() if device is None and self.device is None else \
            (self.device if device is None else device)
        prec = precision or self.precision
        key = (dev, prec)
        eng = self._engines.get(key)
        if eng is None:
            with self._engine_lock:
                eng = self._engines.get(key)
                if eng is None:
                    if prec == "auto":
                        last = None
                        for cand in AUTO_ORDER:
                            try:
                                eng = self._make_engine(cand, dev)
                                break
                            except UnsupportedShapeError as e:
                                last = e
                        if eng is None:
                            raise UnsupportedShapeError(
                                f"no kernel instance serves this model shape in any of {AUTO_ORDER}: {last}")
                    else:
                        eng = self._make_engine(prec, dev)
                    self._engines[key] = eng
        return eng

    def _make_engine(self, precision: str, device: int) -> DeviceModel:
        return DeviceModel(self.config, self.params, self.norm_mean, self.norm_var, precision, device)

    # -- normalization (network.py:118-120; host helper, not the hot path) -------
    def normalize(self, x: np.ndarray) -> np.ndarray:
        return (x - self.norm_mean) / np.sqrt(self.norm_var + _NORM_EPS)

    def attentive_step(self, state: np.ndarray, prior: np.ndarray,
                       step_index: int) -> tuple[np.ndarray, np.ndarray]:
        """network.py:170-191: mask = sparsemax(prior * scores(state)) (sparsemax on GPU)."""
        from .sparsemax import sparsemax
        cfg = self.config
        state = np.atleast_2d(np.asarray(state, dtype=np.float64))
        prior = np.atleast_2d(np.asarray(prior, dtype=np.float64))
        if not 1 <= step_index <= cfg.n_steps:
            raise ConfigurationError(f"step_index {step_index} outside 1..{cfg.n_steps}")
        if state.shape[1] != cfg.n_a:
            raise ConfigurationError(f"attention state width {state.shape[1]} != n_a {cfg.n_a}")
        if prior.shape[1] != cfg.feature_count:
            raise ConfigurationError(
                f"prior width {prior.shape[1]} != feature_count {cfg.feature_count}")
        att = (np.einsum("ba,af->bf", state, self.params[f"step{step_index}_att_W"])
               + self.params[f"step{step_index}_att_b"])
        mask = sparsemax(prior * att)
        new_prior = prior * (cfg.gamma - mask)
        return mask, new_prior

    # -- full forward (network.py:195-267) ----------------------------------------
    def apply(self, x: np.ndarray, *, normalized: bool = False,
              use_batch_stats: bool = False, with_caches: bool = False) -> ForwardResult:
        """Run the batch through all decision steps on the GPU.

        Same validation order and exception types as the reference (width
        mismatch and non-finite features raise InvalidInputError).  Values are
        computed in fp32 with 3xTF32 tensor-core contractions (default) and
        returned as float64 arrays.  ``with_caches`` (training only) is not
        supported by the inference engine.
        """
        if with_caches:
            raise ConfigurationError("with_caches is training-only; the B200 engine is inference-only")
        cfg = self.config
        x = np.asarray(x, dtype=np.float64)
        if x.ndim == 1:
            x = x[None, :]
        if x.ndim != 2 or x.shape[1] != cfg.feature_count:
            raise InvalidInputError(
                f"batch width {x.shape[-1] if x.ndim else 0} != feature_count {cfg.feature_count}")
        b = x.shape[0]
        if b == 0:
            n_out = getattr(self, "n_outputs", cfg.n_classes)
            return ForwardResult(logits=np.empty((0, n_out)),
                                 probabilities=np.empty((0, n_out)),
                                 masks=np.empty((cfg.n_steps, 0, cfg.feature_count)),
                                 importance=np.empty((0, cfg.feature_count)))
        flags = (N.FLAG_NORMALIZED if normalized else 0) | \
                (N.FLAG_BATCH_STATS if (use_batch_stats and not normalized) else 0)
        out = self.engine().forward_host_f64(np.ascontiguousarray(x), flags)
        return ForwardResult(logits=out["logits"], probabilities=out["probabilities"],
                             masks=out["masks"], importance=out["importance"], caches={})

    def forward(self, batch) -> list[PredictionOutput]:
        """Per-sample prediction outputs (network.py:269-281)."""
        values = getattr(batch, "values", batch)
        result = self.apply(values)
        outputs = []
        for i in range(result.probabilities.shape[0]):
            expl = Explanation(step_masks=result.masks[:, i, :].copy(),
                               aggregate_importance=result.importance[i].copy())
            probs = result.probabilities[i]
            outputs.append(PredictionOutput(probabilities=probs,
                                            predicted_class=int(np.argmax(probs)),
                                            explanation=expl))
        return outputs

    def copy(self) -> "TabNetModel":
        return TabNetModel(config=self.config,
                           params={k: v.copy() for k, v in self.params.items()},
                           norm_mean=self.norm_mean.copy(), norm_var=self.norm_var.copy(),
                           model_version=self.model_version, precision=self.precision,
                           device=self.device)


GpuTabNetModel = TabNetModel


@dataclass
class TabNetRegressor(TabNetModel):
    """Regression head on the same encoder (an extension).

    The reference supports only the softmax classifier (config.py:32-33 enforces
    ``n_classes >= 2``).  BASELINE's BLS workload is a regression, so the engine
    offers an identity head: ``logits = d_sum @ head_W[:, c] + head_b[c]`` for one
    column ``c`` of a reference model's head (``TBN_CFG_REGRESSION`` in the C ABI).
    ``apply`` returns logits of shape (B, 1) and the same values as
    ``probabilities``; masks and importance are the classifier's.  Its oracle is
    column ``c`` of the reference's logits (network.py:253).
    """

    head_column: int = 0
    n_outputs: int = 1

    @classmethod
    def from_reference(cls, model, *, head_column: int = 0, precision: str = DEFAULT_PRECISION,
                       device: int | None = None) -> "TabNetRegressor":
        base = TabNetModel.from_reference(model, precision=precision, device=device)
        if not 0 <= head_column < base.config.n_classes:
            raise ConfigurationError(f"head_column {head_column} outside the head's "
                                     f"{base.config.n_classes} columns")
        return cls(config=base.config, params=base.params, norm_mean=base.norm_mean,
                   norm_var=base.norm_var, model_version=base.model_version,
                   precision=precision, device=device, head_column=head_column)

    def _make_engine(self, precision: str, device: int) -> DeviceModel:
        c = self.head_column
        params = dict(self.params)
        params["head_W"] = np.ascontiguousarray(np.asarray(self.params["head_W"])[:, c:c + 1])
        params["head_b"] = np.ascontiguousarray(np.asarray(self.params["head_b"])[c:c + 1])
        return DeviceModel(self.config, params, self.norm_mean, self.norm_var, precision, device,
                           regression=True)

    def forward(self, batch) -> list[PredictionOutput]:
        values = getattr(batch, "values", batch)
        result = self.apply(values)
        return [PredictionOutput(probabilities=result.logits[i], predicted_class=0,
                                 explanation=Explanation(step_masks=result.masks[:, i, :].copy(),
                                                         aggregate_importance=result.importance[i].copy()))
                for i in range(result.logits.shape[0])]

    def copy(self) -> "TabNetRegressor":
        return TabNetRegressor(config=self.config,
                               params={k: v.copy() for k, v in self.params.items()},
                               norm_mean=self.norm_mean.copy(), norm_var=self.norm_var.copy(),
                               model_version=self.model_version, precision=self.precision,
                               device=self.device, head_column=self.head_column)
