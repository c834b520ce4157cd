"""ctypes binding of libtabnet_b200.so (include/tabnet_b200.h).

Loading never needs a GPU; compute entry points fail with DeviceError when no
CUDA device is usable (there is no CPU fallback anywhere in the product path).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import (ChecksumError, ConfigurationError, DeviceError, FormatVersionError,
                     InvalidInputError, ModelFormatError, TabserveError, TruncatedStreamError,
                     UnsupportedShapeError)

LIB_PATH = Path(__file__).resolve().parent / "libtabnet_b200.so"

(TBN_OK, TBN_ERR_INVALID_INPUT, TBN_ERR_CONFIG, TBN_ERR_CUDA, TBN_ERR_UNSUPPORTED, TBN_ERR_FORMAT,
 TBN_ERR_FORMAT_VERSION, TBN_ERR_TRUNCATED, TBN_ERR_CHECKSUM) = range(9)
ABI_VERSION = 2
PREC_TF32X3, PREC_TF32, PREC_BF16, PREC_FP32 = range(4)
CFG_REGRESSION = 1           # tbn_config.flags: identity head, n_classes == 1
PRECISIONS = {"tf32x3": PREC_TF32X3, "tf32": PREC_TF32, "bf16": PREC_BF16, "fp32": PREC_FP32}
FLAG_NORMALIZED = 1
FLAG_BATCH_STATS = 2
FLAG_PACKED = 4          # launch geometry only (TBN_FLAG_PACKED)

# Every symbol include/tabnet_b200.h declares (tests check the .so exports them).
EXPORTED = (
    "tbn_abi_version", "tbn_last_error", "tbn_device_count", "tbn_device_init", "tbn_model_create",
    "tbn_model_destroy", "tbn_model_info", "tbn_workspace_bytes", "tbn_forward",
    "tbn_forward_host", "tbn_forward_host_f64", "tbn_sparsemax",
    "tbn_sparsemax_host_f64", "tbn_partition_mean", "tbn_crc32c",
    "tbn_tbnt_parse", "tbn_tbnt_free", "tbn_tbnt_info", "tbn_tbnt_param", "tbn_tbnt_norm",
    "tbn_model_create_from_tbnt", "tbn_prep_create", "tbn_prep_destroy", "tbn_prep_width",
    "tbn_preprocess",
)


class TbnConfig(C.Structure):
    _fields_ = [("feature_count", C.c_int32), ("n_classes", C.c_int32), ("n_d", C.c_int32),
                ("n_a", C.c_int32), ("n_steps", C.c_int32), ("flags", C.c_int32),
                ("gamma", C.c_double)]


class TbnPrepColumn(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("median", C.c_double), ("mean", C.c_double),
                ("std", C.c_double)]


class TbnOutputs(C.Structure):
    _fields_ = [("logits", C.c_void_p), ("probabilities", C.c_void_p), ("masks", C.c_void_p),
                ("importance", C.c_void_p), ("predicted_class", C.c_void_p)]


TbnOutputsF64 = TbnOutputs   # same layout (pointers)

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load (once) and return the engine library; raises DeviceError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH.name} is not built (run __graft_entry__.build() or "
                              f"python -m paper_2510_19689_b200.build); no CPU fallback exists")
        L = C.CDLL(str(LIB_PATH))
        vp, i32, i64, u32, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_size_t
        L.tbn_abi_version.restype = i32
        L.tbn_last_error.restype = C.c_char_p
        L.tbn_device_count.restype = i32
        L.tbn_device_init.restype = i32
        L.tbn_device_init.argtypes = [i32]
        L.tbn_model_create.restype = i32
        L.tbn_model_create.argtypes = [C.POINTER(TbnConfig), C.POINTER(C.c_char_p),
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_int64), i32,
                                       vp, vp, i32, i32, C.POINTER(vp)]
        L.tbn_model_destroy.restype = None
        L.tbn_model_destroy.argtypes = [vp]
        L.tbn_model_info.restype = i32
        L.tbn_model_info.argtypes = [vp, C.POINTER(TbnConfig), C.POINTER(i32), C.POINTER(i32)]
        L.tbn_workspace_bytes.restype = sz
        L.tbn_workspace_bytes.argtypes = [vp, i64, u32]
        L.tbn_forward.restype = i32
        L.tbn_forward.argtypes = [vp, vp, i64, u32, C.POINTER(TbnOutputs), vp, vp, sz, vp]
        L.tbn_forward_host.restype = i32
        L.tbn_forward_host.argtypes = [vp, vp, i64, u32, C.POINTER(TbnOutputs)]
        L.tbn_forward_host_f64.restype = i32
        L.tbn_forward_host_f64.argtypes = [vp, vp, i64, u32, C.POINTER(TbnOutputs)]
        L.tbn_sparsemax.restype = i32
        L.tbn_sparsemax.argtypes = [vp, i64, i32, vp, vp]
        L.tbn_partition_mean.restype = i32
        L.tbn_partition_mean.argtypes = [vp, i64, i32, i32, vp, vp]
        L.tbn_sparsemax_host_f64.restype = i32
        L.tbn_sparsemax_host_f64.argtypes = [vp, i64, i32, vp]
        L.tbn_crc32c.restype = u32
        L.tbn_crc32c.argtypes = [C.c_char_p, sz, u32]
        L.tbn_tbnt_parse.restype = i32
        L.tbn_tbnt_parse.argtypes = [C.c_char_p, sz, C.POINTER(vp)]
        L.tbn_tbnt_free.restype = None
        L.tbn_tbnt_free.argtypes = [vp]
        L.tbn_tbnt_info.restype = i32
        L.tbn_tbnt_info.argtypes = [vp, C.POINTER(TbnConfig), C.POINTER(C.c_double), C.POINTER(i64),
                                    C.POINTER(C.c_char_p), C.POINTER(i32)]
        L.tbn_tbnt_param.restype = i32
        L.tbn_tbnt_param.argtypes = [vp, i32, C.POINTER(C.c_char_p), C.POINTER(i32), C.POINTER(i64),
                                     C.POINTER(C.POINTER(C.c_double))]
        L.tbn_tbnt_norm.restype = i32
        L.tbn_tbnt_norm.argtypes = [vp, C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.POINTER(C.c_double))]
        L.tbn_model_create_from_tbnt.restype = i32
        L.tbn_model_create_from_tbnt.argtypes = [C.c_char_p, sz, i32, i32, i32, i32, C.POINTER(vp)]
        L.tbn_prep_create.restype = i32
        L.tbn_prep_create.argtypes = [C.POINTER(TbnPrepColumn), i32, i32, C.POINTER(vp)]
        L.tbn_prep_destroy.restype = None
        L.tbn_prep_destroy.argtypes = [vp]
        L.tbn_prep_width.restype = i32
        L.tbn_prep_width.argtypes = [vp]
        L.tbn_preprocess.restype = i32
        L.tbn_preprocess.argtypes = [vp, vp, i64, vp, vp]
        if L.tbn_abi_version() != ABI_VERSION:
            raise DeviceError("libtabnet_b200.so ABI version mismatch")
        _lib = L
        return _lib


def last_error() -> str:
    return lib().tbn_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map tbn_status onto the reference's exception classes (errors.py:8-13)."""
    if status == TBN_OK:
        return
    msg = last_error() or what
    if status == TBN_ERR_INVALID_INPUT:
        raise InvalidInputError(msg)
    if status == TBN_ERR_CONFIG:
        raise ConfigurationError(msg)
    if status == TBN_ERR_UNSUPPORTED:
        raise UnsupportedShapeError(msg)
    if status == TBN_ERR_CUDA:
        raise DeviceError(msg)
    if status == TBN_ERR_FORMAT:
        raise ModelFormatError(msg)
    if status == TBN_ERR_FORMAT_VERSION:
        raise FormatVersionError(msg)
    if status == TBN_ERR_TRUNCATED:
        raise TruncatedStreamError(msg)
    if status == TBN_ERR_CHECKSUM:
        raise ChecksumError(msg)
    raise TabserveError(f"status {status}: {msg}")


def device_count() -> int:
    return int(lib().tbn_device_count())


def crc32c(data: bytes, crc: int = 0) -> int:
    return int(lib().tbn_crc32c(data, len(data), crc))


def ptr(a: np.ndarray | None) -> int | None:
    """Data pointer of an array.  ``ctypes.c_char.from_buffer`` is ~5x cheaper
    than ``a.ctypes.data`` (which builds a ctypes helper object per call) and
    matters on the latency path; read-only, empty or non-contiguous arrays take
    the general route."""
    if a is None:
        return None
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data


def env_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0")) if "TBN_DEVICE" not in os.environ \
        else int(os.environ["TBN_DEVICE"])
