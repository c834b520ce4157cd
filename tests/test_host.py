"""Host-side logic: config/model validation, .tbnt I/O, CRC-32C, the C-ABI
library's exports, workload counts.  No GPU compute."""
import ctypes
import json
import re
import struct
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import _native as N
from paper_2510_19689_b200 import workloads as W


def _crc_py(data: bytes) -> int:
    # restatement of the reference's table loop (io.py:24-36)
    tab = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (c >> 1) ^ 0x82F63B78 if c & 1 else c >> 1
        tab.append(c)
    crc = 0xFFFFFFFF
    for b in data:
        crc = (crc >> 8) ^ tab[(crc ^ b) & 0xFF]
    return crc ^ 0xFFFFFFFF


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "tabnet_b200.h").read_text()
    declared = set(re.findall(r"\b(tbn_[a-z0-9_]+)\s*\(", header))
    assert declared == set(N.EXPORTED)
    lib = ctypes.CDLL(str(N.LIB_PATH))
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert N.lib().tbn_abi_version() == N.ABI_VERSION == 2


def test_crc32c_native_matches_reference_table():
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 9, 63, 1000):
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert P.io.crc32c(data) == _crc_py(data)
    assert P.io.crc32c(b"123456789") == 0xE3069283


def test_tbnt_roundtrip_bytes_identical_to_reference_stream():
    b = (GOLDEN / "adult.tbnt").read_bytes()
    m = P.load_model(b)
    assert m.model_version == "adult-tbnt-v1"
    assert P.save_model(m) == b


def test_tbnt_errors():
    b = bytearray((GOLDEN / "adult.tbnt").read_bytes())
    bad = bytearray(b)
    bad[100] ^= 0xFF
    with pytest.raises(P.ChecksumError):
        P.load_model(bytes(bad))
    fut = bytearray(b)
    fut[4:6] = struct.pack("<H", 2)
    with pytest.raises(P.FormatVersionError):
        P.load_model(bytes(fut))
    with pytest.raises(P.TruncatedStreamError):
        P.load_model(bytes(b[:8]))
    with pytest.raises(P.TruncatedStreamError):
        P.load_model(bytes(b[:200]))
    with pytest.raises(P.ModelFormatError):
        P.load_model(b"XXXX" + bytes(b[4:]))


def test_model_config_validation():
    with pytest.raises(P.ConfigurationError):
        P.ModelConfig(feature_count=0)
    with pytest.raises(P.ConfigurationError):
        P.ModelConfig(feature_count=3, n_classes=1)
    with pytest.raises(P.ConfigurationError):
        P.ModelConfig(feature_count=3, gamma=0.9)
    cfg = P.ModelConfig(feature_count=3)
    assert P.ModelConfig.from_dict(cfg.to_dict()) == cfg
    with pytest.raises(P.ConfigurationError):
        P.TabNetModel(config=cfg, params=P.init_parameters(cfg), norm_mean=np.zeros(3),
                      norm_var=np.array([1.0, 0.0, 1.0]), model_version="x")
    with pytest.raises(P.ConfigurationError):
        P.TabNetModel(config=cfg, params=P.init_parameters(cfg), norm_mean=np.zeros(3),
                      norm_var=np.ones(3), model_version="")


def test_apply_validates_before_touching_the_device():
    m = W.make_model("adult")
    with pytest.raises(P.InvalidInputError):
        m.apply(np.zeros((4, 13)))
    with pytest.raises(P.ConfigurationError):
        m.apply(np.zeros((4, 14)), with_caches=True)
    r = m.apply(np.zeros((0, 14)))
    assert r.masks.shape == (3, 0, 14) and r.probabilities.shape == (0, 2)


@pytest.mark.skipif(N.device_count() > 0, reason="only meaningful without a GPU")
def test_no_cpu_fallback_without_gpu():
    m = W.make_model("adult")
    with pytest.raises(P.DeviceError):
        m.apply(np.zeros((4, 14)))
    with pytest.raises(P.DeviceError):
        P.sparsemax(np.array([0.6, 0.4]))


def test_algorithmic_counts_match_survey():
    # FLOPs/row and bytes/row for predict+explain
    assert W.algorithmic_counts(W.WORKLOADS["adult"])["flops_per_row"] == 16576
    assert W.algorithmic_counts(W.WORKLOADS["hr"])["flops_per_row"] == 106272
    assert W.algorithmic_counts(W.WORKLOADS["wide"])["flops_per_row"] == 4654336
    assert W.algorithmic_counts(W.WORKLOADS["adult"])["bytes_per_row"] == 300
    assert W.algorithmic_counts(W.WORKLOADS["hr"])["bytes_per_row"] == 1000
    # BLS is the regression workload (C=1, one output value, no class)
    assert W.algorithmic_counts(W.WORKLOADS["bls"])["flops_per_row"] == 413760
    assert W.algorithmic_counts(W.WORKLOADS["bls"])["bytes_per_row"] == 1796


def _create(cfg_flags, n_classes, params_cfg):
    L = N.lib()
    cfg = N.TbnConfig(params_cfg.feature_count, n_classes, params_cfg.n_d, params_cfg.n_a,
                      params_cfg.n_steps, cfg_flags, 1.3)
    p = P.init_parameters(params_cfg)
    if n_classes == 1:
        p["head_W"] = p["head_W"][:, :1].copy()
        p["head_b"] = p["head_b"][:1].copy()
    keys = sorted(p)
    arrs = [np.ascontiguousarray(p[k]) for k in keys]
    names = (ctypes.c_char_p * len(keys))(*[k.encode() for k in keys])
    vals = (ctypes.c_void_p * len(keys))(*[a.ctypes.data for a in arrs])
    sizes = (ctypes.c_int64 * len(keys))(*[a.size for a in arrs])
    mean, var = np.zeros(params_cfg.feature_count), np.ones(params_cfg.feature_count)
    h = ctypes.c_void_p()
    st = L.tbn_model_create(ctypes.byref(cfg), names, vals, sizes, len(keys), mean.ctypes.data,
                            var.ctypes.data, 0, 0, ctypes.byref(h))
    if h.value:
        L.tbn_model_destroy(h)
    return st, L.tbn_last_error().decode()


def test_regression_config_validation_in_the_c_abi():
    """TBN_CFG_REGRESSION (the identity-head extension) needs n_classes == 1;
    without it the reference's n_classes >= 2 rule holds (config.py:32-33)."""
    cfg = P.ModelConfig(feature_count=5, n_d=4, n_a=4, n_steps=2)
    st, msg = _create(N.CFG_REGRESSION, 2, cfg)
    assert st == 2 and "n_classes == 1" in msg
    st, msg = _create(0, 1, cfg)
    assert st == 2 and "n_classes must be >= 2" in msg
    st, msg = _create(4, 2, cfg)
    assert st == 2 and "flags" in msg
    st, _ = _create(N.CFG_REGRESSION, 1, cfg)
    assert st in (0, 3, 4)          # valid config: OK on a GPU box, CUDA/UNSUPPORTED without one


def test_regressor_head_column_validation():
    with pytest.raises(P.ConfigurationError):
        P.TabNetRegressor.from_reference(W.make_model("bls"), head_column=2)
    r = P.TabNetRegressor.from_reference(W.make_model("bls"), head_column=1)
    assert r.head_column == 1 and r.n_outputs == 1


def test_workload_inputs_are_a_stream():
    w = W.WORKLOADS["hr"]
    a = W.make_inputs(w, 100)
    b = W.make_inputs(w, 40, start=60)
    assert a.dtype == np.float32 and np.array_equal(a[60:], b)
    g = np.load(GOLDEN / "hr_trained.npz")
    assert np.array_equal(W.make_inputs(w, 512), g["x"])
    mean, var = W.make_norm_stats(w)
    assert np.array_equal(mean, g["norm_mean"]) and np.array_equal(var, g["norm_var"])


def test_from_reference_duck_typing():
    m = W.make_model("hr")
    m2 = P.TabNetModel.from_reference(m, precision="fp32")
    assert m2.precision == "fp32" and m2.config == m.config
    assert all(np.array_equal(m.params[k], m2.params[k]) for k in m.params)


def test_native_tbnt_reader_replays_reference_cases():
    """csrc/tbnt.cpp against the unmodified reference loader (io.py:60-112) on
    the malformed and unusual streams of tests/golden/make_tbnt_cases.py: the same
    exception class for every rejected stream, the same model (re-serialized
    bytes) for every accepted one."""
    g = np.load(GOLDEN / "tbnt_cases.npz")
    names = sorted({k.split("__")[0] for k in g.files})
    assert len(names) >= 20
    classes = {"ok": None, "TruncatedStreamError": P.TruncatedStreamError,
               "ModelFormatError": P.ModelFormatError, "FormatVersionError": P.FormatVersionError,
               "ChecksumError": P.ChecksumError, "ConfigurationError": P.ConfigurationError}
    for name in names:
        stream = g[name + "__stream"].tobytes()
        expect = str(g[name + "__expect"])
        if expect == "ok":
            m = P.load_model(stream)
            assert P.save_model(m) == g[name + "__reserialized"].tobytes(), name
        else:
            with pytest.raises(classes[expect]) as ei:
                P.load_model(stream)
            # the exact class, not a sibling of the ModelFormatError family
            assert type(ei.value) is classes[expect], (name, type(ei.value))
