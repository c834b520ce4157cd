"""Device preprocessing against the reference ETL.

tests/golden/preprocess.npz holds, for HR and Adult, a PreprocessPlan fitted by
the unmodified reference, raw cells of a second table (with extra missing cells
and unseen levels) and the reference's PreprocessPlan.transform output
(preprocess.py:68-122).  CPU: the host encoding + a NumPy restatement of the
device expansion reproduce that matrix; GPU: tbn_preprocess reproduces it
cast to float32 bit for bit, and the table -> forward path equals
model.apply on the reference matrix bit for bit.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import preprocess as PP


def _case(name):
    g = np.load(GOLDEN / "preprocess.npz")
    return (json.loads(str(g[f"{name}__plan"])), json.loads(str(g[f"{name}__columns"])), int(g[f"{name}__rows"]),
            g[f"{name}__matrix"], json.loads(str(g[f"{name}__names"])), json.loads(str(g[f"{name}__unseen"])))


def _expand(pc: PP.PlanCodes, codes: np.ndarray) -> np.ndarray:
    """NumPy restatement of csrc/kernel_prep.cu (float64, then float32)."""
    blocks = []
    for c, t in enumerate(pc.transforms):
        v = codes[:, c]
        if t["kind"] in ("standardize", "passthrough"):
            x = np.where(np.isnan(v), t["median"], v)
            blocks.append(((x - t["mean"]) / t["std"] if t["kind"] == "standardize" else x)[:, None])
        elif t["kind"] == "ordinal":
            blocks.append(v[:, None])
        else:
            blocks.append((v[:, None] == np.arange(len(t["categories"]))[None, :]).astype(np.float64))
    return np.hstack(blocks).astype(np.float32)


@pytest.mark.parametrize("name", ["hr", "adult"])
def test_host_encoding_matches_reference_transform(name):
    plan, cols, rows, matrix, names, unseen = _case(name)
    pc = PP.PlanCodes(plan)
    codes, got_unseen = pc.encode(cols, rows)
    assert pc.column_names == names and pc.width == matrix.shape[1]
    assert got_unseen == unseen
    assert np.array_equal(_expand(pc, codes), matrix.astype(np.float32))


def test_encoding_rejects_non_finite_values():
    plan, cols, rows, *_ = _case("hr")
    pc = PP.PlanCodes(plan)
    num = next(t["label"] for t in pc.transforms if t["kind"] == "standardize")
    bad = dict(cols)
    bad[num] = list(cols[num])
    bad[num][3] = float("nan")
    with pytest.raises(P.InvalidInputError):
        pc.encode(bad, rows)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["hr", "adult"])
def test_device_preprocessing_bitwise(name):
    plan, cols, rows, matrix, names, unseen = _case(name)
    dp = PP.DevicePreprocessor(plan, device=0)
    got, got_unseen = dp.transform(cols, rows)
    assert got_unseen == unseen
    assert got.dtype == np.float32 and np.array_equal(got, matrix.astype(np.float32))


@pytest.mark.gpu
def test_table_to_forward_on_device():
    """Raw HR table (52 features after one-hot) -> codes ->
    device preprocessing -> fused forward equals model.apply on the reference's
    matrix, bit for bit."""
    plan, cols, rows, matrix, names, unseen = _case("hr")
    F = matrix.shape[1]
    cfg = P.ModelConfig(feature_count=F, n_classes=2, n_d=8, n_a=8, n_steps=3)
    prm = P.init_parameters(cfg)
    mean, var = matrix.mean(0), matrix.var(0) + 0.5
    m = P.TabNetModel(config=cfg, params=prm, norm_mean=mean, norm_var=var, model_version="hr52",
                      precision="auto")
    dp = PP.DevicePreprocessor(plan, device=0)
    r = PP.apply_table(m, dp, cols, rows)
    want = m.apply(matrix.astype(np.float32).astype(np.float64))
    for k in ("logits", "probabilities", "masks", "importance"):
        assert np.array_equal(getattr(r, k), getattr(want, k)), k
