"""``metrics.accuracy`` / ``metrics.roc_auc`` against the reference's
``tabserve/model/training.py:177-202`` (bitwise) and a pairwise Mann-Whitney
count; the GPU test drives both the reference's helpers and ours with the GPU
model."""
import sys
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import ROOT
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import metrics

REF = ROOT / "baseline" / "_ref"


def _ref_training():
    if not (REF / "tabserve").exists():
        pytest.skip("reference not installed (tools/install_reference.sh)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from tabserve.model import training
    return training


class _Fixed:
    """A model stand-in whose apply returns fixed probabilities (host logic only)."""

    def __init__(self, p1):
        p1 = np.asarray(p1, dtype=np.float64)
        self.probs = np.stack([1.0 - p1, p1], axis=1)

    def apply(self, x):
        assert x.dtype == np.float64 and x.shape[0] == self.probs.shape[0]
        return SimpleNamespace(probabilities=self.probs)


def _cases():
    rng = np.random.default_rng(7)
    out = []
    for n, levels in [(2, 0), (17, 0), (500, 0), (500, 4), (2000, 37), (4096, 0), (3000, 2)]:
        p1 = rng.random(n) if levels == 0 else rng.integers(0, levels, n) / max(levels - 1, 1)
        y = rng.integers(0, 2, n)
        y[0], y[-1] = 0, 1                      # both classes present
        out.append((p1, y))
    return out


def _auc_pairwise(p1, y):
    pos, neg = p1[y == 1], p1[y == 0]
    gt = (pos[:, None] > neg[None, :]).sum()
    eq = (pos[:, None] == neg[None, :]).sum()
    return (gt + 0.5 * eq) / (pos.size * neg.size)


@pytest.mark.parametrize("i", range(7))
def test_roc_auc_matches_pairwise_count(i):
    p1, y = _cases()[i]
    m = _Fixed(p1)
    x = np.zeros((p1.size, 3))
    assert metrics.roc_auc(m, x, y) == pytest.approx(_auc_pairwise(p1, y), rel=0, abs=1e-12)


@pytest.mark.parametrize("i", range(7))
def test_metrics_bitwise_equal_to_reference(i):
    tr = _ref_training()
    p1, y = _cases()[i]
    m = _Fixed(p1)
    x = np.zeros((p1.size, 3))
    assert metrics.roc_auc(m, x, y) == tr.roc_auc(m, x, y)
    assert metrics.accuracy(m, x, y) == tr.accuracy(m, x, y)


def test_midranks_ties():
    r = metrics.midranks(np.array([3.0, 1.0, 3.0, 2.0, 3.0, 1.0]))
    np.testing.assert_array_equal(r, [5.0, 1.5, 5.0, 3.0, 5.0, 1.5])


def test_roc_auc_one_class_raises():
    m = _Fixed(np.array([0.2, 0.9, 0.4]))
    with pytest.raises(P.TrainingError, match="both classes"):
        metrics.roc_auc(m, np.zeros((3, 2)), np.array([1, 1, 1]))
    assert issubclass(P.TrainingError, P.TabserveError)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_reference_metrics_on_gpu_model(precision):
    """The reference's own accuracy/roc_auc called with the GPU model return the
    same numbers as ours (same apply), and track the CPU reference model's."""
    tr = _ref_training()
    from paper_2510_19689_b200 import workloads as W
    from tabserve.model.config import ModelConfig
    from tabserve.model.network import TabNetModel as RefModel
    m = W.make_engine_model("hr", "trained", precision=precision, device=0)
    x = W.make_inputs(W.WORKLOADS["hr"], 4096).astype(np.float64)
    ref = m.apply(x)
    y = (ref.probabilities[:, 1] > np.median(ref.probabilities[:, 1])).astype(np.int64)
    y[::7] ^= 1                                  # not a perfect separation
    assert metrics.roc_auc(m, x, y) == tr.roc_auc(m, x, y)
    assert metrics.accuracy(m, x, y) == tr.accuracy(m, x, y)
    c = m.config
    cpu = RefModel(config=ModelConfig(feature_count=c.feature_count, n_classes=c.n_classes, n_d=c.n_d,
                                      n_a=c.n_a, n_steps=c.n_steps, gamma=c.gamma),
                   params=m.params, norm_mean=m.norm_mean, norm_var=m.norm_var,
                   model_version=m.model_version)
    tol = 1e-6 if precision == "tf32x3" else 5e-3
    assert abs(metrics.roc_auc(m, x, y) - tr.roc_auc(cpu, x, y)) <= tol
    assert abs(metrics.accuracy(m, x, y) - tr.accuracy(cpu, x, y)) <= (2 / 4096 if precision == "tf32x3" else 0.02)
