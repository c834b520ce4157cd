"""The UNMODIFIED reference callers driving the GPU model (SURVEY.md §8(b)
"callers who must not notice", §8(f)1/3).

``tabserve`` is installed from the reference into ``baseline/_ref`` by
tools/install_reference.sh (git-ignored, shipped to the GPU box); nothing here
reads /root/reference.  The GPU model is duck-typed into
* ``serving.service.InferenceService`` (service.py:112-187, apply at :144) with
  the "baseline" security preset (an empty chain, chain.py:28-29);
* ``interpret.invariance.load_invariance_check`` (invariance.py:56-82), incl.
  its negative control;
* ``interpret.stability.stability_score`` (stability.py:95-110).
"""
import sys
import uuid

import numpy as np
import pytest

from conftest import ROOT
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import workloads as W

REF = ROOT / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "tabserve").exists(),
                                 reason="reference not installed (tools/install_reference.sh)")]


@pytest.fixture(scope="module")
def tabserve():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import tabserve
    return tabserve


def _ref_model(tabserve, m):
    from tabserve.model.config import ModelConfig
    from tabserve.model.network import TabNetModel as RefModel
    c = m.config
    cfg = ModelConfig(feature_count=c.feature_count, n_classes=c.n_classes, n_d=c.n_d, n_a=c.n_a,
                      n_steps=c.n_steps, gamma=c.gamma)
    return RefModel(config=cfg, params=m.params, norm_mean=m.norm_mean, norm_var=m.norm_var,
                    model_version=m.model_version)


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_inference_service_serves_the_gpu_model(tabserve, precision):
    from tabserve.security.chain import SecurityChain, SecurityChainConfig
    from tabserve.serving.batching import BatcherConfig, InferenceRequest
    from tabserve.serving.service import InferenceService
    m = P.TabNetModel.from_reference(W.make_model("hr"), precision=precision)
    svc = InferenceService(m, SecurityChain(SecurityChainConfig.preset("baseline")),
                           batcher=BatcherConfig(max_batch=64, max_delay_ms=2.0), parallelism=4).start()
    try:
        rng = np.random.default_rng(3)
        x = W.make_inputs(W.WORKLOADS["hr"], 600).astype(np.float64)
        sizes = rng.integers(1, 9, 120)
        reqs, off = [], 0
        for n in sizes:
            if off + n > x.shape[0]:
                break
            reqs.append((off, n, svc.submit(InferenceRequest(request_id=str(uuid.uuid4()), features=x[off:off + n]))))
            off += n
        payloads = [(o, n, t.future.result(timeout=60)) for o, n, t in reqs]
    finally:
        svc.stop()
    assert svc.error_responses == 0 and svc.responses == len(payloads)
    direct = m.apply(x[:off])            # the service only slices one apply() per batch
    ref = _ref_model(tabserve, m).apply(x[:off])
    for o, n, pl in payloads:
        assert pl["model_version"] == m.model_version and len(pl["results"]) == n
        for j, rec in enumerate(pl["results"]):
            r = o + j
            assert rec["probabilities"] == direct.probabilities[r].tolist()
            assert rec["masks"] == direct.masks[:, r, :].tolist()
            assert rec["importance"] == direct.importance[r].tolist()
            assert rec["prediction"] == int(np.argmax(direct.probabilities[r]))
    tol = 1e-5 if precision == "tf32x3" else 3e-2
    np.testing.assert_allclose(direct.probabilities, ref.probabilities, atol=tol)


@pytest.mark.parametrize("precision", ["tf32x3", "bf16"])
def test_reference_load_invariance_check_on_gpu_model(tabserve, precision):
    from tabserve.interpret.invariance import load_invariance_check
    m = P.TabNetModel.from_reference(W.make_model("hr"), precision=precision)
    x = W.make_inputs(W.WORKLOADS["hr"], 512).astype(np.float64)
    res = load_invariance_check(m, x)
    assert res.passed, res.detail
    neg = load_invariance_check(m, x, use_batch_stats=True)
    assert not neg.passed and neg.first_diff is not None


def test_reference_stability_score_on_gpu_model(tabserve):
    from tabserve.interpret.stability import stability_score
    m = P.TabNetModel.from_reference(W.make_model("hr"), precision="tf32x3")
    x = W.make_inputs(W.WORKLOADS["hr"], 2048, seed=77).astype(np.float64)
    got = stability_score(m, x, 8)
    want = stability_score(_ref_model(tabserve, m), x, 8)
    g = {f.name: f for f in got.features}
    w = {f.name: f for f in want.features}
    assert g.keys() == w.keys() and got.sample_count == want.sample_count
    for k in w:
        assert abs(g[k].mean_importance - w[k].mean_importance) < 1e-5, k
        assert abs(g[k].stability - w[k].stability) < 1e-3 * max(1.0, abs(w[k].stability)), k
    # the order is by mean importance: equal wherever the reference's means are apart
    means = np.array([f.mean_importance for f in want.features])
    apart = np.all(np.abs(means[:, None] - means[None, :]) + np.eye(len(means)) > 1e-4, axis=1)
    for i, f in enumerate(want.features):
        if apart[i]:
            assert got.features[i].name == f.name
    assert abs(got.rank_variance - want.rank_variance) < 0.05 * max(1.0, abs(want.rank_variance))
