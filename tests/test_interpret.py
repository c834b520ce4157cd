"""Explain consumers (paper_2510_19689_b200/interpret.py): stability against
golden vectors of the reference's interpret/stability.py
(tests/golden/make_stability_golden.py) and the on-device load-invariance check
(interpret/invariance.py)."""
import numpy as np
import pytest

from conftest import load_golden
import paper_2510_19689_b200 as P
from paper_2510_19689_b200 import interpret as I

CASES = ["random", "zeros_ties", "two_partitions", "many_partitions"]


@pytest.fixture(scope="module")
def gold():
    return load_golden("stability")


@pytest.mark.parametrize("case", CASES)
def test_stability_from_batches_matches_reference(gold, case):
    rep = I.stability_from_batches(gold[f"{case}__in"], sample_count=123, load_mode="offline")
    assert [f.name for f in rep.features] == list(gold[f"{case}__names"])
    np.testing.assert_array_equal([f.mean_importance for f in rep.features], gold[f"{case}__mean"])
    np.testing.assert_array_equal([f.stability for f in rep.features], gold[f"{case}__stability"])
    assert rep.rank_variance == float(gold[f"{case}__rank_variance"])
    assert rep.to_csv() == str(gold[f"{case}__csv"])
    assert rep.to_json() == str(gold[f"{case}__json"])
    assert rep.partition_count == gold[f"{case}__in"].shape[0] and rep.sample_count == 123
    assert rep.top(2) == rep.features[:2]


def test_stability_errors():
    with pytest.raises(P.InvalidInputError):
        I.stability_from_batches(np.ones((1, 4)))
    with pytest.raises(P.InvalidInputError):
        I.stability_from_batches(np.ones(4))
    with pytest.raises(P.InvalidInputError):
        I.stability_score(None, np.ones((3, 4)), partitions=1)
    with pytest.raises(P.InvalidInputError):
        I.stability_score(None, np.ones((3, 4)), partitions=4)


@pytest.mark.gpu
def test_partition_mean_kernel():
    import torch
    from paper_2510_19689_b200 import _native as N
    g = torch.Generator().manual_seed(3)
    for parts, per, w in [(1, 1, 1), (3, 1000, 35), (7, 129, 513), (64, 8, 14)]:
        v = torch.rand(parts * per, w, generator=g).cuda()
        out = torch.empty(parts, w, dtype=torch.float64, device="cuda")
        N.check(N.lib().tbn_partition_mean(v.data_ptr(), per, parts, w, out.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream))
        want = v.double().view(parts, per, w).mean(dim=1)
        torch.testing.assert_close(out, want, rtol=1e-12, atol=0)
    assert N.lib().tbn_partition_mean(v.data_ptr(), 0, 1, 1, out.data_ptr(), None) != 0


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol_mean,tol_stab", [("tf32x3", 5e-6, 1e-4), ("bf16", 2e-2, 0.2)])
def test_stability_score_gpu_vs_reference(gold, precision, tol_mean, tol_stab):
    from paper_2510_19689_b200 import workloads as W
    m = W.make_engine_model("hr", "trained", precision=precision)
    rows, parts = int(gold["hr__rows"]), int(gold["hr__partitions"])
    x = W.make_inputs(W.WORKLOADS["hr"], rows, seed=int(gold["hr__x_seed"])).astype(np.float64)
    means = I.partition_mean_importance(m, x, parts)
    ref = gold["hr__means"]
    assert means.shape == ref.shape
    assert np.abs(means - ref).max() <= tol_mean
    rep = I.stability_score(m, x, parts)
    assert rep.partition_count == parts and rep.sample_count == (rows // parts) * parts
    want = dict(zip(gold["hr__names"], gold["hr__stability"]))
    got = {f.name: f.stability for f in rep.features}
    assert max(abs(got[k] - want[k]) for k in want) <= tol_stab
    if precision == "tf32x3":
        # the report built from the reference's own means is the golden one
        rep_ref = I.stability_from_batches(ref)
        assert [f.name for f in rep_ref.features] == list(gold["hr__names"])
        assert rep_ref.rank_variance == float(gold["hr__rank_variance"])
        assert abs(rep.rank_variance - float(gold["hr__rank_variance"])) <= 1e-2


@pytest.mark.gpu
def test_stability_score_rejects_non_finite():
    from paper_2510_19689_b200 import workloads as W
    m = W.make_engine_model("hr", "trained", precision="bf16")
    x = W.make_inputs(W.WORKLOADS["hr"], 64).astype(np.float64)
    x[17, 3] = np.nan
    with pytest.raises(P.InvalidInputError):
        I.stability_score(m, x, 4)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,precision,rows,conc,bss", [
    ("hr", "tf32x3", 300, (1, 32), (1, 256)),
    ("adult", "bf16", 200, (1, 8), (3, 64)),
    ("wide", "bf16", 130, (1, 4), (1, 128)),
])
def test_load_invariance_check_on_device(cfg, precision, rows, conc, bss):
    from paper_2510_19689_b200 import workloads as W
    m = W.make_engine_model(cfg, "trained", precision=precision)
    x = W.make_inputs(W.WORKLOADS[cfg], rows).astype(np.float64)
    res = I.load_invariance_check(m, x, concurrency=conc, batch_sizes=bss)
    assert res.passed and res.first_diff is None and res.detail == ""
    neg = I.load_invariance_check(m, x, concurrency=conc, batch_sizes=bss, use_batch_stats=True)
    assert not neg.passed
    s, f = neg.first_diff
    assert 0 <= s < rows and 0 <= f < x.shape[1]
    assert neg.detail.startswith(("mask diff at sample", "importance diff at sample"))
    # the device explanations are the host apply's values
    ref = m.apply(x)
    import torch
    xd = torch.from_numpy(x.astype(np.float32)).cuda()
    masks, imp = I._device_explanations(m, xd, 7, 3, 0)
    np.testing.assert_array_equal(masks.cpu().numpy().astype(np.float64), ref.masks)
    np.testing.assert_array_equal(imp.cpu().numpy().astype(np.float64), ref.importance)
