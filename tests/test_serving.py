"""Serving response building (paper_2510_19689_b200/serving.py) against the
reference's per-row record loop (serving/service.py:166-183)."""
import numpy as np
import pytest

import paper_2510_19689_b200 as P
from paper_2510_19689_b200.serving import build_records, process_rows, split_records


def _reference_records(results, sizes):
    # restatement of InferenceService._process_batch's response loop
    # (service.py:166-183): offset walk over the stacked requests
    out, offset = [], 0
    for n in sizes:
        sl = slice(offset, offset + n)
        offset += n
        records = []
        for j in range(sl.start, sl.stop):
            records.append({
                "prediction": int(np.argmax(results.probabilities[j])),
                "probabilities": results.probabilities[j].tolist(),
                "masks": results.masks[:, j, :].tolist(),
                "importance": results.importance[j].tolist(),
            })
        out.append(records)
    return out


def _random_result(b, c, s, f, seed=0):
    rng = np.random.default_rng(seed)
    probs = rng.random((b, c))
    if c > 1:
        probs[::3, 1] = probs[::3, 0]             # exact top ties: lowest index wins
    return P.ForwardResult(logits=rng.standard_normal((b, c)), probabilities=probs,
                           masks=rng.random((s, b, f)), importance=rng.random((b, f)))


@pytest.mark.parametrize("shape", [(37, 3, 4, 9), (1, 2, 5, 35), (64, 1, 5, 64), (0, 2, 3, 14)])
def test_records_equal_reference_loop(shape):
    r = _random_result(*shape)
    b = shape[0]
    sizes = [b] if b < 3 else [1, b // 2 - 1, b - b // 2]
    want = _reference_records(r, sizes)
    got = split_records(r, sizes)
    assert got == want
    for recs in got:
        for rec in recs:
            assert type(rec["prediction"]) is int
            assert all(type(v) is float for v in rec["probabilities"])


def test_build_records_slices_and_errors():
    r = _random_result(10, 2, 3, 4)
    assert build_records(r, 3, 7) == _reference_records(r, [3, 4, 3])[1]
    assert build_records(r, 5, 5) == []
    with pytest.raises(P.InvalidInputError):
        build_records(r, 4, 11)
    with pytest.raises(P.InvalidInputError):
        split_records(r, [3, 3])


@pytest.mark.gpu
def test_process_rows_through_the_gpu_model():
    from paper_2510_19689_b200 import workloads as W
    m = W.make_engine_model("hr", "trained")
    x = W.make_inputs(W.WORKLOADS["hr"], 300).astype(np.float64)
    feats = [x[:1], x[1:45], x[45:300]]
    result, recs = process_rows(m, feats)
    assert [len(v) for v in recs] == [1, 44, 255]
    assert recs == _reference_records(result, [1, 44, 255])
    ref = m.apply(x)                                # the same rows in one call: same values
    np.testing.assert_array_equal(result.probabilities, ref.probabilities)
