"""The rounding-faithful K2 emulation oracle (oracle/tabnet_emulate.py), CPU.

Pins its primitives (operand rounding, correctly rounded reciprocals, the
bias hi/lo split) and its relation to the float64 oracle: the emulation is the
reference algorithm with the kernel's operand rounding, so its distance to the
float64 oracle is the single-pass mode's intrinsic error and must shrink from
bf16 to tf32; with exact arithmetic switched in it reproduces the oracle.
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2510_19689_b200 import workloads as W
from oracle import tabnet_emulate as E
from oracle import tabnet_oracle as O


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 20000),
                        np.float32([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 65504.0, 3.3895e38])])
    v = v.astype(np.float32)
    want = torch.from_numpy(v).to(torch.bfloat16).float().numpy()
    assert np.array_equal(E.bf16_rne(v), want)


def test_tf32_roundings():
    x = np.float32([1.0 + 2 ** -11, 1.0 + 2 ** -10 + 2 ** -11, -(1.0 + 2 ** -11), 3.0])
    # round half away: 1 + 2^-11 is exactly halfway between tf32 neighbours 1 and 1 + 2^-10
    assert E.tf32_rna(x).tolist() == [1.0 + 2 ** -10, 1.0 + 2 ** -9, -(1.0 + 2 ** -10), 3.0]
    assert E.tf32_trunc(x).tolist() == [1.0, 1.0 + 2 ** -10, -1.0, 3.0]


def test_correctly_rounded_reciprocals():
    for k in range(1, 600):
        r = E.rcp_rn(k)
        err = abs(Fraction(float(r)) - Fraction(1, k))
        for nb in (np.nextafter(r, np.float32(0)), np.nextafter(r, np.float32(2))):
            assert err <= abs(Fraction(float(nb)) - Fraction(1, k))
    for v in (np.float32(3.0), np.float32(0.7), np.float32(1e-20), np.float32(12345.678)):
        r = E.rcp_rn_float(v)
        assert abs(Fraction(float(r)) * Fraction(float(v)) - 1) <= Fraction(1, 2 ** 23)


def test_bias_hi_lo_rows_keep_fp32_precision():
    """The K2 packer's bias split: hi + lo reaches ~2^-17 relative in bf16 (one
    bf16 rounding alone is 2^-9)."""
    rng = np.random.default_rng(1)
    b = rng.standard_normal(64) * 3.0
    blk = E.PackedB(np.zeros((4, 64)), b, None, "bf16")
    got = blk.bias.astype(np.float64) + blk.bias_lo.astype(np.float64)
    assert np.max(np.abs(got - b) / np.abs(b)) < 2 ** -15
    assert np.max(np.abs(blk.bias.astype(np.float64) - b) / np.abs(b)) > 2 ** -12


@pytest.mark.parametrize("name", ["adult", "hr"])
def test_emulation_error_is_the_modes_intrinsic_error(name):
    m = W.make_model(name, "trained")
    x = W.make_inputs(W.WORKLOADS[name], 512)
    ref = O.apply_model(m, x.astype(np.float64))
    mass = np.abs(ref["masks"]).sum(-1)
    errs = {}
    for mode in ("bf16", "tf32"):
        e = E.apply_model_emulated(m, x, mode=mode)
        errs[mode] = (np.abs(e["masks"] - ref["masks"]).max(-1) / mass).max()
        assert np.abs(e["probabilities"] - ref["probabilities"]).max() < (3e-2 if mode == "bf16" else 5e-3)
        np.testing.assert_allclose(e["masks"].sum(-1), 1.0, atol=1e-5)
        np.testing.assert_allclose(e["importance"].sum(-1), 1.0, atol=1e-5)
    assert errs["tf32"] < errs["bf16"] / 3


def test_emulated_sparsemax_is_the_reference_projection():
    """The K2 Michelot iteration (float32, the kernel's order) against the
    reference's sort/cumsum sparsemax on random logits."""
    rng = np.random.default_rng(5)
    for F in (14, 35, 64):
        z = (rng.standard_normal((2000, F)) * rng.uniform(0.1, 20, (2000, 1))).astype(np.float32)
        rcp = np.array([np.float32(0)] + [E.rcp_rn(k) for k in range(1, F + 1)], np.float32)
        zs, tau = E._sparsemax_k2(z, rcp)
        m = np.maximum(zs - tau[:, None], 0)
        ref = O.sparsemax(z.astype(np.float64))
        assert np.abs(m - ref).max() < 2e-5 * np.abs(z).max()
