"""Rounding-faithful CPU emulation of the K2 single-pass modes — TEST
INFRASTRUCTURE ONLY (same import rule as ``tabnet_oracle``: tests/, smoke()
and bench.py's CPU legs).

``tabnet_oracle.apply`` is the reference's float64 algorithm; the bf16 / tf32
kernels differ from it by their operand rounding, so comparing them to it
needs a loose bound.  This module re-evaluates the same forward
(reference network.py:195-267, sparsemax.py:13-41) with the arithmetic the
K2 kernel (paper_2510_19689_b200/csrc/k2_kernel.cuh) and its packer
(csrc/kernel_k2.cu, csrc/pack_util.h) actually perform, step for step in
float32:

* weights: the packer's folded constants in float64 (GLU columns x 1/2 for the
  tanh form, the residual blocks' linear columns x sqrt(1/2)/2,
  network.py:131-137), then one rounding to the operand format (bf16 RNE;
  tf32 round-half-away); the bias as two rows hi = round(b), lo = round(b - hi);
* A operands: bf16 RNE of the float32 activations (``__floats2bfloat162_rn``),
  or tf32 by truncation (the tensor core reads fp32 as tf32);
* MMA: exact products summed in float64, rounded once to float32 (the tensor
  core's internal summation order is not specified; this differs from it by
  about one float32 ulp of the sum);
* GLU: ``o = fma(l, t, fma(prev, sqrt(1/2), l))`` with ``t = tanh(gate')`` —
  the kernel's ``tanh.approx.f32`` (relative error <= 2^-10.99) is modelled by
  the exact tanh, the one deliberate gap (``tanh_fn`` lets a test perturb it);
* sparsemax: the kernel's sort-free Michelot fixed point with its float32
  accumulation order and start value, tau = (sum - 1) * rcp(count) with the
  correctly rounded reciprocal (the kernel's table);
* head, softmax, argmax, importance (with the all-eta-zero fallback) in the
  kernel's float32 order.

What it is for: the bf16 headline mode can be held to a tight bound against
this emulation (its remaining differences are the tanh approximation and the
MMA summation order), while the float64 oracle can only bound it loosely.
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

R = math.sqrt(0.5)
F32 = np.float32


def bf16_rne(a: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 (ties to even), returned as float32 values."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def tf32_rna(a: np.ndarray) -> np.ndarray:
    """float32 -> tf32, round half away from zero (the packer's B operands)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x1000) & 0xFFFFE000).astype(np.uint32).view(np.float32)


def tf32_trunc(a: np.ndarray) -> np.ndarray:
    """How the tensor core reads an fp32 A operand in kind::tf32."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return (u & np.uint32(0xFFFFE000)).view(np.float32)


def fma32(a, b, c) -> np.ndarray:
    """float32 fused multiply-add (exact product, one rounding)."""
    return (np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(F32)


def rcp_rn(k: int) -> np.float32:
    """Correctly rounded float32 reciprocal of a positive integer (exact rational rounding)."""
    q = Fraction(1, k)
    f = F32(1.0 / k)
    # pick the float32 neighbour nearest to 1/k (ties to even)
    cands = [np.nextafter(f, F32(0)), f, np.nextafter(f, F32(2))]
    best = min(cands, key=lambda c: (abs(Fraction(float(c)) - q), int(np.asarray(c).view(np.uint32)) & 1))
    return F32(best)


class PackedB:
    """One B operand block as the K2 packer builds it: W^T (N x Kp) with rows
    k = 0, 1 = bias hi / lo and rows 2 .. Kin+1 = W, stored as operand-format
    values (float32 holding bf16 / tf32 numbers)."""

    def __init__(self, W: np.ndarray, b: np.ndarray | None, colscale: np.ndarray | None, fmt: str):
        Kin, N = W.shape
        cs = np.ones(N) if colscale is None else np.asarray(colscale, np.float64)
        Wd = np.asarray(W, np.float64) * cs[None, :]
        rnd = bf16_rne if fmt == "bf16" else tf32_rna
        self.W = rnd(Wd.astype(F32))                           # (Kin, N)
        if b is None:
            self.bias = np.zeros(N, F32)
            self.bias_lo = np.zeros(N, F32)
        else:
            bd = np.asarray(b, np.float64) * cs
            hi = rnd(bd.astype(F32))
            self.bias = hi
            self.bias_lo = rnd((bd - hi.astype(np.float64)).astype(F32))

    def matmul(self, A: np.ndarray) -> np.ndarray:
        """D = [1, 1, A] @ [hi; lo; W] with exact products, float64 sum, one float32 rounding."""
        acc = A.astype(np.float64) @ self.W.astype(np.float64)
        acc += self.bias.astype(np.float64)[None, :] + self.bias_lo.astype(np.float64)[None, :]
        return acc.astype(F32)


def _sparsemax_k2(z: np.ndarray, rcp: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """k2_kernel.cuh's per-row sparsemax on float32 logits z (B, F): returns
    (z - zmax, tau) in the kernel's float32 arithmetic."""
    B, F = z.shape
    ev, od = z[:, 0:F - 1:2], z[:, 1:F:2]
    m0 = ev.max(axis=1) if ev.shape[1] else np.full(B, -np.inf, F32)
    m1 = od.max(axis=1) if od.shape[1] else np.full(B, -np.inf, F32)
    # pairwise accumulation: s2.x += z[even], s2.y += z[odd] in index order
    sx = np.zeros(B, F32)
    sy = np.zeros(B, F32)
    for i in range(0, F - 1, 2):
        sx = (sx + z[:, i]).astype(F32)
        sy = (sy + z[:, i + 1]).astype(F32)
    if F % 2:
        m0 = np.maximum(m0, z[:, F - 1])
        sx = (sx + z[:, F - 1]).astype(F32)
    zmax = np.maximum(m0, m1).astype(F32)
    zsum = (sx + sy).astype(F32)
    zs = (z - zmax[:, None]).astype(F32)
    bound = ((zsum - (F32(F) * zmax).astype(F32)).astype(F32) - F32(1.0)).astype(F32) * F32(1.0 / F)
    bound = bound.astype(F32)
    tau = np.maximum(F32(-1.0), (bound - (F32(9.5367431640625e-07) * np.maximum(F32(1.0), np.abs(bound))).astype(F32)).astype(F32))
    cnt_prev = np.full(B, F + 1, F32)
    active = np.ones(B, bool)
    for _ in range(F + 1):
        if not active.any():
            break
        mk = (zs > tau[:, None]).astype(F32)
        # four float2 accumulators: pairs (i, i+1) alternate between a and b by (i/2)%2
        sa = np.zeros((B, 2), F32); ca = np.zeros((B, 2), F32)
        sb = np.zeros((B, 2), F32); cb = np.zeros((B, 2), F32)
        for i in range(0, F - 1, 2):
            zp = zs[:, i:i + 2]
            mp = mk[:, i:i + 2]
            if (i // 2) % 2 == 0:
                sa = fma32(mp, zp, sa)
                ca = (ca + mp).astype(F32)
            else:
                sb = fma32(mp, zp, sb)
                cb = (cb + mp).astype(F32)
        s2 = (sa + sb).astype(F32)
        c2 = (ca + cb).astype(F32)
        sm = (s2[:, 0] + s2[:, 1]).astype(F32)
        cn = (c2[:, 0] + c2[:, 1]).astype(F32)
        if F % 2:
            sm = fma32(mk[:, F - 1], zs[:, F - 1], sm)
            cn = (cn + mk[:, F - 1]).astype(F32)
        stop = cn >= cnt_prev
        upd = active & ~stop
        cnt_prev = np.where(upd, cn, cnt_prev)
        ci = np.clip(cn.astype(np.int64), 1, F)
        tnew = ((sm - F32(1.0)).astype(F32) * rcp[ci]).astype(F32)
        tau = np.where(upd, tnew, tau)
        active &= ~stop
    return zs, tau


def apply_emulated(params: dict, norm_mean: np.ndarray, norm_var: np.ndarray, *, n_d: int, n_steps: int,
                   gamma: float, x: np.ndarray, mode: str = "bf16", normalized: bool = False,
                   tanh_fn=np.tanh) -> dict:
    """The K2 forward in ``mode`` ("bf16" or "tf32") on float32 inputs ``x``.
    Returns float64 copies of logits, probabilities, masks (S,B,F), importance."""
    assert mode in ("bf16", "tf32")
    x = np.asarray(x, F32)
    if x.ndim == 1:
        x = x[None, :]
    B, F = x.shape
    p = params
    h = p["shared2_W"].shape[0]
    n_a = h - n_d
    C = p["head_W"].shape[1]
    fmt = mode
    a_round = bf16_rne if mode == "bf16" else tf32_trunc
    # packer constants (kernel_k2.cu pack_k2): tanh-form GLU folding
    cs_first = np.full(2 * h, 0.5)
    cs_res = np.concatenate([np.full(h, 0.5 * R), np.full(h, 0.5)])
    sh1 = PackedB(p["shared1_W"], p["shared1_b"], cs_first, fmt)
    sh2 = PackedB(p["shared2_W"], p["shared2_b"], cs_res, fmt)
    fc1 = [PackedB(p[f"step{s}_fc1_W"], p[f"step{s}_fc1_b"], cs_res, fmt) for s in range(n_steps + 1)]
    fc2 = [PackedB(p[f"step{s}_fc2_W"], p[f"step{s}_fc2_b"], cs_res, fmt) for s in range(n_steps + 1)]
    att = [None] + [PackedB(p[f"step{s}_att_W"], p[f"step{s}_att_b"], None, fmt) for s in range(1, n_steps + 1)]
    scale = (1.0 / np.sqrt(np.asarray(norm_var, np.float64) + 1e-8)).astype(F32)
    shift = np.asarray(norm_mean, np.float64).astype(F32)
    head_w = np.asarray(p["head_W"], np.float64).astype(F32)
    head_b = np.asarray(p["head_b"], np.float64).astype(F32)
    rcp = np.array([F32(0)] + [rcp_rn(k) for k in range(1, F + 1)], F32)
    R32 = F32(R)
    g32 = F32(gamma)

    xn = x if normalized else ((x - shift).astype(F32) * scale).astype(F32)

    def glu(D: np.ndarray, prev: np.ndarray | None) -> np.ndarray:
        lin, gate = D[:, :h], D[:, h:]
        t = tanh_fn(gate.astype(F32)).astype(F32)
        w = lin if prev is None else fma32(prev, R32, lin)
        return fma32(lin, t, w)

    def transform(v: np.ndarray, s: int) -> np.ndarray:
        g = glu(sh1.matmul(a_round(v)), None)
        g = glu(sh2.matmul(a_round(g)), g)
        g = glu(fc1[s].matmul(a_round(g)), g)
        return glu(fc2[s].matmul(a_round(g)), g)

    gv = transform(xn, 0)
    prior = np.ones((B, F), F32)
    agg = np.zeros((B, F), F32)
    lacc = np.zeros((B, C), F32)
    all_eta_zero = np.ones(B, bool)
    masks = np.empty((n_steps, B, F), F32)

    def step_eta(gv, lacc):
        e0 = np.zeros(B, F32)
        e1 = np.zeros(B, F32)
        for i in range(n_d):
            d = np.maximum(gv[:, i], F32(0))
            lacc = fma32(d[:, None], head_w[i][None, :], lacc)
            if i & 1:
                e1 = (e1 + d).astype(F32)
            else:
                e0 = (e0 + d).astype(F32)
        return (e0 + e1).astype(F32), lacc

    def agg_apply(agg, m, eta, all_eta_zero):
        pos = eta > 0
        reset = all_eta_zero & pos
        w = np.where(all_eta_zero, np.where(pos, eta, F32(1.0)), eta).astype(F32)
        agg = np.where(reset[:, None], F32(0), agg)
        agg = fma32(w[:, None], m, agg)
        return agg, all_eta_zero & ~pos

    for s in range(1, n_steps + 1):
        a = gv[:, n_d:]
        if s > 1:
            eta, lacc = step_eta(gv, lacc)
            agg, all_eta_zero = agg_apply(agg, masks[s - 2], eta, all_eta_zero)
        z = (prior * att[s].matmul(a_round(a))).astype(F32)
        zs, tau = _sparsemax_k2(z, rcp)
        m = np.maximum((zs - tau[:, None]).astype(F32), F32(0))
        prior = (prior * (g32 - m).astype(F32)).astype(F32)
        xm = (m * xn).astype(F32)
        masks[s - 1] = m
        gv = transform(xm, s)
    eta, lacc = step_eta(gv, lacc)
    agg, all_eta_zero = agg_apply(agg, masks[n_steps - 1], eta, all_eta_zero)

    lg = (lacc + head_b[None, :]).astype(F32)
    lmax = lg.max(axis=1)
    ex = np.exp((lg - lmax[:, None]).astype(F32)).astype(F32)
    es = np.zeros(B, F32)
    for c in range(C):
        es = (es + ex[:, c]).astype(F32)
    probs = (ex / es[:, None]).astype(F32)
    t0 = agg[:, 0::2].astype(np.float64)
    t1 = agg[:, 1::2].astype(np.float64)
    s0 = np.zeros(B, F32)
    s1 = np.zeros(B, F32)
    for f in range(F):
        if f & 1:
            s1 = (s1 + agg[:, f]).astype(F32)
        else:
            s0 = (s0 + agg[:, f]).astype(F32)
    del t0, t1
    div = np.where(all_eta_zero, F32(n_steps), (s0 + s1).astype(F32)).astype(F32)
    rdiv = np.array([rcp_rn_float(v) for v in div], F32) if B <= 4096 else (1.0 / div.astype(np.float64)).astype(F32)
    imp = (agg * rdiv[:, None]).astype(F32)
    return dict(logits=lg.astype(np.float64), probabilities=probs.astype(np.float64),
                masks=masks.astype(np.float64), importance=imp.astype(np.float64))


def rcp_rn_float(v: np.float32) -> np.float32:
    """Correctly rounded float32 reciprocal of a float32 value (``__frcp_rn``)."""
    v = float(v)
    if v == 0.0 or not math.isfinite(v):
        return F32(1.0 / v) if v != 0.0 else F32(np.inf)
    q = 1 / Fraction(v)
    f = F32(1.0 / v)
    cands = [np.nextafter(f, F32(-np.inf)), f, np.nextafter(f, F32(np.inf))]
    return F32(min(cands, key=lambda c: (abs(Fraction(float(c)) - q), int(np.asarray(c).view(np.uint32)) & 1)))


def apply_model_emulated(model, x, **kw) -> dict:
    cfg = model.config
    return apply_emulated(model.params, np.asarray(model.norm_mean), np.asarray(model.norm_var),
                          n_d=cfg.n_d, n_steps=cfg.n_steps, gamma=cfg.gamma, x=x, **kw)
