// k2_kernel.cuh — K2: the whole TabNet forward (network.py:195-267) as ONE
// persistent sm_100a kernel, thread-per-row, for the single-pass tensor-core
// modes (TF32, BF16).
//
// Why a second design next to K1 (tc_kernel.cuh): K1 keeps each row's whole
// state (xn, prior, agg) in TMEM and splits a row over two threads, which
// leaves room for only 2 row tiles per SM; its per-tile chain of 29 GEMM ->
// epilogue hand-offs is then latency-bound (~70k cycles per tile pair, ~40%
// issue).  K2 moves the per-row state into registers (one thread owns one
// row: xn, agg, the GLU activations) and keeps only the MMA operands and the
// prior in TMEM, so 3-4 independent row groups (128 rows each) share an SM
// and hide each other's MMA/TMEM latency without any inter-group token.
//
//   TMEM (per row group, 128 lanes)        SMEM (per CTA)
//   [D accumulator  DW cols]               consts: affine, head
//   [A operand      KA cols]               ALL weight blocks, resident (one
//   [prior          F  cols]                 bulk load per CTA)
//                                          per warp: a 32 x F row tile staging
//   registers (per row): xn[F], agg[F],      x on the way in, each step's mask
//   the GLU activations g[H], logits[C]      and the importance on the way out
//
// GLU uses sigma(u) = (1 + tanh(u/2)) / 2 (one MUFU op per element): the
// packer folds the 1/2 (and the residual sqrt(1/2), network.py:131-137) into
// the weights and biases, so one GLU element is tanh + 2 FFMA:
//   out = lin'(1 + t) + sqrt(.5) prev,   lin' = (sqrt(.5)) u_lin / 2,  t = tanh(u_gate / 2)
// Biases ride in the GEMMs (a ones column in A, a bias row in B).
//
// Per-row arithmetic is identical for every row whatever the batch size, tile
// position, grid or group: the batch-invariance contract (network.py:11-14).
#pragma once
#include "tbn_rtc.h"
#include <cuda_bf16.h>
#include "tc_kernel.cuh"

namespace tbn {
namespace k2 {

using tc::chunked;
using tc::cmax;
using tc::kPrecBF16;
using tc::kPrecTF32;
using tc::kR;
using tc::rup;
using tc::tmem_load_n;
using tc::tmem_store_n;

constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int glu_chunk_width(int cw0, int cb, int ce) {
  for (int w = cw0; w >= 2; --w)
    if (w % 2 == 0 && cb % w == 0 && ce % w == 0) return w;
  return 2;
}
constexpr int pow2ceil(int v) { int p = 32; while (p < v) p <<= 1; return p; }

#ifndef TBN_K2_MAXNG
#define TBN_K2_MAXNG 4
#endif
// MAXNG_: row groups per CTA at most.  The throughput instances take 4 (as many
// as registers and TMEM allow); each shape also has a latency instance with 2
// (kernel_k2.cu), used when a CTA gets at most 2 row tiles: more registers per
// thread, xn in registers and (for HR) resident weights shorten the tile chain.
// The arithmetic is the same in both, so outputs are bitwise identical.
// SPLIT_ (with MAXNG_ = 1): the split latency instance, used when a CTA gets a
// single row tile.  One row group of 8 warps: warp q (the row's owner) does
// everything K2 does but compute only the d-half GLU columns [0, n_d); warp
// q + 4 (its helper, same TMEM lanes, same SMSP) computes the a-half [n_d, h)
// and writes the attentive A.  The two halves of a GLU layer run side by side
// instead of one after the other (a tile chain is latency-bound: one warp per
// SMSP); per-column arithmetic is unchanged, so outputs stay bitwise identical.
template <int F_, int ND_, int NA_, int S_, int C_, int PREC_, int MAXNG_ = TBN_K2_MAXNG, bool SPLIT_ = false>
struct Cfg {
  static constexpr int F = F_, ND = ND_, NA = NA_, S = S_, C = C_, PREC = PREC_;
  static constexpr bool SPLIT = SPLIT_;
  static_assert(!SPLIT || (MAXNG_ == 1 && ND % 2 == 0 && NA % 2 == 0), "split instance: one group, even halves");
  static_assert(PREC == kPrecTF32 || PREC == kPrecBF16 || PREC == tc::kPrecTF32x3, "K2 precision");
  static constexpr int H = ND + NA, N2 = 2 * H;
  // MMA N of the GLU GEMMs: 2h padded to the M=128 granule (B rows beyond 2h are 0)
  static constexpr int NP = rup(N2, 16);
  static constexpr bool X3 = (PREC == tc::kPrecTF32x3);   // 3xTF32: A and B split hi/lo, 3 MMAs
  static constexpr bool BF = (PREC == kPrecBF16);
  static constexpr int KG = BF ? 16 : 8;               // MMA K granule
  static constexpr int ESZ = BF ? 2 : 4;
  // A operand = [1, 1, data..., stale]: the two ones (written once per tile)
  // meet the bias hi/lo rows 0, 1 of every B block; data starts at element 2
  static constexpr int A0 = 2;
  static constexpr int K1 = rup(F + A0, KG);
  static constexpr int KHID = rup(H + A0, KG);
  static constexpr int KATT = rup(NA + A0, KG);
  static constexpr int FN = rup(F, 16);                // attentive N
  static constexpr int KA_EL = cmax(cmax(K1, KHID), KATT);
  static constexpr int KA = BF ? KA_EL / 2 : KA_EL;    // A operand TMEM columns
  static constexpr int DW = cmax(NP, FN);
  static constexpr int T_D = 0, T_A = DW, T_AL = T_A + KA, T_PR = T_AL + (X3 ? KA : 0), T_END = T_PR + F;
  static constexpr int TCG = rup(T_END, 32);           // TMEM columns per group
  static constexpr int NG_TMEM = 512 / TCG;
  // Register file: a row's live state is about 2F + H + 48 registers with xn
  // in registers (variant R), F + H + 48 with xn in shared memory (variant S).
  static constexpr int NG_R = cmin(MAXNG_, cmin(NG_TMEM, 65536 / (128 * (2 * F + H + 48))));
  static constexpr int NG_S = cmin(MAXNG_, cmin(NG_TMEM, 65536 / (128 * (F + H + 48))));
  // weight blocks (B operands, N x K K-major canonical)
  static constexpr int PARTS = X3 ? 2 : 1;            // hi [+ lo] B blocks
  static constexpr int B_SH1 = PARTS * NP * K1 * ESZ;
  static constexpr int B_HID = PARTS * NP * KHID * ESZ;
  static constexpr int B_ATT = PARTS * FN * KATT * ESZ;
  static constexpr int HBR = rup(B_HID, 128), ABR = rup(B_ATT, 128);
  // consts (floats): scale F | shift F | head_W ND*C | head_b C
  static constexpr int C_SCALE = 0, C_SHIFT = rup(F, 4), C_HW = C_SHIFT + rup(F, 4);
  static constexpr int C_HB = C_HW + rup(ND * C, 4), C_END = rup(C_HB + C, 4);
  static constexpr int CONST_BYTES = C_END * 4;
  // global image: [consts][sh1][sh2][fc1_0..S][fc2_0..S][att_1..S], 128-B aligned blocks
  static constexpr int O_SH1 = rup(CONST_BYTES, 128);
  static constexpr int O_SH2 = O_SH1 + rup(B_SH1, 128);
  static constexpr int O_FC1 = O_SH2 + HBR;
  static constexpr int O_FC2 = O_FC1 + (S + 1) * HBR;
  static constexpr int O_ATT = O_FC2 + (S + 1) * HBR;
  static constexpr int IMG_BYTES = O_ATT + S * ABR;
  static constexpr int STG = rup(32 * F * 4, 128);     // per-warp 32 x F row tile
  static constexpr int SMEM_MAX = 227 * 1024 - 512;
  // variant S (xn in SMEM, one more group): the fc1/fc2 blocks stream through a
  // CTA-wide ring shared by the groups when the whole image does not fit
  static constexpr int FIX_S = O_FC1 + S * ABR;        // consts, sh1, sh2, att resident
  static constexpr int STG_S = 2 * (NG_S * 4) * STG;
  static constexpr bool S_RES = IMG_BYTES + STG_S <= SMEM_MAX;
  static constexpr int S_SLOTS = cmin(6, (SMEM_MAX - FIX_S - STG_S) / HBR);
  static constexpr bool S_OK = NG_S > NG_R && (S_RES || S_SLOTS >= 3);
  static constexpr bool XS = S_OK;                     // xn in shared memory
  static constexpr int NG = XS ? NG_S : NG_R;
  // fc1/fc2 blocks resident, or streamed through the ring when the image does not fit
  static constexpr int STG_ALL = (XS ? 2 : 1) * (NG * 4) * STG;
  static constexpr bool RING = IMG_BYTES + STG_ALL > SMEM_MAX;
  // 4 slots (measured: 8 buys nothing and takes L1 away)
  static constexpr int NSLOT_FIT = RING ? cmin(4, (SMEM_MAX - FIX_S - STG_ALL) / HBR) : 0;
  static constexpr int NSLOT_SH = NSLOT_FIT >= 8 ? 8 : NSLOT_FIT >= 4 ? 4 : NSLOT_FIT >= 2 ? 2 : 0;  // power of 2
  static constexpr int NSLOT = NSLOT_SH;               // slots in SMEM
  static_assert(!RING || NSLOT >= 2, "not even a 2-slot weight ring fits");
  static_assert(NSLOT <= 16, "ring barriers");
  static constexpr int NB = 2 * (S + 1);               // ring blocks per tile: fc1_s, fc2_s
  static_assert(NG >= 1, "per-row state does not fit");
  static constexpr int TCOLS = pow2ceil(NG * TCG);
  static_assert(TCOLS <= 512, "TMEM");
  static_assert(NP <= 256 && FN <= 256, "MMA N > 256");
  static constexpr int THREADS = NG * 128 * (SPLIT ? 2 : 1);
  static constexpr int NW = NG * 4 * (SPLIT ? 2 : 1);
  static constexpr int BAR_THREADS = SPLIT ? 256 : 128;   // one group's named barrier
  // shared-memory plan: resident image (or its fixed part + att + ring) | staging | bars
  static constexpr int S_ATT = RING ? O_FC1 : O_ATT;   // where att_1 lives in SMEM
  static constexpr int OFF_RING = O_FC1 + S * ABR;
  static constexpr int RES_BYTES = RING ? OFF_RING + NSLOT * HBR : IMG_BYTES;
  static constexpr int OFF_STG = rup(RES_BYTES, 1024);
  static constexpr int OFF_XS = OFF_STG + NW * STG;    // variant S: per-warp xn tiles
  static constexpr int OFF_BAR = OFF_XS + (XS ? NW * STG : 0);
  static constexpr int OFF_RCP = OFF_BAR + 512;        // rcp_rn(k), k = 0..F (sparsemax tau)
  static constexpr int SMEM_BYTES = OFF_RCP + rup(4 * (F + 1), 128);
  static_assert(SMEM_BYTES <= 227 * 1024, "weights + staging exceed shared memory");
};

struct Params {
  const uint8_t* wimg;     // device image (layout above)
  float gamma;
};

struct Bars {
  uint64_t cfull;
  uint64_t dfull[4];       // per group: MMA chain complete
  uint64_t xfull[16];      // per warp: x row tile landed
  uint64_t rfull[16];      // ring slots (variant S, streamed fc1/fc2 blocks)
  uint32_t rcnt[16];       // shared ring slots: monotonic release counters
  uint32_t tmem_base;
};

__device__ __forceinline__ float tanh_approx(float x) {
#ifdef TBN_K2_FAKETANH      // dev experiment only: how much of the time is the MUFU pipe
  return fminf(fmaxf(x, -1.0f), 1.0f);
#elif defined(TBN_K2_FAKETANH2)   // dev experiment only: no MUFU, ~no issue cost
  return x * 0.25f;
#else
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// 1 + tanh(g) for a pair on the FMA/ALU pipes only (no MUFU), to take part of
// the GLU's sigmoid load off the MUFU pipe (FA4-style split):
//   1 + tanh(g) = 2 r,  r = 1 / (1 + 2^y),  y = -2 log2(e) g  (clamped to +-64)
//   2^y = 2^j p(f): j = round(y) by the 1.5*2^23 magic add, f = y - j in [-.5, .5],
//   p a degree-3 fit of 2^f (relative error 2.1e-4), 2^j added to the exponent bits;
//   r by two Newton steps from the integer-magic seed (relative error 6.6e-6).
// Overall within ~2.2e-4 relative of 1 + tanh, the class of tanh.approx.f32 (2^-11).
__device__ __forceinline__ float2 one_plus_tanh_fma(float2 g) {
  float2 y = __fmul2_rn(g, f2(-2.8853900817779268f, -2.8853900817779268f));
  y.x = fminf(fmaxf(y.x, -64.0f), 64.0f);
  y.y = fminf(fmaxf(y.y, -64.0f), 64.0f);
  const float2 t = __fadd2_rn(y, f2(12582912.0f, 12582912.0f));
  const float2 j = __fadd2_rn(t, f2(-12582912.0f, -12582912.0f));
  const float2 fr = __ffma2_rn(j, f2(-1.0f, -1.0f), y);
  float2 pp = __ffma2_rn(fr, f2(0.05484800413250923f, 0.05484800413250923f),
                         f2(0.24180661141872406f, 0.24180661141872406f));
  pp = __ffma2_rn(pp, fr, f2(0.6932482123374939f, 0.6932482123374939f));
  pp = __ffma2_rn(pp, fr, f2(0.9999886751174927f, 0.9999886751174927f));
  const float2 e = f2(__int_as_float(__float_as_int(pp.x) + (__float_as_int(t.x) << 23)),
                      __int_as_float(__float_as_int(pp.y) + (__float_as_int(t.y) << 23)));
  const float2 d = __fadd2_rn(e, f2(1.0f, 1.0f));
  const float2 nd = f2(-d.x, -d.y);
  float2 r = f2(__int_as_float(0x7EF311C3 - __float_as_int(d.x)), __int_as_float(0x7EF311C3 - __float_as_int(d.y)));
  r = __ffma2_rn(r, __ffma2_rn(nd, r, f2(1.0f, 1.0f)), r);
  r = __ffma2_rn(r, __ffma2_rn(nd, r, f2(1.0f, 1.0f)), r);
  return __fadd2_rn(r, r);
}
#ifndef TBN_K2_FMA_EVERY     // every Nth GLU pair takes the FMA-pipe sigmoid (0: none)
#define TBN_K2_FMA_EVERY 0
#endif

// A operand: L elements of v starting at element E (E, L even for bf16)
template <class CF, int E, int L, int M>
__device__ __forceinline__ void put_a(uint32_t tA, const float (&v)[M]) {
  if constexpr (CF::BF) {
    static_assert(E % 2 == 0 && L % 2 == 0, "bf16 A elements come in pairs");
    float pk[L / 2];
#pragma unroll
    for (int i = 0; i < L / 2; ++i) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);   // low = even
      pk[i] = *reinterpret_cast<const float*>(&b);
    }
    tmem_store_n<L / 2>(tA + E / 2, pk);
  } else {
    tmem_store_n<L>(tA + E, v);
    if constexpr (CF::X3) {
      // 3xTF32: the MMA reads fp32 as tf32 by truncation, so A_hi = v and
      // A_lo = v - trunc_tf32(v) (exact in fp32), stored KA columns further on
      float lo[L];
#pragma unroll
      for (int i = 0; i < L; ++i) lo[i] = v[i] - __uint_as_float(__float_as_uint(v[i]) & 0xFFFFE000u);
      tmem_store_n<L>(tA + CF::KA + E, lo);
    }
  }
}

template <class CF>
__global__ void __launch_bounds__(CF::THREADS, 1)
tabnet_rowthread(const Params p, const ForwardArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int F = CF::F, H = CF::H, ND = CF::ND, NA = CF::NA, S = CF::S, C = CF::C, NG = CF::NG;
  constexpr int NB = CF::NB, NSLOT = CF::NSLOT;
  const float* cst = reinterpret_cast<const float*>(smem);
  Bars* bars = reinterpret_cast<Bars*>(smem + CF::OFF_BAR);
  // warp index through a shuffle: provably warp-uniform, so the TMEM and SMEM
  // addresses derived from it live in uniform registers (no R2UR per tcgen05 op)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const bool helper = CF::SPLIT && warp >= 4;      // split instance: the a-half warp
  const int g = CF::SPLIT ? 0 : warp >> 2, q = warp & 3;
  const int t = q * 32 + lane;                      // row within the tile == TMEM lane
  const bool x_bulk_ok = ((reinterpret_cast<uintptr_t>(a.x) & 15u) == 0);
  // this CTA's rows: a contiguous block of R = ceil(rows / grid) rounded up to 4
  // rows (16-byte aligned row runs); its tiles are 128-row pieces of it, tile m
  // = g + NG * round.  Every SM gets the same row count, so the batch's last
  // partial tile per CTA has whole warps without rows, which skip their math.
  const int64_t rpc = (((a.rows + gridDim.x - 1) / gridDim.x) + 3) & ~(int64_t)3;
  const int64_t cta_r0 = (int64_t)blockIdx.x * rpc;
  const int64_t cta_end = cta_r0 + rpc < a.rows ? cta_r0 + rpc : a.rows;
  const int64_t tiles_cta = cta_end > cta_r0 ? (cta_end - cta_r0 + 127) / 128 : 0;
  const int64_t rounds = (tiles_cta + NG - 1) / NG;
  const uint32_t nblk = (uint32_t)(rounds * NB);    // ring blocks this CTA streams

  // ring block v (variant S): fc1_s / fc2_s of tile round v / NB, s = (v % NB) / 2
  auto ring_src = [&](uint32_t v) -> const uint8_t* {
    const uint32_t i = v % NB;
    return p.wimg + ((i & 1) ? CF::O_FC2 : CF::O_FC1) + (i >> 1) * CF::HBR;
  };
  // slot and phase parity of ring block v (v % NSLOT, use v / NSLOT);
  // (measured and dropped: per-group 2-slot rings, 8% slower at 262,144 rows)
  auto ring_slot = [&](uint32_t v) -> int { return NSLOT ? (int)(v % (NSLOT ? NSLOT : 1)) : 0; };
  auto ring_parity = [&](uint32_t v) -> uint32_t { return NSLOT ? (v / (NSLOT ? NSLOT : 1)) & 1u : 0u; };
  auto ring_load = [&](uint32_t v) {
    const int sl = ring_slot(v);
    ptx::mbar_arrive_expect_tx(&bars->rfull[sl], CF::B_HID);
    ptx::bulk_g2s(smem + CF::OFF_RING + sl * CF::HBR, ring_src(v), CF::B_HID, &bars->rfull[sl]);
  };

  if (threadIdx.x == 0) {
    ptx::mbar_init(&bars->cfull, 1);
    for (int i = 0; i < NG; ++i) ptx::mbar_init(&bars->dfull[i], 1);
    for (int i = 0; i < CF::NW; ++i) ptx::mbar_init(&bars->xfull[i], 1);
    for (int i = 0; i < CF::NSLOT; ++i) {
      ptx::mbar_init(&bars->rfull[i], 1);
      bars->rcnt[i] = 0;
    }
    ptx::fence_mbar_init();
    constexpr int CH = 32768;
    if constexpr (!CF::RING) {
      ptx::mbar_arrive_expect_tx(&bars->cfull, CF::IMG_BYTES);
      for (int o = 0; o < CF::IMG_BYTES; o += CH)
        ptx::bulk_g2s(smem + o, p.wimg + o, (uint32_t)(CF::IMG_BYTES - o < CH ? CF::IMG_BYTES - o : CH),
                      &bars->cfull);
    } else {
      // consts + sh1 + sh2 (image prefix), then the attentive blocks behind them
      constexpr int ATT_BYTES = S * CF::ABR;
      ptx::mbar_arrive_expect_tx(&bars->cfull, CF::O_FC1 + ATT_BYTES);
      for (int o = 0; o < CF::O_FC1; o += CH)
        ptx::bulk_g2s(smem + o, p.wimg + o, (uint32_t)(CF::O_FC1 - o < CH ? CF::O_FC1 - o : CH), &bars->cfull);
      for (int o = 0; o < ATT_BYTES; o += CH)
        ptx::bulk_g2s(smem + CF::S_ATT + o, p.wimg + CF::O_ATT + o,
                      (uint32_t)(ATT_BYTES - o < CH ? ATT_BYTES - o : CH), &bars->cfull);
      for (uint32_t v = 0; v < (uint32_t)NSLOT && v < nblk; ++v) ring_load(v);
    }
  }
  if (warp == 0) ptx::tmem_alloc<CF::TCOLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tg = bars->tmem_base + (uint32_t)(g * CF::TCG) + ((uint32_t)(q * 32) << 16);
  const uint32_t tD = tg + CF::T_D, tA = tg + CF::T_A, tPR = tg + CF::T_PR;
  float* stg = reinterpret_cast<float*>(smem + CF::OFF_STG + warp * CF::STG);
  // where x lands and xn lives: its own per-warp tile (variant S) or the staging tile
  float* xst = CF::XS ? reinterpret_cast<float*>(smem + CF::OFF_XS + warp * CF::STG) : stg;
  float* const my_stg = stg + lane * F;             // this thread's row in the staging tile
  float* const my_xs = xst + lane * F;
  const uint32_t bar_id = 1 + g;                    // A ready (before the MMA issue)
  uint32_t dphase = 0, xphase = 0;

  // stage this warp's rows [r0w, r0w + nw) of x into xst: the TMA bulk part is
  // issued early (issue_x), the unaligned tail is loaded by the lanes (wait_x)
  auto x_bulk_elems = [&](int nw) -> int { return x_bulk_ok ? ((nw * F * 4) & ~15) / 4 : 0; };
  auto issue_x = [&](int64_t r0w, int nw) {
    const int nb = x_bulk_elems(nw);
    if (lane == 0) {
      if (nb > 0) {
        ptx::mbar_arrive_expect_tx(&bars->xfull[warp], (uint32_t)nb * 4u);
        ptx::bulk_g2s(xst, a.x + r0w * F, (uint32_t)nb * 4u, &bars->xfull[warp]);
      } else {
        ptx::mbar_arrive(&bars->xfull[warp]);
      }
    }
  };
  auto wait_x = [&](int64_t r0w, int nw) {
    const int ne = nw * F, nb = x_bulk_elems(nw);
    for (int e = nb + lane; e < 32 * F; e += 32) xst[e] = e < ne ? __ldg(a.x + r0w * F + e) : 0.0f;
    ptx::mbar_wait(&bars->xfull[warp], xphase);
    xphase ^= 1;
    __syncwarp();
  };
  // rows of this warp in the tile of group-local index m (0 when past the end)
  auto warp_rows = [&](int64_t m, int64_t& r0w) -> int {
    const int64_t r0 = cta_r0 + m * 128;
    r0w = r0 + q * 32;
    const int64_t n = cta_end - r0w;
    return m >= tiles_cta || n <= 0 ? 0 : (n > 32 ? 32 : (int)n);
  };
  // stg (32 x F, this warp's rows) -> dst rows [0, nw): bulk store when aligned
  auto flush = [&](float* dst, int nw) {
    const int ne = nw * F;
    const bool al = ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0);
    const int nb = al ? ((ne * 4) & ~15) / 4 : 0;
    ptx::fence_async_shared();
    __syncwarp();
    if (lane == 0 && nb > 0) {
      ptx::bulk_s2g(dst, stg, (uint32_t)nb * 4u);
      ptx::bulk_commit();
    }
    for (int e = nb + lane; e < ne; e += 32) dst[e] = stg[e];
    __syncwarp();
  };
  auto claim_stg = [&]() {      // the previous bulk store has finished reading stg
    if (lane == 0) ptx::bulk_wait_read0();
    __syncwarp();
  };
  // ring block v no longer needed by this group: the last of the NG groups to
  // release it refills its slot with block v + NSLOT.  Counters are monotonic:
  // use u = v / NSLOT of a slot completes at arrival (u + 1) * NG.
  auto ring_release = [&](uint32_t v) {
    const uint32_t sl = (uint32_t)ring_slot(v);
    const uint32_t old = atomicAdd(&bars->rcnt[sl], 1u);
    if (old == (v / (NSLOT ? NSLOT : 1)) * NG + NG - 1 && v + NSLOT < nblk) ring_load(v + NSLOT);
  };

  // Programmatic dependent launch: everything before the wait (barriers, TMEM,
  // the weight-image TMA, an L2 prefetch of this warp's first x rows, the
  // reciprocal table) overlaps the tail of the previous kernel on the stream;
  // from the wait on this grid reads and writes data that kernel may produce
  // or consume (x, the batch-statistics affine, the outputs).  The next launch
  // may start its own prologue as SMs free up.  On a cold start the weights and
  // the first x rows are in flight together (the weights' landing is awaited
  // after the x tile is requested).
  {   // warm L2 with this warp's first x rows (a hint; L2 is where the previous
      // kernel's writes land, so a prefetch ahead of the wait cannot read stale data)
    int64_t r0p;
    const int nwp = warp_rows(g, r0p);
    if (lane == 0 && nwp > 0 && x_bulk_ok && !helper) {
      const uint32_t bytes = (uint32_t)((nwp * F * 4) & ~15);
      if (bytes) ptx::bulk_prefetch_l2(a.x + r0p * F, bytes);
    }
  }
  float* const rcp_tab = reinterpret_cast<float*>(smem + CF::OFF_RCP);
  for (int i = threadIdx.x; i <= F; i += blockDim.x) rcp_tab[i] = i ? __frcp_rn((float)i) : 0.0f;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  {   // this warp's first x tile
    int64_t r0w;
    const int nw0 = warp_rows(g, r0w);
    if (nw0 > 0 && !helper) issue_x(r0w, nw0);
  }
  ptx::mbar_wait(&bars->cfull, 0);                   // the weights have landed
  if (a.scale) {     // batch-statistics control: override the affine in this CTA's copy
    float* cw = reinterpret_cast<float*>(smem);
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      cw[CF::C_SCALE + f] = a.scale[f];
      cw[CF::C_SHIFT + f] = a.shift[f];
    }
  }
  __syncthreads();

  const uint32_t wbase = ptx::smem_u32(smem);
  // One GEMM: A (this group's TMEM) x B (SMEM block at byte offset bo, or ring
  // block rv).  The group meets at its barrier, warp 0 of the group issues the
  // chain and commits it; `post` overlaps the MMA; then everyone waits for D.
  int jt = 0;                                    // trace: GEMM counter
  int64_t ring_pending = -1;                     // ring block awaiting release (same in every warp)
  const bool tr = (q == 0 && lane == 0 && !helper);
  auto gemm = [&](int kind, uint32_t bo, int64_t rv, auto&& post) {
    if (tr) TBN_TRACE(g * 4000 + 4 * jt);
    // the issuing warp rotates over the group's four warps (measured 1.3%
    // faster at HR @ 65,536 than always warp 0: the issue work is spread)
    const int iq = jt & 3;
    if constexpr (CF::RING) {
      // the issuing warp checks its ring block while the other warps finish
      // writing A (off the barrier -> MMA critical path)
      if (rv >= 0) {
        const uint32_t v = (uint32_t)rv;
        if (q == iq && !helper) ptx::mbar_wait(&bars->rfull[ring_slot(v)], ring_parity(v));
        bo = CF::OFF_RING + ring_slot(v) * CF::HBR;
      }
    }
    __syncwarp();                                  // bar.sync / tcgen05 .aligned: converged warp
    ptx::tmem_st_wait();
    ptx::tc_fence_before();
#ifndef TBN_K2_NOBAR          // dev experiment only (with TBN_K2_NOMMA): the barrier's cost
    ptx::named_bar_sync(bar_id, CF::BAR_THREADS);
#endif
    if (tr) TBN_TRACE(g * 4000 + 4 * jt + 1);
    if (q == iq && !helper) {
      ptx::tc_fence_after();
      const uint32_t tAL = tA + CF::KA;              // A_lo (3xTF32 only)
#ifndef TBN_K2_NOMMA          // dev experiment only: the tensor core's share of the chain
      if (kind == 0) tc::issue_gemm<CF, CF::K1, CF::NP>(tD, tA, tAL, wbase + bo);
      else if (kind == 1) tc::issue_gemm<CF, CF::KHID, CF::NP>(tD, tA, tAL, wbase + bo);
      else tc::issue_gemm<CF, CF::KATT, CF::FN>(tD, tA, tAL, wbase + bo);
#endif
      ptx::mma_commit(&bars->dfull[g]);
      if constexpr (CF::RING) {
        // the previous GEMM's ring block: its MMAs completed before this chain
        // was issued, so release it now, off the critical path
        if (ring_pending >= 0 && lane == 0) ring_release((uint32_t)ring_pending);
      }
    }
    ring_pending = -1;         // every warp tracks the same block sequence
    if (tr) TBN_TRACE(g * 4000 + 4 * jt + 2);
    post();
    // every warp parks on the commit barrier (suspend-time hint: no spinning)
    ptx::mbar_wait_sleep(&bars->dfull[g], dphase);
    dphase ^= 1;
    ptx::tc_fence_after();
    if constexpr (CF::RING) {
      if (rv >= 0) ring_pending = rv;            // released under the next MMA chain
    }
    if (tr) TBN_TRACE(g * 4000 + 4 * jt + 3);
    ++jt;
  };
  auto nopost = [] {};

  float xnr[CF::XS ? 1 : F], agg[F], gv[H], lacc[C];
  auto xn_at = [&](int f) -> float {
    if constexpr (CF::XS) return my_xs[f];
    else return xnr[f];
  };

  // GLU block over D = [lin' | gate'] (H + H columns): gv <- lin'(1+t) [+ R gv]
  // for the output columns [CB, CE) (the whole block but where the reference's
  // result is unused, Appendix A of SURVEY.md: step 0's d half, step S's a half)
  auto glu_range = [&](bool residual, auto cb, auto ce) {
    constexpr int CB = decltype(cb)::value, CE = decltype(ce)::value;
    constexpr int CW0 = CF::XS ? (H < 8 ? H : 8) : (H < 16 ? H : 16);   // 16 measured no faster
    // the widest even chunk up to CW0 that tiles [CB, CE) (any h, pruned ranges)
    constexpr int CW = glu_chunk_width(CW0, CB, CE);
    static_assert(CB % CW == 0 && CE % CW == 0, "GLU chunking");
    float lin[CW], gate[CW];
    tmem_load_n<CW>(tD + CB, lin);
    tmem_load_n<CW>(tD + H + CB, gate);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int c0 = CB; c0 < CE; c0 += CW) {
      float ln2[CW], gt2[CW];
      if (c0 + CW < CE) {          // next chunk in flight while this one computes
        tmem_load_n<CW>(tD + c0 + CW, ln2);
        tmem_load_n<CW>(tD + H + c0 + CW, gt2);
      }
#pragma unroll
      for (int i = 0; i < CW; i += 2) {
        float2 o;
        if constexpr (CF::X3) {
          // fp32-faithful sigmoid (as K1): gate columns carry -log2(e), so
          // e = 2^gate' = exp(-u); one reciprocal per pair: q = 1/(d0 d1)
          const float a0 = fminf(gate[i], 63.0f), a1 = fminf(gate[i + 1], 63.0f);
          const float2 d = __fadd2_rn(f2(tc::ex2_approx(a0), tc::ex2_approx(a1)), f2(1.0f, 1.0f));
          const float qq = tc::rcp_approx(d.x * d.y);
          const float2 sg = __fmul2_rn(f2(d.y, d.x), f2(qq, qq));
          const float2 l = f2(lin[i], lin[i + 1]);
          o = residual ? __ffma2_rn(l, sg, __fmul2_rn(f2(gv[c0 + i], gv[c0 + i + 1]), f2(kR, kR)))
                       : __fmul2_rn(l, sg);
        } else if (TBN_K2_FMA_EVERY > 0 && ((c0 + i) / 2) % (TBN_K2_FMA_EVERY > 0 ? TBN_K2_FMA_EVERY : 1) ==
                                              (TBN_K2_FMA_EVERY > 0 ? TBN_K2_FMA_EVERY : 1) - 1) {
          // o = lin'(1 + t) [+ sqrt(.5) prev] with 1 + t off the MUFU pipe
          const float2 opt = one_plus_tanh_fma(f2(gate[i], gate[i + 1]));
          const float2 l = f2(lin[i], lin[i + 1]);
          o = residual ? __ffma2_rn(l, opt, __fmul2_rn(f2(gv[c0 + i], gv[c0 + i + 1]), f2(kR, kR)))
                       : __fmul2_rn(l, opt);
        } else {
          const float2 th = f2(tanh_approx(gate[i]), tanh_approx(gate[i + 1]));
          const float2 l = f2(lin[i], lin[i + 1]);
          float2 w = l;
          if (residual) w = __ffma2_rn(f2(gv[c0 + i], gv[c0 + i + 1]), f2(kR, kR), l);
          o = __ffma2_rn(l, th, w);
        }
        gv[c0 + i] = o.x;
        gv[c0 + i + 1] = o.y;
      }
      if (c0 + CW < CE) {
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < CW; ++i) { lin[i] = ln2[i]; gate[i] = gt2[i]; }
      }
    }
  };
  // the owner's GLU columns: all h, or the d-half [0, n_d) in the split instance
  constexpr int GE = CF::SPLIT ? ND : H;
  auto glu = [&](bool residual) { glu_range(residual, std::integral_constant<int, 0>{}, std::integral_constant<int, GE>{}); };
  auto store_g = [&]() { put_a<CF, CF::A0, GE>(tA, gv); };

#ifdef TBN_K2_STAGGER      // dev experiment: de-phase the groups' chains
  {
    const long long t0 = clock64();
#if TBN_K2_STAGGER_MODE == 1
    const long long dly = (long long)g * (TBN_K2_STAGGER / 2);
#else
    const long long dly = (g & 1) ? TBN_K2_STAGGER : 0;
#endif
    while (clock64() - t0 < dly) { }
    __syncwarp();
  }
#endif
  for (int64_t k = 0; k < rounds; ++k) {
    const int64_t m = g + (int64_t)NG * k;
    if (m >= tiles_cta) {
      // no tile for this group in the last round: release its ring blocks
      if constexpr (CF::RING) {
        if (tr) {
          if (ring_pending >= 0) ring_release((uint32_t)ring_pending);
          ring_pending = -1;
          for (uint32_t i = 0; i < (uint32_t)NB; ++i) {
            const uint32_t v = (uint32_t)(k * NB) + i;
            ptx::mbar_wait(&bars->rfull[ring_slot(v)], ring_parity(v));
            ring_release(v);
          }
        }
      }
      break;
    }
    const int64_t r0 = cta_r0 + m * 128;
    const int nrows = (int)(cta_end - r0 < 128 ? cta_end - r0 : 128);
    const int nw = nrows - q * 32 < 0 ? 0 : (nrows - q * 32 > 32 ? 32 : nrows - q * 32);
    const bool valid = lane < nw;
    const int64_t row = r0 + t;
    const int64_t r0w = r0 + q * 32;
    const int64_t rv0 = CF::RING ? k * NB : -1;     // this tile's first ring block

    if (nw == 0) {
      // no rows for this warp (only in a CTA's last, partial tile; warp 0 of the
      // group always has rows and issues): keep the group's barrier/MMA protocol
      // — the same GEMM sequence as below — and skip all the math
      auto skel = [&](int s) {
        gemm(0, CF::O_SH1, -1, nopost);
        gemm(1, CF::O_SH2, -1, nopost);
        gemm(1, CF::O_FC1 + (uint32_t)s * CF::HBR, CF::RING ? rv0 + 2 * s : -1, nopost);
        gemm(1, CF::O_FC2 + (uint32_t)s * CF::HBR, CF::RING ? rv0 + 2 * s + 1 : -1, nopost);
      };
      skel(0);
      for (int s = 1; s <= S; ++s) {
        gemm(2, CF::S_ATT + (uint32_t)(s - 1) * CF::ABR, -1, nopost);
        skel(s);
      }
      continue;
    }
    if constexpr (CF::SPLIT) {
      if (helper) {
        // split instance, warp q + 4: the a-half [n_d, h) of every GLU layer and
        // the attentive A (a = f[:, n_d:], network.py:233), same GEMM sequence
        auto hglu = [&](bool residual) {
          glu_range(residual, std::integral_constant<int, ND>{}, std::integral_constant<int, H>{});
        };
        auto hstore = [&](auto e0) {
          float av[NA];
#pragma unroll
          for (int e = 0; e < NA; ++e) av[e] = gv[ND + e];
          put_a<CF, decltype(e0)::value, NA>(tA, av);
        };
        auto htransform = [&](int s) {
          const std::integral_constant<int, CF::A0 + ND> at_a;
          gemm(0, CF::O_SH1, -1, nopost);
          hglu(false);
          hstore(at_a);
          gemm(1, CF::O_SH2, -1, nopost);
          hglu(true);
          hstore(at_a);
          gemm(1, CF::O_FC1 + (uint32_t)s * CF::HBR, -1, nopost);
          hglu(true);
          hstore(at_a);
          gemm(1, CF::O_FC2 + (uint32_t)s * CF::HBR, -1, nopost);
          if (s != S) hglu(true);          // step S's a-half is unused
        };
        htransform(0);
        for (int s = 1; s <= S; ++s) {
          hstore(std::integral_constant<int, CF::A0>{});
          gemm(2, CF::S_ATT + (uint32_t)(s - 1) * CF::ABR, -1, nopost);
          htransform(s);
        }
        continue;
      }
    }

    // ---- x -> xn (network.py:118-120), prior = 1, agg = 0 ----
    if (tr) TBN_TRACE(g * 4000 + 3000 + 8 * (int)k);
    if (k > 0) {                  // (round 0's x was issued in the prologue)
      claim_stg();
      ptx::fence_async_shared();
      __syncwarp();
      if (nw > 0) issue_x(r0w, nw);
    }
    if (nw > 0) wait_x(r0w, nw);
    {   // warm L2 with this warp's rows of the group's next tile
      int64_t r0n;
      const int nwn = warp_rows(m + NG, r0n);
      if (lane == 0 && nwn > 0 && x_bulk_ok) {
        const uint32_t bytes = (uint32_t)((nwn * F * 4) & ~15);
        if (bytes) ptx::bulk_prefetch_l2(a.x + r0n * F, bytes);
      }
    }
    if (tr) TBN_TRACE(g * 4000 + 3001 + 8 * (int)k);
    {
      int bad = 0;
      float xv[F];
#pragma unroll
      for (int f = 0; f < F; ++f) {
        xv[f] = nw > 0 ? my_xs[f] : 0.0f;
        bad |= !isfinite(xv[f]);
        agg[f] = 0.0f;
      }
      if (!a.normalized) {        // (x - mean) * rsqrt(var + eps), pairwise
#pragma unroll
        for (int f = 0; f + 1 < F; f += 2) {
          const float2 v = __fmul2_rn(__fadd2_rn(f2(xv[f], xv[f + 1]),
                                                 f2(-cst[CF::C_SHIFT + f], -cst[CF::C_SHIFT + f + 1])),
                                      f2(cst[CF::C_SCALE + f], cst[CF::C_SCALE + f + 1]));
          xv[f] = v.x;
          xv[f + 1] = v.y;
        }
        if constexpr (F % 2) xv[F - 1] = (xv[F - 1] - cst[CF::C_SHIFT + F - 1]) * cst[CF::C_SCALE + F - 1];
      }
      if (valid && bad && a.err_flag) raise_flag(a.err_flag);
      __syncwarp();
#pragma unroll
      for (int f = 0; f < F; ++f) {
        if constexpr (CF::XS) my_xs[f] = xv[f];
        else xnr[f] = xv[f];
      }
      float one[F];
#pragma unroll
      for (int f = 0; f < F; ++f) one[f] = 1.0f;
      tmem_store_n<F>(tPR, one);
      // the whole A row once per tile: the ones, xn, and zeros over every
      // GEMM's padded K range (stale A elements must be finite: B rows are 0 there)
      float av[CF::KA_EL];
#pragma unroll
      for (int e = 0; e < CF::KA_EL; ++e) av[e] = e < CF::A0 ? 1.0f : (e - CF::A0 < F ? xv[e - CF::A0] : 0.0f);
      put_a<CF, 0, CF::KA_EL>(tA, av);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) lacc[c] = 0.0f;
    bool all_eta_zero = true;

    // feature transformer (network.py:124-141)
    auto transform = [&](int s, auto&& post_first) {
      const uint32_t o1 = CF::O_FC1 + (uint32_t)s * CF::HBR;
      const uint32_t o2 = CF::O_FC2 + (uint32_t)s * CF::HBR;
      gemm(0, CF::O_SH1, -1, post_first);
      glu(false);
      store_g();
      gemm(1, CF::O_SH2, -1, nopost);
      glu(true);
      store_g();
      gemm(1, o1, CF::RING ? rv0 + 2 * s : -1, nopost);
      glu(true);
      store_g();
      gemm(1, o2, CF::RING ? rv0 + 2 * s + 1 : -1, nopost);
#ifndef TBN_K2_NOPRUNE     // the unused halves are skipped: +0.7%
      if constexpr (CF::SPLIT) { if (s != 0) glu(true); }    // (the helper: the a-half)
      else if constexpr (ND % 2 != 0) glu(true);     // (pairs would straddle the d/a boundary)
      else if (s == 0) glu_range(true, std::integral_constant<int, ND>{}, std::integral_constant<int, H>{});
      else if (s == S) glu_range(true, std::integral_constant<int, 0>{}, std::integral_constant<int, ND>{});
      else glu(true);
#else
      glu(true);
#endif
    };
    // d = relu(f[:, :n_d]); eta = sum d; logits accumulate (the head is linear,
    // network.py:244, :253)
    auto step_eta = [&]() -> float {
      float e0 = 0.0f, e1 = 0.0f;
#pragma unroll
      for (int i = 0; i < ND; ++i) {
        const float d = fmaxf(gv[i], 0.0f);
        if constexpr (C % 2 == 0) {
#pragma unroll
          for (int c = 0; c < C; c += 2) {
            const float2 v = __ffma2_rn(f2(d, d), f2(cst[CF::C_HW + i * C + c], cst[CF::C_HW + i * C + c + 1]),
                                        f2(lacc[c], lacc[c + 1]));
            lacc[c] = v.x;
            lacc[c + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) lacc[c] = fmaf(d, cst[CF::C_HW + i * C + c], lacc[c]);
        }
        if (i & 1) e1 += d; else e0 += d;
      }
      return e0 + e1;
    };
    // agg += eta * m (network.py:245) from the staged mask; while every eta so
    // far is 0 agg holds sum_s m instead, which is exactly the importance
    // fallback's numerator (network.py:259-261); the first eta > 0 resets it.
    auto agg_apply = [&](float eta) {
      const bool reset = all_eta_zero && eta > 0.0f;
      const float w = all_eta_zero ? (eta > 0.0f ? eta : 1.0f) : eta;
      all_eta_zero = all_eta_zero && !(eta > 0.0f);
      if (reset) {              // rare: only rows whose earlier steps all had eta == 0
#pragma unroll
        for (int f = 0; f < F; ++f) agg[f] = 0.0f;
      }
#pragma unroll
      for (int f = 0; f < F; ++f) agg[f] = fmaf(w, my_stg[f], agg[f]);
      __syncwarp();
    };

    transform(0, nopost);                                        // network.py:226-227
    float eta_prev = 0.0f;
    for (int s = 1; s <= S; ++s) {
      // A <- [1, 1, a = f[:, n_d:]]; under the attentive MMA: the previous
      // step's d/eta/logits and agg update
      if constexpr (CF::SPLIT) {
        if (s > 1) eta_prev = step_eta();         // (the helper writes the attentive A)
      } else {
        float av[NA];
#pragma unroll
        for (int e = 0; e < NA; ++e) av[e] = gv[ND + e];
        if (s > 1) eta_prev = step_eta();
        put_a<CF, CF::A0, NA>(tA, av);
      }
      gemm(2, CF::S_ATT + (uint32_t)(s - 1) * CF::ABR, -1, [&] {
        if (s > 1) agg_apply(eta_prev);
      });
      // attentive transformer + sparsemax (network.py:233-238, sparsemax.py:13-41)
      float z[F];
      {
        float pr[F];
        tmem_load_n<F>(tD, z);
        tmem_load_n<F>(tPR, pr);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i + 1 < F; i += 2) {                       // bias already in D
          const float2 v = __fmul2_rn(f2(pr[i], pr[i + 1]), f2(z[i], z[i + 1]));
          z[i] = v.x;
          z[i + 1] = v.y;
        }
        if constexpr (F % 2) z[F - 1] = pr[F - 1] * z[F - 1];
      }
      float zmax, tau;
      if (tr) TBN_TRACE(g * 4000 + 3500 + 4 * s);
      {
        float m0 = -INFINITY, m1 = -INFINITY;
        float2 s2 = f2(0.0f, 0.0f);
#pragma unroll
        for (int i = 0; i + 1 < F; i += 2) {
          m0 = fmaxf(m0, z[i]);
          m1 = fmaxf(m1, z[i + 1]);
          s2 = __fadd2_rn(s2, f2(z[i], z[i + 1]));
        }
        if constexpr (F % 2) {
          m0 = fmaxf(m0, z[F - 1]);
          s2.x += z[F - 1];
        }
        zmax = fmaxf(m0, m1);
        const float zsum = s2.x + s2.y;
#pragma unroll
        for (int i = 0; i + 1 < F; i += 2) {                        // sparsemax.py:32
          const float2 v = __fadd2_rn(f2(z[i], z[i + 1]), f2(-zmax, -zmax));
          z[i] = v.x;
          z[i + 1] = v.y;
        }
        if constexpr (F % 2) z[F - 1] -= zmax;
        // tau: Michelot's fixed point tau <- (sum_{z>tau} z - 1)/|{z > tau}|, monotone
        // from a lower bound; its support equals the reference's sort/cumsum/count
        // k (sparsemax.py:33-39).  Start: max(-1, (sum z - 1)/F) nudged down 2^-20.
        const float bound = (zsum - (float)F * zmax - 1.0f) * (1.0f / (float)F);
        tau = fmaxf(-1.0f, bound - 9.5367431640625e-07f * fmaxf(1.0f, fabsf(bound)));
        float cnt_prev = (float)(F + 1);
        for (int it = 0; it <= F; ++it) {
          float2 sa = f2(0.0f, 0.0f), ca = f2(0.0f, 0.0f), sb = f2(0.0f, 0.0f), cb = f2(0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i + 1 < F; i += 2) {
            const float2 mk = f2(z[i] > tau ? 1.0f : 0.0f, z[i + 1] > tau ? 1.0f : 0.0f);
            if ((i / 2) % 2 == 0) {
              sa = __ffma2_rn(mk, f2(z[i], z[i + 1]), sa);
              ca = __fadd2_rn(ca, mk);
            } else {
              sb = __ffma2_rn(mk, f2(z[i], z[i + 1]), sb);
              cb = __fadd2_rn(cb, mk);
            }
          }
          const float2 s2 = __fadd2_rn(sa, sb), c2 = __fadd2_rn(ca, cb);
          float sm = s2.x + s2.y, cn = c2.x + c2.y;
          if constexpr (F % 2) {
            const float mk = z[F - 1] > tau ? 1.0f : 0.0f;
            sm = fmaf(mk, z[F - 1], sm);
            cn += mk;
          }
#ifdef TBN_K2_FAKEMICH      // dev experiment only: the cost of the Michelot passes
          if (it >= 1) break;
#endif
          if (cn >= cnt_prev) break;
          cnt_prev = cn;
          // sparsemax.py:39: (sum - 1) / k as (sum - 1) * rcp_rn(k), k from the
          // table (one rounding per operation: the emulation oracle repeats it)
          tau = (sm - 1.0f) * rcp_tab[(int)cn];
        }
        // the lanes left the loop at different passes: reconverge before the
        // warp-collective (.aligned) tcgen05 loads/stores and named barriers
        __syncwarp();
      }
      // mask, prior update, x*mask -> A (elements 2 ..); mask -> staging
      // (network.py:236-238, :246), in 16-feature chunks
      if (tr) TBN_TRACE(g * 4000 + 3501 + 4 * s);
      claim_stg();
      {
        const float2 gm2 = f2(p.gamma, p.gamma), nt2 = f2(-tau, -tau);
        chunked<(F + 1) / 2 * 2, 16>([&](auto o, auto l) {
          constexpr int O = decltype(o)::value, L = decltype(l)::value;
          constexpr int LF = (O + L <= F) ? L : (O < F ? F - O : 0);   // features in this chunk
          float pr[LF > 0 ? LF : 1], av[L];
          if constexpr (LF > 0) {
            tmem_load_n<LF>(tPR + O, pr);
            ptx::tmem_ld_wait();
          }
#pragma unroll
          for (int i = 0; i < L; i += 2) {
            const int f = O + i;
            if (f + 1 < F) {
              const float2 d = __fadd2_rn(f2(z[f], z[f + 1]), nt2);
              const float2 mk = f2(fmaxf(d.x, 0.0f), fmaxf(d.y, 0.0f));      // sparsemax.py:40
              const float2 np = __fmul2_rn(f2(pr[i], pr[i + 1]), __fadd2_rn(gm2, f2(-mk.x, -mk.y)));  // :237
              const float2 xm = __fmul2_rn(mk, f2(xn_at(f), xn_at(f + 1)));    // network.py:238
              pr[i] = np.x; pr[i + 1] = np.y;
              av[i] = xm.x; av[i + 1] = xm.y;
              my_stg[f] = mk.x;
              my_stg[f + 1] = mk.y;
            } else {
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int fu = f + u;
                if (fu < F) {
                  const float mk = fmaxf(z[fu] - tau, 0.0f);
                  pr[i + u] = pr[i + u] * (p.gamma - mk);
                  av[i + u] = mk * xn_at(fu);
                  my_stg[fu] = mk;
                } else {
                  av[i + u] = 0.0f;                                       // odd F: pad element
                }
              }
            }
          }
          if constexpr (LF > 0) tmem_store_n<LF>(tPR + O, pr);
          put_a<CF, O + CF::A0, L>(tA, av);
        });
      }
      // masks[s-1] of this warp's rows leave while the shared1 MMA runs
      transform(s, [&] {
        if (a.masks && nw > 0) flush(a.masks + ((int64_t)(s - 1) * a.rows + r0w) * F, nw);
      });
    }
    agg_apply(step_eta());                       // the last step (no attentive GEMM follows)
    if (tr) TBN_TRACE(g * 4000 + 3002 + 8 * (int)k);

    // ---- head + softmax + argmax (network.py:253-256, :279); importance =
    // agg / sum(agg) or mean_s(masks) (network.py:258-261) ----
    {
      float lg[C], lmax = -INFINITY;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        lg[c] = lacc[c] + cst[CF::C_HB + c];
        lmax = fmaxf(lmax, lg[c]);
      }
      float ex[C], es = 0.0f;
#pragma unroll
      for (int c = 0; c < C; ++c) { ex[c] = expf(lg[c] - lmax); es += ex[c]; }
      if (valid) {
        int best = 0;
        float bv = -1.0f;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float pv = ex[c] / es;
          if (a.logits) a.logits[row * C + c] = lg[c];
          if (a.probs) a.probs[row * C + c] = pv;
          if (pv > bv) { bv = pv; best = c; }
        }
        if (a.pred) a.pred[row] = best;
      }
      float t0 = 0.0f, t1 = 0.0f;
#pragma unroll
      for (int f = 0; f < F; ++f) { if (f & 1) t1 += agg[f]; else t0 += agg[f]; }
      const float div = all_eta_zero ? (float)S : (t0 + t1);
      const float rdiv = __frcp_rn(div);
      claim_stg();
#pragma unroll
      for (int f = 0; f < F; ++f) my_stg[f] = agg[f] * rdiv;
      if (a.importance && nw > 0) flush(a.importance + r0w * F, nw);
    }
    if (tr) TBN_TRACE(g * 4000 + 3003 + 8 * (int)k);
  }
  if constexpr (CF::RING) {
    if (tr && ring_pending >= 0) ring_release((uint32_t)ring_pending);
  }
  if (lane == 0) ptx::bulk_wait0();

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<CF::TCOLS>(bars->tmem_base);
}

}  // namespace k2
}  // namespace tbn
