// k3x_kernel.cuh — K3X: the wide-model forward (F = 512, h = 128: BASELINE
// config 5; network.py:195-267) in the fp32-faithful 3xTF32 mode, so that the
// parity mode (precision "tf32x3", the Python default) of wide models runs on
// the tensor cores instead of the fp32 CUDA-core kernel.
//
// Same skeleton as K3 (k3_kernel.cuh): one 128-row tile per CTA, 16 warps,
// warp w owns TMEM lane quarter q = w % 4 and slice c = w / 4 (features
// [128c, 128c+128), GLU outputs [32c, 32c+32)); every B operand streams
// through a TMA ring in K-chunks; the 4 slice threads of a row combine their
// sparsemax partials through SMEM.  What changes for 3xTF32:
//
//  * operands are tf32 hi/lo pairs: B split by the packer (hi = rna(w),
//    lo = rna(w - hi)), A split on the fly (hi = v rounded to tf32, lo = v - hi); 3 MMAs per K-step (hi.hi, lo.hi, hi.lo);
//  * TMEM: the attentive D = z takes all 512 columns; the transforms use
//    A hi [0,128) | A lo [128,256) | D [256,512), so the hidden GEMMs (K = 128)
//    take A from TMEM and shared1 (K = 512) runs as 4 K-chunks of 128, slice k
//    writing chunk k into the A columns once chunk k-1's MMAs completed;
//  * the attentive A (a = f[:, n_d:], K = 64) is hi/lo in SMEM (SS MMA);
//  * every bias is added on the CUDA cores in fp32 (no ones column: the A
//    columns are exactly 128 / 64 wide);
//  * GLU uses the exact sigmoid of K1/K2's 3xTF32 mode: gate columns carry
//    -log2(e), sigma = 1/(1 + 2^gate') with ex2.approx and one shared
//    reciprocal per pair;
//  * the row state (xn, prior, agg, the step's mask) is fp32 in the per-CTA
//    scratch ([F/4][128 rows][4] layout, 1 MB per CTA).
//
// Per-row arithmetic is identical for every row whatever the batch size, tile
// position or grid (network.py:11-14).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include "k3_kernel.cuh"

namespace tbn {
namespace k3x {

using tc::rup;
using tc::tmem_load_n;
using tc::tmem_store_n;
using tc::kR;
using k3::f2;
using k3::ld32s;
using k3::st32s;

template <int F_, int ND_, int NA_, int S_, int C_>
struct Cfg {
  static constexpr int F = F_, ND = ND_, NA = NA_, S = S_, C = C_;
  static constexpr int H = ND + NA, N2 = 2 * H;
  static constexpr bool BF = false, X3 = true;
  static constexpr int FS = F / 4;                  // features per slice
  static constexpr int HS = H / 4;                  // GLU outputs per slice
  static_assert(F % 128 == 0 && F <= 512, "K3X: F in {128, ..., 512}, multiple of 128");
  static_assert(H == 128 && ND == NA, "K3X: h = 128 (hidden A hi|lo = 256 TMEM columns), n_d = n_a");
  // B chunks: tf32 hi block then lo block, N x Kc K-major canonical, 32 KB per chunk
  static constexpr int SLOT = 32768;
  static constexpr int KC_N2 = SLOT / (N2 * 8);     // 16: K per chunk for N = 256
  static constexpr int KC_ATT = SLOT / (F * 8);     // 8: K per chunk for N = F (512)
  static_assert(KC_N2 % 8 == 0 && KC_ATT % 8 == 0, "tf32 MMA K granule");
  static constexpr int AC = 128;                    // shared1 A chunk (TMEM hi|lo = 256 cols)
  static constexpr int NAC = F / AC;                // shared1 A chunks (4)
  static constexpr int CH_PER_AC = AC / KC_N2;      // ring chunks per A chunk (8)
  static constexpr int NCH_SH1 = F / KC_N2;         // 32
  static constexpr int NCH_HID = H / KC_N2;         // 8
  static constexpr int NCH_ATT = NA / KC_ATT;       // 8
  static constexpr int NSLOT = 3;
  // chunk sequence of one tile: transform(0) = sh1, sh2, fc1_0, fc2_0; then
  // per step: att_s, sh1, sh2, fc1_s, fc2_s
  static constexpr int TR_CH = NCH_SH1 + 3 * NCH_HID;
  static constexpr int STEP_CH = NCH_ATT + TR_CH;
  static constexpr int TILE_CH = TR_CH + S * STEP_CH;
  // global image: [consts][biases][sh1 chunks][sh2][fc1_0..S][fc2_0..S][att_1..S]
  static constexpr int C_SCALE = 0, C_SHIFT = F, C_HW = 2 * F;
  static constexpr int C_HB = C_HW + rup(ND * C, 4), C_END = rup(C_HB + C, 4);
  static constexpr int CONST_BYTES = C_END * 4;
  // folded biases (fp32, read through L1): sh1 | sh2 | fc1_0..S | fc2_0..S | att_1..S
  static constexpr int B_SH1 = 0, B_SH2 = N2, B_FC1 = 2 * N2, B_FC2 = B_FC1 + (S + 1) * N2;
  static constexpr int B_ATT = B_FC2 + (S + 1) * N2, B_END = B_ATT + S * F;
  static constexpr int O_BIAS = rup(CONST_BYTES, 128);
  static constexpr int BLK_SH1 = N2 * F * 8;        // hi + lo
  static constexpr int BLK_HID = N2 * H * 8;
  static constexpr int BLK_ATT = F * NA * 8;
  static constexpr int O_SH1 = rup(O_BIAS + B_END * 4, 128);
  static constexpr int O_SH2 = O_SH1 + BLK_SH1;
  static constexpr int O_FC1 = O_SH2 + BLK_HID;
  static constexpr int O_FC2 = O_FC1 + (S + 1) * BLK_HID;
  static constexpr int O_ATT = O_FC2 + (S + 1) * BLK_HID;
  static constexpr int IMG_BYTES = O_ATT + S * BLK_ATT;
  // SMEM plan
  static constexpr int OFF_RING = 0;
  static constexpr int OFF_AATT = OFF_RING + NSLOT * SLOT;     // A_att hi | lo, 128 x NA tf32 canonical
  static constexpr int AATT_BYTES = 128 * NA * 4;
  static constexpr int OFF_CONST = OFF_AATT + 2 * AATT_BYTES;
  static constexpr int OFF_XCH = rup(OFF_CONST + CONST_BYTES, 128);   // [2][4 q][4 c][32 lanes] float4
  static constexpr int OFF_STG = OFF_XCH + 2 * 4 * 4 * 32 * 16;
  static constexpr int STG_WARP = 32 * 16 * 4;
  static constexpr int OFF_LACC = OFF_STG + 16 * STG_WARP;     // head accumulators of slices 0, 1
  static constexpr int OFF_BAR = OFF_LACC + rup(256 * C * 4, 128);
  static constexpr int SMEM_BYTES = OFF_BAR + 256;
  static_assert(SMEM_BYTES <= 227 * 1024, "K3X shared-memory plan");
  // global scratch per CTA: prior, agg, the step's mask and xn, fp32 [F/4][128][4] each
  static constexpr size_t SCRATCH_PER_CTA = 4ull * 128 * F * 4;
  static constexpr int THREADS = 512;
};

struct Params {
  const uint8_t* wimg;
  float gamma;
};

struct Bars {
  uint64_t full[4];       // ring slot loaded (TMA complete_tx)
  uint64_t empty[4];      // ring slot's MMAs completed (tcgen05.commit)
  uint64_t cfull;         // consts
  uint64_t dfull;         // GEMM complete
  uint64_t afree;         // shared1: the A chunk's MMAs completed (its TMEM columns reusable)
  uint32_t tmem_base;
};

// Chunk v of the CTA's chunk stream -> (byte offset in the image, bytes, K of
// the chunk, N of the chunk)
template <class CF>
__device__ __forceinline__ void chunk_of(uint32_t v, uint32_t& off, int& kc, int& n) {
  int i = (int)(v % CF::TILE_CH);
  int step = 0, base_tr;
  if (i < CF::TR_CH) {
    base_tr = i;
  } else {
    i -= CF::TR_CH;
    step = i / CF::STEP_CH + 1;
    const int r = i % CF::STEP_CH;
    if (r < CF::NCH_ATT) {
      kc = CF::KC_ATT;
      n = CF::F;
      off = CF::O_ATT + (step - 1) * CF::BLK_ATT + r * CF::SLOT;
      return;
    }
    base_tr = r - CF::NCH_ATT;
  }
  kc = CF::KC_N2;
  n = CF::N2;
  if (base_tr < CF::NCH_SH1) {
    off = CF::O_SH1 + base_tr * CF::SLOT;
  } else {
    const int j = base_tr - CF::NCH_SH1;
    const int blk = j / CF::NCH_HID, r = j % CF::NCH_HID;
    const uint32_t bo = blk == 0 ? CF::O_SH2 : (blk == 1 ? CF::O_FC1 + step * CF::BLK_HID
                                                         : CF::O_FC2 + step * CF::BLK_HID);
    off = bo + r * CF::SLOT;
  }
}

// A operand split as the packer splits B: hi = rna_tf32(v), lo = rna_tf32(v - hi)
// (both exact tf32 operands; v - hi - lo <= 2^-22 |v|)
__device__ __forceinline__ float tf32_hi(float v) {
  return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}

template <class CF>
__global__ void __launch_bounds__(CF::THREADS, 1)
tabnet_wide_x3(const Params p, const ForwardArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int F = CF::F, H = CF::H, ND = CF::ND, NA = CF::NA, S = CF::S, C = CF::C;
  constexpr int FS = CF::FS, HS = CF::HS, N2 = CF::N2;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int q = warp & 3, c = warp >> 2;
  const int r = q * 32 + lane;                       // row within the tile (TMEM lane)
  Bars* bars = reinterpret_cast<Bars*>(smem + CF::OFF_BAR);
  const float* cst = reinterpret_cast<const float*>(smem + CF::OFF_CONST);
  const float* __restrict__ bias = reinterpret_cast<const float*>(p.wimg + CF::O_BIAS);
  float4* xch = reinterpret_cast<float4*>(smem + CF::OFF_XCH);
  const int64_t ntiles = (a.rows + 127) / 128;
  const uint32_t sbase = ptx::smem_u32(smem);
  const bool issuer = (warp == 0);                   // converged warp; elected lane inside the asm
  // scratch (fp32, [F/4][128][4]): feature f of row r at ((f/4)*128 + r)*4 + f%4
  float* prior_s = a.scratch + (size_t)blockIdx.x * (CF::SCRATCH_PER_CTA / 4);
  float* agg_s = prior_s + 128 * F;
  float* msk_s = agg_s + 128 * F;
  float* xn_s = msk_s + 128 * F;
  const size_t my_off = (size_t)(c * FS / 4) * 512 + (size_t)r * 4;
  float* my_prior = prior_s + my_off;
  float* my_agg = agg_s + my_off;
  float* my_msk = msk_s + my_off;
  float* my_xn = xn_s + my_off;
  auto at = [](float* base, int o) { return base + (o / 4) * 512; };   // slice feature o (multiple of 4)

  // row-major outputs through the warp's SMEM stage (as K3)
  float4* stg = reinterpret_cast<float4*>(smem + CF::OFF_STG + warp * CF::STG_WARP);
  auto out32 = [&](float* gbase, int nvalid, const float (&v)[32]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        stg[lane * 4 + (i ^ ((lane >> 1) & 3))] =
            make_float4(v[16 * h + 4 * i], v[16 * h + 4 * i + 1], v[16 * h + 4 * i + 2], v[16 * h + 4 * i + 3]);
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rr = j * 8 + (lane >> 2), qq = lane & 3;
        const float4 t = stg[rr * 4 + (qq ^ ((rr >> 1) & 3))];
        if (rr < nvalid) __stcs(reinterpret_cast<float4*>(gbase + (int64_t)rr * F + 16 * h + 4 * qq), t);
      }
      __syncwarp();
    }
  };

  const int64_t tiles_cta = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint32_t nchunks = (uint32_t)(tiles_cta * CF::TILE_CH);
  auto load_chunk = [&](uint32_t v) {
    uint32_t off;
    int kc, n;
    chunk_of<CF>(v, off, kc, n);
    const int sl = (int)(v % CF::NSLOT);
    ptx::mbar_arrive_expect_tx(&bars->full[sl], CF::SLOT);
    ptx::bulk_g2s(smem + CF::OFF_RING + sl * CF::SLOT, p.wimg + off, CF::SLOT, &bars->full[sl]);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < CF::NSLOT; ++i) {
      ptx::mbar_init(&bars->full[i], 1);
      ptx::mbar_init(&bars->empty[i], 1);
    }
    ptx::mbar_init(&bars->cfull, 1);
    ptx::mbar_init(&bars->dfull, 1);
    ptx::mbar_init(&bars->afree, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bars->cfull, CF::CONST_BYTES);
    ptx::bulk_g2s(smem + CF::OFF_CONST, p.wimg, CF::CONST_BYTES, &bars->cfull);
    for (uint32_t v = 0; v < (uint32_t)CF::NSLOT && v < nchunks; ++v) load_chunk(v);
  }
  if (warp == 0) ptx::tmem_alloc<512>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = bars->tmem_base;
  const uint32_t tq = tb + ((uint32_t)(q * 32) << 16);   // this warp's lane quarter
  ptx::mbar_wait(&bars->cfull, 0);
  if (a.scale) {
    float* cw = reinterpret_cast<float*>(smem + CF::OFF_CONST);
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      cw[CF::C_SCALE + f] = a.scale[f];
      cw[CF::C_SHIFT + f] = a.shift[f];
    }
  }
  __syncthreads();

  // TMEM column map
  constexpr uint32_t T_ATT = 0;                      // att D: [0, F)
  constexpr uint32_t T_A = 0, T_AL = 128;            // transform A hi | lo: [0, 256)
  constexpr uint32_t T_D = 256;                      // transform D: [256, 512)

  uint32_t v_next = 0;          // issuer: next chunk of the stream
  uint32_t dphase = 0, aphase = 0;
  // issue the MMAs of `nch` ring chunks: A from TMEM (kind 0: columns
  // [kbase, kbase + nch*KC) of the hi | lo A) or from SMEM (kind 1: A_att);
  // `first`: the first MMA overwrites D
  auto issue = [&](int kind, int nch, int kbase, bool first) {
    for (int ch = 0; ch < nch; ++ch) {
      const uint32_t v = v_next++;
      const int sl = (int)(v % CF::NSLOT);
      uint32_t off;
      int kc, n;
      chunk_of<CF>(v, off, kc, n);
      ptx::mbar_wait(&bars->full[sl], (v / CF::NSLOT) & 1u);
      ptx::tc_fence_after();
      const uint32_t bsm = sbase + CF::OFF_RING + sl * CF::SLOT;
      const uint32_t sbo = (uint32_t)(kc / 4) * 128u;
      const uint64_t bd0 = ptx::smem_desc(bsm, 128u, sbo);
      const uint64_t blo = (uint64_t)((n * kc * 4) >> 4);     // hi -> lo block, 16 B units
      if (kind == 0) {
        constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtTF32, 128, 256);
        for (int k0 = 0; k0 < kc; k0 += 8) {
          const uint64_t bd = bd0 + (uint64_t)(k0 * 2);
          const uint32_t ka = (uint32_t)(kbase + ch * kc + k0);
          const uint32_t acc = (first && ch == 0 && k0 == 0) ? 0u : 1u;
          ptx::mma_tf32_ts(tb + T_D, tb + T_A + ka, bd, idesc, acc);
          ptx::mma_tf32_ts(tb + T_D, tb + T_AL + ka, bd, idesc, 1u);
          ptx::mma_tf32_ts(tb + T_D, tb + T_A + ka, bd + blo, idesc, 1u);
        }
      } else {
        constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtTF32, 128, 256);
        // A_att canonical tf32: 8-row x 16-byte cores, LBO 128 B (K), SBO (NA/4)*128 B (M)
        const uint64_t ad0 = ptx::smem_desc(sbase + CF::OFF_AATT, 128u, (uint32_t)(NA / 4) * 128u);
        const uint64_t alo = (uint64_t)(CF::AATT_BYTES >> 4);
        for (int k0 = 0; k0 < kc; k0 += 8) {
          const uint64_t ad = ad0 + (uint64_t)((kbase + ch * kc + k0) * 2);
          for (int nh = 0; nh < F / 256; ++nh) {
            const uint64_t bd = bd0 + (uint64_t)(k0 * 2) + (uint64_t)((nh * 256 / 8) * sbo / 16);
            const uint32_t acc = (ch == 0 && k0 == 0) ? 0u : 1u;
            if (ptx::elect_one()) {
              ptx::mma_tf32_ss(tb + T_ATT + nh * 256, ad, bd, idesc, acc);
              ptx::mma_tf32_ss(tb + T_ATT + nh * 256, ad + alo, bd, idesc, 1u);
              ptx::mma_tf32_ss(tb + T_ATT + nh * 256, ad, bd + blo, idesc, 1u);
            }
            __syncwarp();
          }
        }
      }
      ptx::mma_commit(&bars->empty[sl]);
      // refill the previous chunk's slot once its MMAs are done
      if (v >= 1 && v - 1 + CF::NSLOT < nchunks) {
        const uint32_t pv = v - 1;
        if (lane == 0) {
          ptx::mbar_wait(&bars->empty[pv % CF::NSLOT], (pv / CF::NSLOT) & 1u);
          load_chunk(pv + CF::NSLOT);
        }
        __syncwarp();
      }
    }
  };
  // everyone waits for the GEMM's D
  auto wait_d = [&]() {
    ptx::mbar_wait_sleep(&bars->dfull, dphase);
    dphase ^= 1;
    ptx::tc_fence_after();
  };
  auto sync_all = [&]() {          // A writes (TMEM or SMEM) visible to the MMA issuer
    ptx::tmem_st_wait();
    ptx::fence_async_shared();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
  };

  // quarter-wide exchange of one float4 per slice thread (as K3)
  const uint32_t qbar = 2 + q;
  uint32_t xpar = 0;
  auto exchange = [&](float4 v, float4 (&o)[4]) {
    float4* slot = xch + ((xpar * 4 + q) * 4) * 32;
    slot[c * 32 + lane] = v;
    ptx::named_bar_sync(qbar, 128);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = slot[j * 32 + lane];
    xpar ^= 1u;
  };

  float gv[HS];                                      // this slice's GLU activations
  // d_sum @ head_W, accumulated per step by slices 0, 1: in SMEM (registers are the limit)
  float* const lacc = reinterpret_cast<float*>(smem + CF::OFF_LACC) + (c < 2 ? (c * 128 + r) * C : 0);

  // GLU over D = [lin' | gate'] (+ the folded biases) for this slice's outputs:
  // gv <- lin' sigma [+ sqrt(.5) gv], sigma = 1 / (1 + 2^gate')
  float dacc[2 * HS];                                // shared1 partial sums: lin [0, HS) | gate [HS, 2HS)
  auto glu_chunk = [&](bool residual, const float* __restrict__ b, int c0, const float (&lin)[16],
                       const float (&gate)[16]) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      const float l0 = lin[i] + __ldg(b + c * HS + c0 + i), l1 = lin[i + 1] + __ldg(b + c * HS + c0 + i + 1);
      const float g0 = gate[i] + __ldg(b + H + c * HS + c0 + i);
      const float g1 = gate[i + 1] + __ldg(b + H + c * HS + c0 + i + 1);
      const float a0 = fminf(g0, 63.0f), a1 = fminf(g1, 63.0f);
      const float2 d = __fadd2_rn(f2(tc::ex2_approx(a0), tc::ex2_approx(a1)), f2(1.0f, 1.0f));
      const float qq = tc::rcp_approx(d.x * d.y);
      const float2 sg = __fmul2_rn(f2(d.y, d.x), f2(qq, qq));
      const float2 l = f2(l0, l1);
      const float2 o = residual ? __ffma2_rn(l, sg, __fmul2_rn(f2(gv[c0 + i], gv[c0 + i + 1]), f2(kR, kR)))
                                : __fmul2_rn(l, sg);
      gv[c0 + i] = o.x;
      gv[c0 + i + 1] = o.y;
    }
  };
  // GLU over D = [lin' | gate'] (+ the folded biases) for this slice's outputs:
  // gv <- lin' sigma [+ sqrt(.5) gv], sigma = 1 / (1 + 2^gate')
  auto glu = [&](bool residual, const float* __restrict__ b) {
#pragma unroll
    for (int c0 = 0; c0 < HS; c0 += 16) {
      float lin[16], gate[16];
      tmem_load_n<16>(tq + T_D + c * HS + c0, lin);
      tmem_load_n<16>(tq + T_D + H + c * HS + c0, gate);
      ptx::tmem_ld_wait();
      glu_chunk(residual, b, c0, lin, gate);
    }
  };
  // the same from shared1's register partial sums
  auto glu_acc = [&](const float* __restrict__ b) {
#pragma unroll
    for (int c0 = 0; c0 < HS; c0 += 16) {
      float lin[16], gate[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        lin[i] = dacc[c0 + i];
        gate[i] = dacc[HS + c0 + i];
      }
      glu_chunk(false, b, c0, lin, gate);
    }
  };
  // dacc (+)= this slice's D columns (lin, gate)
  auto add_d = [&](auto first) {
    constexpr bool FIRST = decltype(first)::value;
#pragma unroll
    for (int j = 0; j < 2 * HS; j += 16) {
      float t[16];
      tmem_load_n<16>(tq + (j < HS ? T_D + c * HS + j : T_D + H + c * HS + (j - HS)), t);
      ptx::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if constexpr (FIRST) dacc[j + i] = t[i];
        else dacc[j + i] += t[i];
      }
    }
  };
  // hidden A <- g: slice c writes hi/lo of outputs [32c, 32c+32)
  auto store_g = [&]() {
    float hi[HS], lo[HS];
#pragma unroll
    for (int i = 0; i < HS; ++i) {
      hi[i] = tf32_hi(gv[i]);
      lo[i] = tf32_hi(gv[i] - hi[i]);
    }
    tmem_store_n<HS>(tq + T_A + c * HS, hi);
    tmem_store_n<HS>(tq + T_AL + c * HS, lo);
  };
  // shared1 (K = F) in NAC chunks of 128: slice k writes A = xn (* mask) for its
  // features into the A columns once the previous chunk's MMAs completed.  Each
  // chunk's MMAs start a fresh D and every thread adds its columns into fp32
  // register sums (dacc): the tensor core accumulates 3 x K/8 MMAs per D, and
  // 192 of them (K = 512) cost ~1e-5 relative; 48 per chunk keep the sum at the
  // K = 128 level of the hidden GEMMs
  auto shared1 = [&](bool with_mask) {
#pragma unroll
    for (int k = 0; k < CF::NAC; ++k) {
      if (k > 0) {                 // chunk k-1 done: its D into dacc, its A columns free
        ptx::mbar_wait(&bars->afree, aphase);
        aphase ^= 1u;
        ptx::tc_fence_after();
        if (k == 1) add_d(std::true_type{});
        else add_d(std::false_type{});
      }
      if (c == k) {
#pragma unroll 1
        for (int o = 0; o < FS; o += 16) {
          float xv[16], lo[16];
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 v = *reinterpret_cast<const float4*>(at(my_xn, o + i));
            xv[i] = v.x; xv[i + 1] = v.y; xv[i + 2] = v.z; xv[i + 3] = v.w;
          }
          if (with_mask) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const float4 mv = *reinterpret_cast<const float4*>(at(my_msk, o + i));
              xv[i] *= mv.x; xv[i + 1] *= mv.y; xv[i + 2] *= mv.z; xv[i + 3] *= mv.w;   // network.py:238
            }
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float h = tf32_hi(xv[i]);
            lo[i] = tf32_hi(xv[i] - h);
            xv[i] = h;
          }
          tmem_store_n<16>(tq + T_A + o, xv);
          tmem_store_n<16>(tq + T_AL + o, lo);
        }
      }
      sync_all();
      if (issuer) {
        issue(0, CF::CH_PER_AC, 0, true);
        ptx::mma_commit(&bars->afree);
      }
    }
    ptx::mbar_wait(&bars->afree, aphase);
    aphase ^= 1u;
    ptx::tc_fence_after();
    add_d(std::false_type{});
  };
#ifndef TBN_K3X_HID_SPLIT
#define TBN_K3X_HID_SPLIT 1
#endif
  // hidden GEMM (K = H): with TBN_K3X_HID_SPLIT, as two K-halves whose partial
  // D are summed in fp32 registers (halves the tensor core's accumulation chain)
  auto hidden = [&]() {
    sync_all();
    if constexpr (TBN_K3X_HID_SPLIT) {
      if (issuer) {
        issue(0, CF::NCH_HID / 2, 0, true);
        ptx::mma_commit(&bars->afree);
      }
      ptx::mbar_wait(&bars->afree, aphase);
      aphase ^= 1u;
      ptx::tc_fence_after();
      add_d(std::true_type{});
      ptx::tc_fence_before();
      __syncthreads();                               // every thread has read the half-K D
      ptx::tc_fence_after();
      if (issuer) {
        issue(0, CF::NCH_HID / 2, H / 2, true);
        ptx::mma_commit(&bars->dfull);
      }
    } else {
      if (issuer) {
        issue(0, CF::NCH_HID, 0, true);
        ptx::mma_commit(&bars->dfull);
      }
    }
  };
  // GLU of a hidden GEMM: D (+ the first K-half's partial sums)
  auto glu_hid = [&](const float* __restrict__ b) {
    if constexpr (TBN_K3X_HID_SPLIT) {
#pragma unroll
      for (int c0 = 0; c0 < HS; c0 += 16) {
        float lin[16], gate[16];
        tmem_load_n<16>(tq + T_D + c * HS + c0, lin);
        tmem_load_n<16>(tq + T_D + H + c * HS + c0, gate);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          lin[i] += dacc[c0 + i];
          gate[i] += dacc[HS + c0 + i];
        }
        glu_chunk(true, b, c0, lin, gate);
      }
    } else {
      glu(true, b);
    }
  };
  auto transform = [&](int s, bool with_mask) {     // network.py:124-141
    // shared1's A chunks overwrite TMEM columns [0, 256), i.e. z of features
    // [0, 256): the quarter's four slices must be done reading z first
    if (with_mask) ptx::named_bar_sync(qbar, 128);
    shared1(with_mask);
    glu_acc(bias + CF::B_SH1);
    store_g();
    hidden();
    wait_d();
    glu_hid(bias + CF::B_SH2);
    store_g();
    hidden();
    wait_d();
    glu_hid(bias + CF::B_FC1 + s * N2);
    store_g();
    hidden();
    wait_d();
    glu_hid(bias + CF::B_FC2 + s * N2);
  };
  // A_att (SMEM, canonical K-major tf32, no swizzle): element (row, k) at
  // (row/8)*SBO + (k/4)*128 + (row%8)*16 + (k%4)*4, SBO = NA/4*128; lo block after hi
  auto store_att_a = [&]() {
    if (c >= 2) {       // a = f[:, n_d:] lives in slices 2, 3: elements [32(c-2), +32)
      uint8_t* base = smem + CF::OFF_AATT + (r / 8) * (NA / 4) * 128 + (r % 8) * 16;
      const int k0 = (c - 2) * HS;
#pragma unroll
      for (int j = 0; j < HS; j += 4) {
        const float4 h = make_float4(tf32_hi(gv[j]), tf32_hi(gv[j + 1]), tf32_hi(gv[j + 2]), tf32_hi(gv[j + 3]));
        *reinterpret_cast<float4*>(base + ((k0 + j) / 4) * 128) = h;
        *reinterpret_cast<float4*>(base + CF::AATT_BYTES + ((k0 + j) / 4) * 128) =
            make_float4(tf32_hi(gv[j] - h.x), tf32_hi(gv[j + 1] - h.y), tf32_hi(gv[j + 2] - h.z), tf32_hi(gv[j + 3] - h.w));
      }
    }
  };

  for (int64_t m = 0; m < tiles_cta; ++m) {
    const int64_t tile = (int64_t)blockIdx.x + (int64_t)gridDim.x * m;
    const int64_t r0 = tile * 128;
    const int64_t row = r0 + r;
    const bool valid = row < a.rows;
    const int64_t wrow0 = r0 + q * 32;
    const int wvalid = a.rows - wrow0 < 32 ? (int)(a.rows - wrow0) : 32;
    const float* xrow = a.x + (valid ? row : 0) * F + c * FS;

    {   // xn slice from x (network.py:118-120) -> scratch
      int bad = 0;
#pragma unroll 1
      for (int o = 0; o < FS; o += 32) {
        float xv[32];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(xrow + o + i)) : make_float4(0, 0, 0, 0);
          bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
          xv[i] = v.x; xv[i + 1] = v.y; xv[i + 2] = v.z; xv[i + 3] = v.w;
        }
        if (!a.normalized) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            xv[i] = (xv[i] - cst[CF::C_SHIFT + c * FS + o + i]) * cst[CF::C_SCALE + c * FS + o + i];
        }
        st32s(at(my_xn, o), xv);
      }
      if (bad && a.err_flag) raise_flag(a.err_flag);
    }
    if (c < 2)
      for (int k = 0; k < C; ++k) lacc[k] = 0.0f;
    bool all_eta_zero = true;
    transform(0, false);                             // network.py:226-227
    store_att_a();                                   // A of step 1's attentive GEMM

    bool agg_pend = false, agg_zero = false;
    float agg_w = 0.0f;
    auto agg_update = [&]() {                        // agg += eta_s * m_s (network.py:245)
      if (!agg_pend) return;
      agg_pend = false;
#pragma unroll 1
      for (int o = 0; o < FS; o += 32) {
        float mv[32], ag[32];
        ld32s(at(my_msk, o), mv);
        if (agg_zero) {
#pragma unroll
          for (int i = 0; i < 32; ++i) ag[i] = 0.0f;
        } else {
          ld32s(at(my_agg, o), ag);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) ag[i] = fmaf(agg_w, mv[i], ag[i]);
        st32s(at(my_agg, o), ag);
      }
    };

    for (int s = 1; s <= S; ++s) {
      // ---- attentive transformer: z = prior * (a @ W_att + b) (network.py:233-235) ----
      sync_all();
      if (issuer) {
        issue(1, CF::NCH_ATT, 0, true);
        ptx::mma_commit(&bars->dfull);
      }
      agg_update();                                  // the previous step's, under the MMA
      wait_d();
      const float* __restrict__ batt = bias + CF::B_ATT + (s - 1) * F + c * FS;
      float pmax = -INFINITY, psum = 0.0f;
#pragma unroll 1
      for (int o = 0; o < FS; o += 32) {
        float z[32], pr[32];
        if (s > 1) ld32s(at(my_prior, o), pr);
        tmem_load_n<32>(tq + T_ATT + c * FS + o, z);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          z[i] += __ldg(batt + o + i);
          if (s > 1) z[i] *= pr[i];
        }
        tmem_store_n<32>(tq + T_ATT + c * FS + o, z);
#pragma unroll
        for (int i = 0; i < 32; ++i) { pmax = fmaxf(pmax, z[i]); psum += z[i]; }
      }
      ptx::tmem_st_wait();
      float4 o4[4];
      exchange(make_float4(pmax, psum, 0.0f, 0.0f), o4);
      const float zmax = fmaxf(fmaxf(o4[0].x, o4[1].x), fmaxf(o4[2].x, o4[3].x));
      const float zsum = (o4[0].y + o4[1].y) + (o4[2].y + o4[3].y);
      // Michelot's fixed point (sparsemax.py:32-39), as K3
      const float bound = (zsum - (float)F * zmax - 1.0f) * (1.0f / (float)F);
      float tau = fmaxf(-1.0f, bound - 9.5367431640625e-07f * fmaxf(1.0f, fabsf(bound)));
      float cnt_prev = (float)(F + 1);
      bool done = false;
      for (int it = 0; it <= F; ++it) {
        if (!__any_sync(0xffffffffu, !done)) break;
        float2 sa = f2(0.0f, 0.0f), ca = f2(0.0f, 0.0f);
        const float th = tau + zmax;
#pragma unroll 1
        for (int o = 0; o < FS; o += 64) {
          float z[64];
          tmem_load_n<32>(tq + T_ATT + c * FS + o, z);
          tmem_load_n<32, 32>(tq + T_ATT + c * FS + o + 32, z);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            const float2 mk = f2(z[i] > th ? 1.0f : 0.0f, z[i + 1] > th ? 1.0f : 0.0f);
            sa = __ffma2_rn(mk, f2(z[i], z[i + 1]), sa);
            ca = __fadd2_rn(ca, mk);
          }
        }
        const float cnt_slice = ca.x + ca.y;
        exchange(make_float4(fmaf(-cnt_slice, zmax, sa.x + sa.y), cnt_slice, 0.0f, 0.0f), o4);
        const float sm = (o4[0].x + o4[1].x) + (o4[2].x + o4[3].x);
        const float cn = (o4[0].y + o4[1].y) + (o4[2].y + o4[3].y);
        if (!done) {
          if (cn >= cnt_prev) {
            done = true;
          } else {
            cnt_prev = cn;
            tau = __fdividef(sm - 1.0f, cn);          // sparsemax.py:39
          }
        }
      }
      // mask, prior update (network.py:236-237) -> scratch; masks output
      float* mrow = a.masks ? a.masks + ((int64_t)(s - 1) * a.rows + wrow0) * F + c * FS : nullptr;
#pragma unroll 1
      for (int o = 0; o < FS; o += 32) {
        float z[32], pr[32];
        if (s > 1) ld32s(at(my_prior, o), pr);
        tmem_load_n<32>(tq + T_ATT + c * FS + o, z);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float mk = fmaxf((z[i] - zmax) - tau, 0.0f);               // sparsemax.py:40
          pr[i] = (s > 1 ? pr[i] : 1.0f) * (p.gamma - mk);                   // network.py:237
          z[i] = mk;
        }
        st32s(at(my_prior, o), pr);
        st32s(at(my_msk, o), z);
        if (mrow) out32(mrow + o, wvalid, z);
      }
      transform(s, true);                            // network.py:238-240
      // ---- d = relu(f[:, :n_d]); logits += d @ head_W; eta; agg += eta * m ----
      float pe = 0.0f;
      if (c < 2) {
#pragma unroll
        for (int i = 0; i < HS; ++i) {
          const float d = fmaxf(gv[i], 0.0f);
#pragma unroll
          for (int k = 0; k < C; ++k) lacc[k] = fmaf(d, cst[CF::C_HW + (c * HS + i) * C + k], lacc[k]);
          pe += d;
        }
      }
      exchange(make_float4(pe, 0.0f, 0.0f, 0.0f), o4);
      const float eta = o4[0].x + o4[1].x;
      if (s < S) store_att_a();                      // next step's attentive A
      const bool reset = all_eta_zero && eta > 0.0f;
      const float w = all_eta_zero ? (eta > 0.0f ? eta : 1.0f) : eta;
      all_eta_zero = all_eta_zero && !(eta > 0.0f);
      agg_pend = true;
      agg_zero = (s == 1 || reset);
      agg_w = w;
    }
    agg_update();                                    // the last step's

    // ---- head + softmax + argmax (network.py:253-256, :279) ----
    {
      float lg[C];
      for (int k0 = 0; k0 < C; k0 += 4) {
        float4 o4[4];
        exchange(make_float4(lacc[k0], k0 + 1 < C ? lacc[k0 + 1] : 0.0f, k0 + 2 < C ? lacc[k0 + 2] : 0.0f,
                             k0 + 3 < C ? lacc[k0 + 3] : 0.0f), o4);
        const float v[4] = {o4[0].x + o4[1].x, o4[0].y + o4[1].y, o4[0].z + o4[1].z, o4[0].w + o4[1].w};
        for (int u = 0; u < 4 && k0 + u < C; ++u) lg[k0 + u] = v[u] + cst[CF::C_HB + k0 + u];
      }
      if (c == 0 && valid) {
        float lmax = -INFINITY;
        for (int k = 0; k < C; ++k) lmax = fmaxf(lmax, lg[k]);
        float ex[C], es = 0.0f;
        for (int k = 0; k < C; ++k) { ex[k] = expf(lg[k] - lmax); es += ex[k]; }
        int best = 0;
        float bv = -1.0f;
        for (int k = 0; k < C; ++k) {
          const float pv = ex[k] / es;
          if (a.logits) a.logits[row * C + k] = lg[k];
          if (a.probs) a.probs[row * C + k] = pv;
          if (pv > bv) { bv = pv; best = k; }
        }
        if (a.pred) a.pred[row] = best;
      }
    }
    // ---- importance = agg / sum(agg) or mean_s(masks) (network.py:258-261) ----
    {
      float t0 = 0.0f;
#pragma unroll 1
      for (int o = 0; o < FS; o += 32) {
        float ag[32];
        ld32s(at(my_agg, o), ag);
#pragma unroll
        for (int i = 0; i < 32; ++i) t0 += ag[i];
      }
      float4 o4[4];
      exchange(make_float4(t0, 0.0f, 0.0f, 0.0f), o4);
      const float div = all_eta_zero ? (float)S : (o4[0].x + o4[1].x) + (o4[2].x + o4[3].x);
      const float rdiv = __frcp_rn(div);
      if (a.importance) {
        float* irow = a.importance + wrow0 * F + c * FS;
#pragma unroll 1
        for (int o = 0; o < FS; o += 32) {
          float ag[32];
          ld32s(at(my_agg, o), ag);
#pragma unroll
          for (int i = 0; i < 32; ++i) ag[i] *= rdiv;
          out32(irow + o, wvalid, ag);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(bars->tmem_base);
}

}  // namespace k3x
}  // namespace tbn
