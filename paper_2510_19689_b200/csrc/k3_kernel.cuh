// k3_kernel.cuh — K3: the whole TabNet forward (network.py:195-267) for WIDE
// models (F = 512 features, h = 128: BASELINE config 5) as one persistent
// sm_100a kernel, bf16 tcgen05 contractions.
//
// Why a third design: a wide row's state (xn, prior, agg, mask: 4 x 512 values)
// fits neither TMEM nor registers, and the model (1M params, 2 MB in bf16)
// does not fit shared memory.  So K3 keeps ONE 128-row tile per CTA on chip
// and streams everything else:
//
//   TMEM (512 cols, one tile)            SMEM
//   att   : D = z, 512 cols              B ring: 4 x 32 KB chunks (TMA bulk)
//   shared1: A = xm bf16 (K=512) 256 |   A_att (128 x 80 bf16, canonical)
//            D 256                       consts, shared1 bias, head
//   hidden: A = g (K=144) 72 | D 256     per-quarter exchange slots
//
//   global scratch per CTA (L2-resident, evict_last): xn, prior, agg and the
//   step's mask, each [F/8][128 rows][8] bf16 (512 KB per CTA at F = 512)
//
// 16 warps: warp w owns TMEM lane quarter q = w % 4 (rows 32q..32q+31) and
// slice c = w / 4: features [128c, 128c+128) and GLU outputs [32c, 32c+32).
// A row's 4 slice threads are the same lane of warps q, q+4, q+8, q+12; they
// combine sparsemax reductions through SMEM behind a per-quarter named barrier.
// The B operands stream in K-chunks (<= 32 KB) in a fixed per-tile sequence;
// the MMA-issuing thread refills a slot as soon as the MMAs that read it
// completed (tcgen05.commit -> the slot's empty barrier).
//
// GLU as in K2: sigma(u) = (1 + tanh(u/2))/2 with the halves (and the residual
// sqrt(1/2)) folded into the packed weights; the hidden/attentive biases ride
// in the GEMMs (ones column), shared1's bias (K = 512 has no spare column) is
// added on the CUDA cores.  Per-row arithmetic is identical for every row
// whatever the batch, tile position or grid (network.py:11-14).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "tc_kernel.cuh"

namespace tbn {
namespace k3 {

#ifdef TBN_ENABLE_TRACE
#ifdef TBN_TRACE_SYSFENCE      // hang debugging with TBN_TRACE_MAPPED (slow: perturbs timing)
#define TBN_K3_FENCE() __threadfence_system()
#else
#define TBN_K3_FENCE() do { } while (0)
#endif
#define TBN_K3T(k, v)                                                     \
  do {                                                                    \
    if (a.trace && blockIdx.x == 0 && (k) < 16384) {                      \
      ((volatile unsigned long long*)a.trace)[(k)] = (unsigned long long)(v); \
      TBN_K3_FENCE();                                                     \
    }                                                                     \
  } while (0)
#else
#define TBN_K3T(k, v) do { } while (0)
#endif

using tc::rup;
using tc::tmem_load_n;
using tc::tmem_store_n;
using tc::kR;

template <int F_, int ND_, int NA_, int S_, int C_>
struct Cfg {
  static constexpr int F = F_, ND = ND_, NA = NA_, S = S_, C = C_;
  static constexpr int H = ND + NA, N2 = 2 * H;
  static constexpr bool BF = true, X3 = false;
  static constexpr int FS = F / 4;                  // features per slice
  static constexpr int HS = H / 4;                  // GLU outputs per slice
  static_assert(F % 128 == 0 && F <= 512, "K3: F in {128, ..., 512}, multiple of 128");
  static_assert(N2 == 256 && ND == NA && HS % 16 == 0, "K3: h = 128, n_d = n_a");
  static constexpr int K1 = F;                      // shared1: no bias column (added on CUDA cores)
  static constexpr int KHID = H + 16;               // ones column at H
  static constexpr int KATT = NA + 16;              // ones column at NA
  // B chunks (N x Kc, K-major canonical, bf16): 32 KB max
  static constexpr int KC_N2 = 64;                  // K per chunk for N = 256
  static constexpr int KC_ATT = 32;                 // K per chunk for N = F (512)
  static constexpr int NCH_SH1 = K1 / KC_N2;        // 8
  static constexpr int NCH_HID = (KHID + KC_N2 - 1) / KC_N2;   // 3 (64, 64, 16)
  static constexpr int NCH_ATT = (KATT + KC_ATT - 1) / KC_ATT; // 3 (32, 32, 16)
  static constexpr int SLOT = 32768;
  static constexpr int NSLOT = 4;
  // chunk sequence of one tile: transform(0) = sh1, sh2, fc1_0, fc2_0; then
  // per step: att_s, sh1, sh2, fc1_s, fc2_s
  static constexpr int TR_CH = NCH_SH1 + 3 * NCH_HID;
  static constexpr int STEP_CH = NCH_ATT + TR_CH;
  static constexpr int TILE_CH = TR_CH + S * STEP_CH;
  // global image: [consts][sh1 chunks][sh2][fc1_0..S][fc2_0..S][att_1..S]
  static constexpr int C_SCALE = 0, C_SHIFT = F, C_B1 = 2 * F, C_HW = C_B1 + N2;
  static constexpr int C_HB = C_HW + rup(ND * C, 4), C_END = rup(C_HB + C, 4);
  static constexpr int CONST_BYTES = C_END * 4;
  static constexpr int BLK_SH1 = N2 * K1 * 2;
  static constexpr int BLK_HID = N2 * rup(KHID, 16) * 2;      // chunks packed back to back
  static constexpr int BLK_ATT = F * rup(KATT, 16) * 2;
  static constexpr int O_SH1 = rup(CONST_BYTES, 128);
  static constexpr int O_SH2 = O_SH1 + BLK_SH1;
  static constexpr int O_FC1 = O_SH2 + BLK_HID;
  static constexpr int O_FC2 = O_FC1 + (S + 1) * BLK_HID;
  static constexpr int O_ATT = O_FC2 + (S + 1) * BLK_HID;
  static constexpr int IMG_BYTES = O_ATT + S * BLK_ATT;
  // SMEM plan
  static constexpr int OFF_RING = 0;
  static constexpr int OFF_AATT = OFF_RING + NSLOT * SLOT;     // 128 x KATT bf16 canonical
  static constexpr int AATT_BYTES = 128 * KATT * 2;
  static constexpr int OFF_CONST = rup(OFF_AATT + AATT_BYTES, 128);
  static constexpr int OFF_XCH = rup(OFF_CONST + CONST_BYTES, 128);   // [4 q][4 c][32 lanes] float4
  static constexpr int OFF_STG = OFF_XCH + 2 * 4 * 4 * 32 * 16;   // double-buffered
  static constexpr int STG_WARP = 32 * 16 * 4;     // a warp's 32 rows x 16 features fp32
  static constexpr int OFF_BAR = OFF_STG + 16 * STG_WARP;
  static constexpr int SMEM_BYTES = OFF_BAR + 256;
  static_assert(SMEM_BYTES <= 227 * 1024, "K3 shared-memory plan");
  // global scratch per CTA: prior, agg, the step's mask and xn, bf16 each
  static constexpr size_t SCRATCH_PER_CTA = 4ull * 128 * F * 2;
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
  uint32_t tmem_base;
};

// Chunk v of the CTA's chunk stream -> (byte offset in the image, bytes, K of the chunk)
template <class CF>
__device__ __forceinline__ void chunk_of(uint32_t v, uint32_t& off, uint32_t& bytes, int& kc) {
  int i = (int)(v % CF::TILE_CH);
  int step = 0, base_tr;
  if (i < CF::TR_CH) {
    base_tr = i;
  } else {
    i -= CF::TR_CH;
    step = i / CF::STEP_CH + 1;
    const int r = i % CF::STEP_CH;
    if (r < CF::NCH_ATT) {
      const int k0 = r * CF::KC_ATT;
      kc = (CF::KATT - k0 < CF::KC_ATT) ? CF::KATT - k0 : CF::KC_ATT;
      off = CF::O_ATT + (step - 1) * CF::BLK_ATT + k0 * CF::F * 2;
      bytes = (uint32_t)(kc * CF::F * 2);
      return;
    }
    base_tr = r - CF::NCH_ATT;
  }
  if (base_tr < CF::NCH_SH1) {
    const int k0 = base_tr * CF::KC_N2;
    kc = CF::KC_N2;
    off = CF::O_SH1 + k0 * CF::N2 * 2;
  } else {
    const int j = base_tr - CF::NCH_SH1;
    const int blk = j / CF::NCH_HID, r = j % CF::NCH_HID;
    const int k0 = r * CF::KC_N2;
    kc = (CF::KHID - k0 < CF::KC_N2) ? CF::KHID - k0 : CF::KC_N2;
    const uint32_t bo = blk == 0 ? CF::O_SH2 : (blk == 1 ? CF::O_FC1 + step * CF::BLK_HID
                                                         : CF::O_FC2 + step * CF::BLK_HID);
    off = bo + k0 * CF::N2 * 2;
  }
  bytes = (uint32_t)(kc * CF::N2 * 2);
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
// 32 consecutive floats (16-B aligned): 8 independent 128-bit accesses, issued back to back
__device__ __forceinline__ void ld32(const float* p, float (&v)[32]) {
  float4 t[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) t[i] = *reinterpret_cast<const float4*>(p + 4 * i);
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[4 * i] = t[i].x; v[4 * i + 1] = t[i].y; v[4 * i + 2] = t[i].z; v[4 * i + 3] = t[i].w; }
}
// the same over a scratch in the coalesced [F/4][128 rows][4] layout: a row's
// consecutive float4s are 128*4 floats apart, the 32 lanes (rows) of a warp hit
// 512 consecutive bytes per access
__device__ __forceinline__ void ld32s(const float* p, float (&v)[32]) {
  float4 t[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) t[i] = *reinterpret_cast<const float4*>(p + 512 * i);
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[4 * i] = t[i].x; v[4 * i + 1] = t[i].y; v[4 * i + 2] = t[i].z; v[4 * i + 3] = t[i].w; }
}
__device__ __forceinline__ void st32s(float* p, const float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    *reinterpret_cast<float4*>(p + 512 * i) = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&b);
}
// 32 features as bf16 over a [F/8][128 rows][8] scratch (16 B per row-octet;
// a row's consecutive octets are 128*8 bf16 apart)
// The scratch is re-read every step and must survive the streaming outputs
// (masks/importance, ~18 KB per row) in L2: its accesses carry an evict_last
// policy and the output stores are streaming (st.global.cs).
#ifndef TBN_K3_L2HINT
#define TBN_K3_L2HINT 1
#endif
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void sth4(uint16_t* p, uint4 v, uint64_t pol) {
#if TBN_K3_L2HINT
  asm volatile("st.global.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
#else
  *reinterpret_cast<uint4*>(p) = v;
#endif
}
__device__ __forceinline__ uint4 ldh4(const uint16_t* p, uint64_t pol) {
#if TBN_K3_L2HINT
  uint4 v;
  asm volatile("ld.global.L2::cache_hint.v4.b32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol) : "memory");
  return v;
#else
  return *reinterpret_cast<const uint4*>(p);
#endif
}
__device__ __forceinline__ void st32h(uint16_t* p, const float (&v)[32], uint64_t pol) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    sth4(p + 1024 * i,
         make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                    pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7])), pol);
}
__device__ __forceinline__ void ld32h(const uint16_t* p, float (&v)[32], uint64_t pol) {
  uint4 t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = ldh4(p + 1024 * i, pol);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t w[4] = {t[i].x, t[i].y, t[i].z, t[i].w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[8 * i + 2 * j] = __uint_as_float(w[j] << 16);
      v[8 * i + 2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
    }
  }
}

// The per-feature-chunk loops that read the row-state scratch: unrolled by
// TBN_K3_UNR so the next chunk's L2 loads are in flight while this one is used.
#ifndef TBN_K3_UNR
#define TBN_K3_UNR 1
#endif
#define TBN_K3_STR2(x) #x
#define TBN_K3_STR(x) TBN_K3_STR2(x)
#define K3_SCRATCH_UNROLL _Pragma(TBN_K3_STR(unroll TBN_K3_UNR))

template <class CF>
__global__ void __launch_bounds__(CF::THREADS, 1)
tabnet_wide(const Params p, const ForwardArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int F = CF::F, H = CF::H, ND = CF::ND, NA = CF::NA, S = CF::S, C = CF::C;
  constexpr int FS = CF::FS, HS = CF::HS, N2 = CF::N2;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int q = warp & 3, c = warp >> 2;
  const int r = q * 32 + lane;                       // row within the tile (TMEM lane)
  Bars* bars = reinterpret_cast<Bars*>(smem + CF::OFF_BAR);
  const float* cst = reinterpret_cast<const float*>(smem + CF::OFF_CONST);
  float4* xch = reinterpret_cast<float4*>(smem + CF::OFF_XCH);
  const int64_t ntiles = (a.rows + 127) / 128;
  const uint32_t sbase = ptx::smem_u32(smem);
  const bool issuer = (warp == 0);                   // converged warp; elected lane inside the asm
  float* prior_s = a.scratch + (size_t)blockIdx.x * (CF::SCRATCH_PER_CTA / 4);
  float* agg_s = prior_s + 128 * F / 2;
  float* msk_s = agg_s + 128 * F / 2;
  // scratch layout (bf16) [F/8][128][8]: feature f of row r at ((f/8)*128 + r)*8 + f%8;
  // my_*(o) = this thread's 32-feature run starting at slice feature o
  const uint64_t pol = l2_evict_last();
  uint16_t* my_prior = reinterpret_cast<uint16_t*>(prior_s) + (size_t)(c * FS / 8) * 1024 + (size_t)r * 8;
  uint16_t* my_agg = reinterpret_cast<uint16_t*>(agg_s) + (size_t)(c * FS / 8) * 1024 + (size_t)r * 8;
  // the step's mask as bf16 (feeds x*m, itself rounded to bf16 for the MMA, and
  // the agg update) — halves its L2 footprint
  uint16_t* my_msk = reinterpret_cast<uint16_t*>(msk_s) + (size_t)(c * FS / 8) * 1024 + (size_t)r * 8;
  uint16_t* my_xn = my_msk + 128 * F;               // the tile's normalized x (bf16): x*m is bf16 anyway

  // Row-major outputs (masks, importance): a thread holds 32 features of its
  // own row, so direct stores touch 32 rows (lines) per warp instruction.  The
  // warp transposes through its SMEM stage, 16 features at a time (XOR-swizzled
  // float4 slots, conflict-free both ways), and stores 8 rows x 64 B per
  // instruction.  gbase = this warp's first row at the run's first feature.
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
    uint32_t off, bytes;
    int kc;
    chunk_of<CF>(v, off, bytes, kc);
    const int sl = (int)(v % CF::NSLOT);
    ptx::mbar_arrive_expect_tx(&bars->full[sl], bytes);
    ptx::bulk_g2s(smem + CF::OFF_RING + sl * CF::SLOT, p.wimg + off, bytes, &bars->full[sl]);
  };
  TBN_K3T(threadIdx.x == 0 ? 1 : 16383, 7);
  if (threadIdx.x == 0) {
    for (int i = 0; i < CF::NSLOT; ++i) {
      ptx::mbar_init(&bars->full[i], 1);
      ptx::mbar_init(&bars->empty[i], 1);
    }
    ptx::mbar_init(&bars->cfull, 1);
    ptx::mbar_init(&bars->dfull, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bars->cfull, CF::CONST_BYTES);
    ptx::bulk_g2s(smem + CF::OFF_CONST, p.wimg, CF::CONST_BYTES, &bars->cfull);
    for (uint32_t v = 0; v < (uint32_t)CF::NSLOT && v < nchunks; ++v) load_chunk(v);
  }
  if (warp == 0) ptx::tmem_alloc<512>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tq = bars->tmem_base + ((uint32_t)(q * 32) << 16);   // this warp's lane quarter
  if (threadIdx.x == 0) TBN_K3T(2, 8);
  ptx::mbar_wait(&bars->cfull, 0);
  if (threadIdx.x == 0) TBN_K3T(3, 9);
  if (a.scale) {
    float* cw = reinterpret_cast<float*>(smem + CF::OFF_CONST);
    for (int f = threadIdx.x; f < F; f += blockDim.x) {
      cw[CF::C_SCALE + f] = a.scale[f];
      cw[CF::C_SHIFT + f] = a.shift[f];
    }
  }
  __syncthreads();

  uint32_t v_next = 0;          // issuer: next chunk of the stream
  uint32_t dphase = 0;
  // One GEMM: barrier (all A written) -> warp 0 streams its nch chunks through
  // the ring -> everyone waits for D.  a_smem: A from SMEM (attentive) or TMEM.
  // kind: 0 = N2 output with A from TMEM, 1 = attentive (N = F, A in SMEM).
  uint32_t gcount = 0;
  auto gemm = [&](int kind, int nch, uint32_t tA, uint32_t tD, auto&& post) {
    if (lane == 0 && warp < 2) TBN_K3T(100 + warp * 400 + (gcount % 200) * 2, clock64());
    ptx::tmem_st_wait();
    ptx::fence_async_shared();
    ptx::tc_fence_before();
    __syncthreads();
    if (issuer) {
      ptx::tc_fence_after();
      int kbase = 0;
      for (int ch = 0; ch < nch; ++ch) {
        const uint32_t v = v_next++;
        const int sl = (int)(v % CF::NSLOT);
        uint32_t off, bytes;
        int kc;
        chunk_of<CF>(v, off, bytes, kc);
        if (lane == 0) TBN_K3T(8000 + (v % 4000), clock64());
        ptx::mbar_wait(&bars->full[sl], (v / CF::NSLOT) & 1u);
        if (lane == 0) TBN_K3T(12000 + (v % 4000), clock64());
        ptx::tc_fence_after();
        const uint32_t bsm = sbase + CF::OFF_RING + sl * CF::SLOT;
        const uint32_t sbo = (uint32_t)(kc / 8) * 128u;
        const uint64_t bd0 = ptx::smem_desc(bsm, 128u, sbo);
        if (kind == 0) {
          constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtBF16, 128, 256);
          for (int k0 = 0; k0 < kc; k0 += 16)
            ptx::mma_f16_ts(tD, tA + (kbase + k0) / 2, bd0 + (uint64_t)k0, idesc,
                            (kbase + k0) > 0 ? 1u : 0u);
        } else {
          constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtBF16, 128, 256);
          // A_att canonical: 8-row x 16-byte cores, LBO 128 B (K), SBO (KATT/8)*128 B (M)
          const uint64_t ad0 = ptx::smem_desc(sbase + CF::OFF_AATT, 128u, (uint32_t)(CF::KATT / 8) * 128u);
          for (int k0 = 0; k0 < kc; k0 += 16) {
            const uint64_t ad = ad0 + (uint64_t)(kbase + k0);          // +2 core matrices per 16 K
            for (int nh = 0; nh < F / 256; ++nh) {
              const uint64_t bd = bd0 + (uint64_t)k0 + (uint64_t)((nh * 256 / 8) * sbo / 16);
              if (ptx::elect_one())
                ptx::mma_f16_ss(tD + nh * 256, ad, bd, idesc, (kbase + k0) > 0 ? 1u : 0u);
              __syncwarp();
            }
          }
        }
        ptx::mma_commit(&bars->empty[sl]);
        // refill the previous chunk's slot once its MMAs are done (they were
        // queued before this chunk's, so the tensor pipe stays fed)
        if (v >= 1 && v - 1 + CF::NSLOT < nchunks) {
          const uint32_t pv = v - 1;
          if (lane == 0) {
            ptx::mbar_wait(&bars->empty[pv % CF::NSLOT], (pv / CF::NSLOT) & 1u);
            load_chunk(pv + CF::NSLOT);
          }
          __syncwarp();
        }
        kbase += kc;
      }
      ptx::mma_commit(&bars->dfull);
    }
    post();                                          // CUDA-core work in the MMA's shadow
    if (lane == 0 && warp < 2) TBN_K3T(101 + warp * 400 + (gcount % 200) * 2, clock64());
    ptx::mbar_wait_sleep(&bars->dfull, dphase);
    dphase ^= 1;
    ptx::tc_fence_after();
    ++gcount;
  };

  // quarter-wide exchange of one float4 per slice thread: returns the 4 slices' values
  const uint32_t qbar = 2 + q;                       // named barrier of lane quarter q (128 threads)
  uint32_t xpar = 0;
  auto exchange = [&](float4 v, float4 (&o)[4]) {
    // double-buffered [parity][q][c][lane]: the barrier of exchange k+1 proves
    // every thread has read exchange k, so one barrier per exchange suffices
    float4* slot = xch + ((xpar * 4 + q) * 4) * 32;
    slot[c * 32 + lane] = v;
    ptx::named_bar_sync(qbar, 128);
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = slot[j * 32 + lane];
    xpar ^= 1u;
  };

  // TMEM column map
  constexpr uint32_t T_ATT = 0;                      // att D: [0, F)
  constexpr uint32_t T_A = 0;                        // shared1/hidden A: [0, K/2)
  constexpr uint32_t T_D = 256;                      // shared1/hidden D: [256, 512)

  float gv[HS];                                      // this slice's GLU activations
  float lacc[C];                                     // d_sum @ head_W, accumulated per step (slices 0, 1)

  // GLU over D = [lin' | gate'] for this slice's outputs: gv <- lin'(1+t) [+ R gv]
  auto glu = [&](bool residual, bool add_b1) {
#pragma unroll
    for (int c0 = 0; c0 < HS; c0 += 16) {
      float lin[16], gate[16];
      tmem_load_n<16>(tq + T_D + c * HS + c0, lin);
      tmem_load_n<16>(tq + T_D + H + c * HS + c0, gate);
      ptx::tmem_ld_wait();
      if (add_b1) {                                  // shared1 bias (folded like the weights)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          lin[i] += cst[CF::C_B1 + c * HS + c0 + i];
          gate[i] += cst[CF::C_B1 + H + c * HS + c0 + i];
        }
      }
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float2 th = f2(tanh_approx(gate[i]), tanh_approx(gate[i + 1]));
        const float2 l = f2(lin[i], lin[i + 1]);
        float2 w = l;
        if (residual) w = __ffma2_rn(f2(gv[c0 + i], gv[c0 + i + 1]), f2(kR, kR), l);
        const float2 o = __ffma2_rn(l, th, w);
        gv[c0 + i] = o.x;
        gv[c0 + i + 1] = o.y;
      }
    }
  };
  // hidden A <- [g, 1, 0..]: slice c writes g[32c, 32c+32) (16 bf16 columns);
  // slice 0 also writes the ones column block [H, KHID)
  auto store_g = [&]() {
    float pk[HS / 2];
#pragma unroll
    for (int i = 0; i < HS / 2; ++i) pk[i] = __uint_as_float(pack_bf16(gv[2 * i], gv[2 * i + 1]));
    tmem_store_n<HS / 2>(tq + T_A + c * (HS / 2), pk);
    if (c == 0) {
      float ones[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) ones[i] = __uint_as_float(i == 0 ? pack_bf16(1.0f, 0.0f) : 0u);
      tmem_store_n<8>(tq + T_A + H / 2, ones);
    }
  };
  auto nopost = [] {};
  auto transform = [&]() {
    gemm(0, CF::NCH_SH1, tq + T_A, tq + T_D, nopost);
    glu(false, true);
    store_g();
    gemm(0, CF::NCH_HID, tq + T_A, tq + T_D, nopost);
    glu(true, false);
    store_g();
    gemm(0, CF::NCH_HID, tq + T_A, tq + T_D, nopost);
    glu(true, false);
    store_g();
    gemm(0, CF::NCH_HID, tq + T_A, tq + T_D, nopost);
    glu(true, false);
  };
  // A_att (SMEM, canonical K-major no-swizzle): element (row, k) at
  // (row/8)*SBO + (k/8)*128 + (row%8)*16 + (k%8)*2, SBO = KATT/8*128
  auto store_att_a = [&]() {
    uint8_t* base = smem + CF::OFF_AATT + (r / 8) * (CF::KATT / 8) * 128 + (r % 8) * 16;
    if (c >= 2) {       // a = f[:, n_d:] lives in slices 2, 3: elements [32(c-2), +32)
      const int k0 = (c - 2) * HS;
#pragma unroll
      for (int j = 0; j < HS; j += 8) {
        uint4 v;
        v.x = pack_bf16(gv[j], gv[j + 1]);
        v.y = pack_bf16(gv[j + 2], gv[j + 3]);
        v.z = pack_bf16(gv[j + 4], gv[j + 5]);
        v.w = pack_bf16(gv[j + 6], gv[j + 7]);
        *reinterpret_cast<uint4*>(base + ((k0 + j) / 8) * 128) = v;
      }
    } else if (c == 0) {  // the ones column block [NA, KATT)
      for (int k = NA; k < CF::KATT; k += 8)
        *reinterpret_cast<uint4*>(base + (k / 8) * 128) =
            make_uint4(k == NA ? pack_bf16(1.0f, 0.0f) : 0u, 0u, 0u, 0u);
    }
  };

  for (int64_t m = 0; m < tiles_cta; ++m) {
    const int64_t tile = (int64_t)blockIdx.x + (int64_t)gridDim.x * m;
    const int64_t r0 = tile * 128;
    const int64_t row = r0 + r;
    const bool valid = row < a.rows;
    const int64_t wrow0 = r0 + q * 32;               // this warp's first row
    const int wvalid = a.rows - wrow0 < 32 ? (int)(a.rows - wrow0) : 32;   // may be <= 0
    const float* xrow = a.x + (valid ? row : 0) * F + c * FS;

    // xn slice from x (network.py:118-120): this slice's 128 features
    auto xn_chunk = [&](int o, float (&xv)[32]) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 v = valid ? __ldg(reinterpret_cast<const float4*>(xrow + o + i)) : make_float4(0, 0, 0, 0);
        xv[i] = v.x; xv[i + 1] = v.y; xv[i + 2] = v.z; xv[i + 3] = v.w;
      }
      if (!a.normalized) {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          xv[i] = (xv[i] - cst[CF::C_SHIFT + c * FS + o + i]) * cst[CF::C_SCALE + c * FS + o + i];
      }
    };
    {   // transform(0)'s A = xn (bf16, K = F): slice c -> A cols [64c, 64c + 64)
      int bad = 0;
#pragma unroll 1
      for (int o = 0; o < FS; o += 32) {
        float xv[32];
        xn_chunk(o, xv);
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 raw = __ldg(reinterpret_cast<const float4*>(xrow + o + i));
            bad |= !isfinite(raw.x) | !isfinite(raw.y) | !isfinite(raw.z) | !isfinite(raw.w);
          }
        }
        float pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = __uint_as_float(pack_bf16(xv[2 * i], xv[2 * i + 1]));
        tmem_store_n<16>(tq + T_A + (c * FS + o) / 2, pk);
        st32h(my_xn + (o / 8) * 1024, xv, pol);
      }
      if (bad && a.err_flag) raise_flag(a.err_flag);
    }
#pragma unroll
    for (int k = 0; k < C; ++k) lacc[k] = 0.0f;
    bool all_eta_zero = true;
    transform();                                     // network.py:226-227
    store_att_a();                                   // A of step 1's attentive GEMM

    // agg += eta_s * m_s (network.py:245) needs step s's eta, known after its
    // transform; it runs in the shadow of step s+1's attentive MMA
    bool agg_pend = false, agg_zero = false;
    float agg_w = 0.0f;
    auto agg_update = [&]() {
      if (!agg_pend) return;
      agg_pend = false;
K3_SCRATCH_UNROLL
      for (int o = 0; o < FS; o += 32) {
        float mv[32], ag[32];
        ld32h(my_msk + (o / 8) * 1024, mv, pol);
        if (agg_zero) {
#pragma unroll
          for (int i = 0; i < 32; ++i) ag[i] = 0.0f;
        } else {
          ld32h(my_agg + (o / 8) * 1024, ag, pol);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) ag[i] = fmaf(agg_w, mv[i], ag[i]);
        st32h(my_agg + (o / 8) * 1024, ag, pol);
      }
    };

    for (int s = 1; s <= S; ++s) {
      // ---- attentive transformer: z = prior * (a @ W_att + b) (network.py:233-235) ----
      gemm(1, CF::NCH_ATT, 0, tq + T_ATT, agg_update);
      if (threadIdx.x == 0) TBN_K3T(1000 + 10 * s, clock64());
      // z' = prior * z in TMEM; slice max / sum
      float pmax = -INFINITY, psum = 0.0f;
K3_SCRATCH_UNROLL
      for (int o = 0; o < FS; o += 32) {
        float z[32], pr[32];
        if (s > 1) ld32h(my_prior + (o / 8) * 1024, pr, pol);   // in flight with the TMEM load
        tmem_load_n<32>(tq + T_ATT + c * FS + o, z);
        ptx::tmem_ld_wait();
        if (s > 1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] *= pr[i];
          tmem_store_n<32>(tq + T_ATT + c * FS + o, z);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) { pmax = fmaxf(pmax, z[i]); psum += z[i]; }
      }
      float4 o4[4];
      exchange(make_float4(pmax, psum, 0.0f, 0.0f), o4);
      const float zmax = fmaxf(fmaxf(o4[0].x, o4[1].x), fmaxf(o4[2].x, o4[3].x));
      const float zsum = (o4[0].y + o4[1].y) + (o4[2].y + o4[3].y);
      // Michelot's fixed point on the shifted logits (sparsemax.py:32-39), sort-free;
      // start max(-1, (sum z - 1)/F) nudged down 2^-20 (see K1/K2)
      if (threadIdx.x == 0) TBN_K3T(1001 + 10 * s, clock64());
      const float bound = (zsum - (float)F * zmax - 1.0f) * (1.0f / (float)F);
      float tau = fmaxf(-1.0f, bound - 9.5367431640625e-07f * fmaxf(1.0f, fabsf(bound)));
      float cnt_prev = (float)(F + 1);
      // the exchanges inside need warp-uniform control flow: a converged row
      // keeps exchanging (its values unused) until every row of the warp has
      // converged; lane l of the quarter's 4 warps is the same row, so the 4
      // warps run the same number of iterations
      bool done = false;
      for (int it = 0; it <= F; ++it) {
        if (!__any_sync(0xffffffffu, !done)) break;
        // compare the unshifted logits with tau + max (the shift of sparsemax.py:32
        // folded into the threshold; the sum is shifted back below) and keep two
        // 32-column TMEM loads in flight
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
      if (threadIdx.x == 0) TBN_K3T(1002 + 10 * s, clock64());
      // mask, prior update (network.py:236-237); the mask goes to the masks
      // output (or the scratch when none is requested), read back below
      // the mask goes to the coalesced scratch (read back for x*m and the agg
      // update) and, when requested, to the masks output
      float* mrow = a.masks ? a.masks + ((int64_t)(s - 1) * a.rows + wrow0) * F + c * FS : nullptr;
K3_SCRATCH_UNROLL
      for (int o = 0; o < FS; o += 32) {
        float z[32], pr[32];
        if (s > 1) ld32h(my_prior + (o / 8) * 1024, pr, pol);
        tmem_load_n<32>(tq + T_ATT + c * FS + o, z);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float mk = fmaxf((z[i] - zmax) - tau, 0.0f);               // sparsemax.py:40
          pr[i] = (s > 1 ? pr[i] : 1.0f) * (p.gamma - mk);                   // network.py:237
          z[i] = mk;
        }
        st32h(my_prior + (o / 8) * 1024, pr, pol);
        st32h(my_msk + (o / 8) * 1024, z, pol);
        if (mrow) out32(mrow + o, wvalid, z);
      }
      if (threadIdx.x == 0) TBN_K3T(1003 + 10 * s, clock64());
      ptx::named_bar_sync(qbar, 128);                // every slice of the quarter is done with z
      // x * mask -> shared1 A (network.py:238), bf16, slice c -> A cols [64c, 64c + 64)
K3_SCRATCH_UNROLL
      for (int o = 0; o < FS; o += 32) {
        float xv[32], mv[32];
        ld32h(my_msk + (o / 8) * 1024, mv, pol);
        ld32h(my_xn + (o / 8) * 1024, xv, pol);
        float pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = __uint_as_float(pack_bf16(mv[2 * i] * xv[2 * i], mv[2 * i + 1] * xv[2 * i + 1]));
        tmem_store_n<16>(tq + T_A + (c * FS + o) / 2, pk);
      }
      if (threadIdx.x == 0) TBN_K3T(1004 + 10 * s, clock64());
      transform();                                   // network.py:239-240
      if (threadIdx.x == 0) TBN_K3T(1005 + 10 * s, clock64());
      // ---- d = relu(f[:, :n_d]); logits += d @ head_W; eta; agg += eta * m
      // (network.py:241-246, :253: the head is linear so d_sum @ W accumulates) ----
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
      if (s < S) store_att_a();                      // next step's attentive A (frees gv)
      if (threadIdx.x == 0) TBN_K3T(1006 + 10 * s, clock64());
      // while every eta so far is 0, agg holds sum_s m (the fallback numerator,
      // network.py:259-261); the first eta > 0 resets it (see K2)
      const bool reset = all_eta_zero && eta > 0.0f;
      const float w = all_eta_zero ? (eta > 0.0f ? eta : 1.0f) : eta;
      all_eta_zero = all_eta_zero && !(eta > 0.0f);
      agg_pend = true;
      agg_zero = (s == 1 || reset);
      agg_w = w;

    }
    agg_update();                                    // the last step's (no attentive MMA follows)

    // ---- head + softmax + argmax (network.py:253-256, :279) ----
    {
      const float* pl = lacc;
      float lg[C];
      for (int k0 = 0; k0 < C; k0 += 4) {
        float4 o4[4];
        exchange(make_float4(pl[k0], k0 + 1 < C ? pl[k0 + 1] : 0.0f, k0 + 2 < C ? pl[k0 + 2] : 0.0f,
                             k0 + 3 < C ? pl[k0 + 3] : 0.0f), o4);
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
        ld32h(my_agg + (o / 8) * 1024, ag, pol);
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
          ld32h(my_agg + (o / 8) * 1024, ag, pol);
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

}  // namespace k3
}  // namespace tbn
