// tc_kernel.cuh — K1: the whole TabNet forward (network.py:195-267) as ONE
// persistent sm_100a kernel.  Row tiles of 128 (one TMEM lane per row) stay
// on-chip for all decision steps:
//
//   TMEM (per row-group of 128 rows)      SMEM (per CTA)
//   [D  accumulator, DW cols ]            consts: affine, folded biases, head
//   [A  operand hi,  KA cols ]            resident shared1/shared2 (if they fit)
//   [A  operand lo,  KA cols ] (3xTF32)   weight ring (per-step B operands, TMA bulk)
//   [xn F][prior F][agg F]  per-row state x staging (TMA bulk, one tile ahead)
//                                         row staging for coalesced/bulk output
//
// Warp roles: NG row-groups x 8 warps, nothing else.  Within a
// group, warps w and w+4 share TMEM lane quarter w%4 (= the same 32 rows) and
// split each row's columns: "half 0" owns GLU columns [0, H/2) — the decision
// part d — and "half 1" owns [H/2, H) — the attention state a (n_d == n_a).
// Sparsemax is computed redundantly by both halves from TMEM; features are
// split for the prior/mask/A updates.  After every A write the group meets at
// a 256-thread named barrier and one elected thread issues the tcgen05.mma
// chain (kind::tf32, A from TMEM, B from SMEM) and commits it to the group's
// mbarrier — no separate MMA or producer warp, no cross-group lockstep: that
// thread also streams the group's own weight ring and next x tile (TMA bulk),
// so the NG groups run independently and overlap each other's MMA / epilogue.
//
// Per-row arithmetic is identical for every row whatever the batch size, tile
// position, grid size or group: the batch-invariance contract (network.py:11-14).
#pragma once
#include "tbn_rtc.h"
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
#include "tbn_args.h"

namespace tbn {
namespace tc {

constexpr int kPrecTF32x3 = 0;
constexpr int kPrecTF32 = 1;
constexpr int kPrecBF16 = 2;

constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }
constexpr int pow2ceil(int v) { int p = 32; while (p < v) p <<= 1; return p; }

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kR = 0.70710678118654752440f;   // sqrt(0.5), network.py:29

template <int F_, int ND_, int NA_, int S_, int C_, int PREC_>
struct Cfg {
  static constexpr int F = F_, ND = ND_, NA = NA_, S = S_, C = C_, PREC = PREC_;
  static constexpr int H = ND + NA, N2 = 2 * H;
  static constexpr bool X3 = (PREC == kPrecTF32x3);
  static constexpr bool BF = (PREC == kPrecBF16);    // kind::f16 with bf16 operands
  static constexpr int KG = BF ? 16 : 8;             // MMA K granule
  static constexpr int ESZ = BF ? 2 : 4;             // operand element bytes
  // Every GEMM carries its bias as an extra K row of B, multiplied by a column
  // of ones in A at index F (shared1), H (hidden) or NA (attentive).
  static constexpr int K1 = rup(F + 1, KG);            // shared1 K
  static constexpr int KHID = H + KG;                  // shared2 / fc1 / fc2 K
  static constexpr int KATT = NA + KG;                 // attentive K
  static constexpr int FN = rup(F, 16);                // attentive N (M=128 needs N%16==0)
  static constexpr int KA_EL = cmax(cmax(K1, KHID), KATT); // A operand elements
  static constexpr int KA = BF ? KA_EL / 2 : KA_EL;          // A operand TMEM columns
  static constexpr int DW = cmax(N2, FN);              // accumulator columns
  // TMEM column map (per group)
  static constexpr int T_D = 0, T_A = DW, T_AL = T_A + KA, T_XN = T_AL + (X3 ? KA : 0);
  static constexpr int T_PR = T_XN + F, T_AG = T_PR + F, T_END = T_AG + F;
  static constexpr int TCOLS_G = pow2ceil(T_END);
  static constexpr int NG = (2 * TCOLS_G <= 512) ? 2 : 1;
  static constexpr int TCOLS = NG * TCOLS_G;
  static_assert(TCOLS <= 512, "per-row state does not fit in TMEM");
  static_assert(N2 <= 256 && FN <= 256, "MMA N > 256");
  // weight blocks (B operands, K-major canonical, hi [+ lo])
  static constexpr int PARTS = X3 ? 2 : 1;
  static constexpr int B_SH1 = PARTS * N2 * K1 * ESZ;
  static constexpr int B_HID = PARTS * N2 * KHID * ESZ;  // shared2, fc1_s, fc2_s
  static constexpr int B_ATT = PARTS * FN * KATT * ESZ;
  // consts (floats): scale F | shift F | bias sh1 N2 | sh2 N2 | fc1 (S+1)N2 | fc2 (S+1)N2 |
  //                  att S*FN | head_W ND*C | head_b C
  static constexpr int C_SCALE = 0, C_SHIFT = C_SCALE + rup(F, 4), C_BSH1 = C_SHIFT + rup(F, 4);
  static constexpr int C_BSH2 = C_BSH1 + N2, C_BFC1 = C_BSH2 + N2, C_BFC2 = C_BFC1 + (S + 1) * N2;
  static constexpr int C_BATT = C_BFC2 + (S + 1) * N2, C_HW = C_BATT + S * FN;
  static constexpr int C_HB = C_HW + rup(ND * C, 4), C_END = rup(C_HB + C, 4);
  static constexpr int CONST_BYTES = C_END * 4;
  // shared-memory plan
  // Row I/O: thread-per-row reads/writes of a dense [128][F] tile are bank-
  // conflict-free for odd F (and cheap for small F); otherwise go through a
  // [F][129] transpose buffer with cooperative coalesced global accesses.
  static constexpr bool DENSE_IO = (F % 2 == 1) || (F <= 16);
  static constexpr int XSTAGE = rup(128 * F * 4, 128);
  static constexpr int TSTAGE = DENSE_IO ? rup(128 * F * 4, 128) : rup(F * 129 * 4, 128);
  static constexpr int FIXED = rup(CONST_BYTES, 128) + NG * (XSTAGE + TSTAGE + 8192) + 1024;
  static constexpr int RING_SLOT_ALL = cmax(cmax(B_SH1, B_HID), B_ATT);
  static constexpr int RING_SLOT_RES = cmax(B_HID, B_ATT);
  static constexpr int SMEM_BUDGET = 225 * 1024;
  // Each row group streams its own weight ring (NSLOT slots); shared1/shared2
  // stay resident for the whole CTA when they fit.
  static constexpr bool RESIDENT = FIXED + B_SH1 + B_HID + NG * 2 * RING_SLOT_RES <= SMEM_BUDGET;
  static constexpr int SLOT = RESIDENT ? RING_SLOT_RES : RING_SLOT_ALL;
  static constexpr int RES_BYTES = RESIDENT ? (B_SH1 + B_HID) : 0;
  static constexpr int NSLOT = (FIXED + RES_BYTES + NG * 3 * SLOT <= SMEM_BUDGET) ? 3 : 2;
  static constexpr int SMEM_BYTES = FIXED + RES_BYTES + NG * NSLOT * SLOT;
  // non-resident blocks per tile (the ring sequence)
  static constexpr int NB = RESIDENT ? 2 + 3 * S : 4 + 5 * S;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared-memory plan exceeds 227 KB");
  // GEMMs per tile: step 0 transform (4) + S x (att + transform 4)
  static constexpr int GEMMS = 4 + 5 * S;
  static constexpr int HH = H / 2;                      // GLU columns per half
  static constexpr int KH = K1 / 2;                     // shared1 K columns per half
  static_assert(ND == NA, "column split assumes n_d == n_a (all BASELINE configs)");
  static_assert(!BF || (KH % 2 == 0 && HH % 2 == 0), "bf16 A chunks pack element pairs");
  static_assert(HH % 4 == 0, "half split granularity");
  static constexpr int THREADS = NG * 256;
};

// Global-memory weight image (built by the host packer, tc_pack):
//   [consts][sh1 blk][sh2 blk][fc1_0..fc1_S blks][fc2_0..fc2_S blks][att_1..att_S blks]
struct TcParams {
  const uint8_t* wimg;     // device image
  uint32_t off_sh1, off_sh2, off_fc1, off_fc2, off_att;   // byte offsets of block 0 of each kind
  float gamma;
};

// ---- TMEM <-> registers helpers over an exact column count (any N) ----------
template <int N, int OFF = 0, int M>
__device__ __forceinline__ void tmem_load_n(uint32_t taddr, float (&v)[M]) {
  if constexpr (N >= 16) {
    uint32_t r[16];
    TBN_TMEM_LD16(taddr, r);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[OFF + i] = __uint_as_float(r[i]);
    tmem_load_n<N - 16, OFF + 16>(taddr + 16, v);
  } else if constexpr (N >= 8) {
    uint32_t r[8];
    TBN_TMEM_LD8(taddr, r);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[OFF + i] = __uint_as_float(r[i]);
    tmem_load_n<N - 8, OFF + 8>(taddr + 8, v);
  } else if constexpr (N >= 4) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr));
    v[OFF] = __uint_as_float(r0); v[OFF + 1] = __uint_as_float(r1);
    v[OFF + 2] = __uint_as_float(r2); v[OFF + 3] = __uint_as_float(r3);
    tmem_load_n<N - 4, OFF + 4>(taddr + 4, v);
  } else if constexpr (N >= 2) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr));
    v[OFF] = __uint_as_float(r0); v[OFF + 1] = __uint_as_float(r1);
    tmem_load_n<N - 2, OFF + 2>(taddr + 2, v);
  } else if constexpr (N == 1) {
    uint32_t r0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(taddr));
    v[OFF] = __uint_as_float(r0);
  }
}

template <int N, int OFF = 0, int M>
__device__ __forceinline__ void tmem_store_n(uint32_t taddr, const float (&v)[M]) {
  if constexpr (N >= 16) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(v[OFF + i]);
    TBN_TMEM_ST16(taddr, r);
    tmem_store_n<N - 16, OFF + 16>(taddr + 16, v);
  } else if constexpr (N >= 8) {
    uint32_t r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(v[OFF + i]);
    TBN_TMEM_ST8(taddr, r);
    tmem_store_n<N - 8, OFF + 8>(taddr + 8, v);
  } else if constexpr (N >= 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
                 "r"(__float_as_uint(v[OFF])), "r"(__float_as_uint(v[OFF + 1])),
                 "r"(__float_as_uint(v[OFF + 2])), "r"(__float_as_uint(v[OFF + 3])));
    tmem_store_n<N - 4, OFF + 4>(taddr + 4, v);
  } else if constexpr (N >= 2) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr),
                 "r"(__float_as_uint(v[OFF])), "r"(__float_as_uint(v[OFF + 1])));
    tmem_store_n<N - 2, OFF + 2>(taddr + 2, v);
  } else if constexpr (N == 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr),
                 "r"(__float_as_uint(v[OFF])));
  }
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Round-to-nearest (ties away) to TF32 on the bit pattern: the result has its
// 13 low mantissa bits zero, so the tensor core's operand truncation is exact.
__device__ __forceinline__ float tf32_rna(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// Compile-time loop over [0, N) in chunks of CH columns: fn(integral_constant<O>, integral_constant<L>).
template <int N, int CH = 16, int O = 0, class Fn>
__device__ __forceinline__ void chunked(Fn&& fn) {
  if constexpr (O < N) {
    constexpr int L = (N - O < CH) ? (N - O) : CH;
    fn(std::integral_constant<int, O>{}, std::integral_constant<int, L>{});
    chunked<N, CH, O + L>(fn);
  }
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// Write L columns of an A operand row to TMEM.  The tensor core reads fp32
// operands as tf32 by truncation, so A_hi = v itself (read as trunc(v)) and,
// for 3xTF32, A_lo = v - trunc(v) (exact in fp32; itself truncated by the MMA,
// leaving a 2^-22 relative error per product).
template <class CF, int L, int M>
__device__ __forceinline__ void store_a(uint32_t t_a, uint32_t t_al, const float (&v)[M]) {
  if constexpr (CF::BF) {
    static_assert(L % 2 == 0, "bf16 A chunks pack element pairs");
    float pk[L / 2];
#pragma unroll
    for (int i = 0; i < L / 2; ++i) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);   // low = even
      pk[i] = *reinterpret_cast<const float*>(&b);
    }
    tmem_store_n<L / 2>(t_a, pk);
    return;
  }
  tmem_store_n<L>(t_a, v);
  if constexpr (CF::X3) {
    float lo[L];
#pragma unroll
    for (int i = 0; i + 1 < L; i += 2) {
      const float2 d = __fadd2_rn(f2(v[i], v[i + 1]),
                                  f2(-__uint_as_float(__float_as_uint(v[i]) & 0xFFFFE000u),
                                     -__uint_as_float(__float_as_uint(v[i + 1]) & 0xFFFFE000u)));
      lo[i] = d.x;
      lo[i + 1] = d.y;
    }
    if constexpr (L % 2)
      lo[L - 1] = v[L - 1] - __uint_as_float(__float_as_uint(v[L - 1]) & 0xFFFFE000u);
    tmem_store_n<L>(t_al, lo);
  }
}
// TMEM column of A element e (bf16 packs two elements per column)
template <class CF>
__host__ __device__ constexpr uint32_t acol(int e) { return CF::BF ? (uint32_t)(e / 2) : (uint32_t)e; }

// A <- v[0..K) in 16-column chunks
template <class CF, int K, int M>
__device__ __forceinline__ void store_a_all(uint32_t t_a, uint32_t t_al, const float (&v)[M]) {
  chunked<K>([&](auto o, auto l) {
    constexpr int O = decltype(o)::value, L = decltype(l)::value;
    float c[L];
#pragma unroll
    for (int i = 0; i < L; ++i) c[i] = v[O + i];
    store_a<CF, L>(t_a + acol<CF>(O), t_al + acol<CF>(O), c);
  });
}

// One GEMM's tcgen05.mma chain, fully unrolled: D = A(TMEM, K cols) x B(SMEM,
// N x K K-major canonical); 3xTF32 adds A_lo x B_hi and A_hi x B_lo.
template <class CF, int K, int N>
__device__ __forceinline__ void issue_gemm(uint32_t tD, uint32_t tA, uint32_t tAL, uint32_t bsm) {
  if constexpr (CF::BF) {
    constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtBF16, 128, N);
    constexpr uint32_t sbo = (K / 8) * 128u;
    const uint64_t d0 = ptx::smem_desc(bsm, 128u, sbo);
#pragma unroll
    for (int k0 = 0; k0 < K; k0 += 16)       // 16 K elements = 2 core matrices = 32 B
      ptx::mma_f16_ts(tD, tA + k0 / 2, d0 + (uint64_t)k0, idesc, k0 > 0 ? 1u : 0u);
    return;
  }
  constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtTF32, 128, N);
  constexpr uint32_t sbo = (K / 4) * 128u;
  constexpr uint64_t lo = (uint64_t)((N * K * 4) >> 4);     // hi -> lo block, in 16 B units
  const uint64_t d0 = ptx::smem_desc(bsm, 128u, sbo);
#pragma unroll
  for (int k0 = 0; k0 < K; k0 += 8) {
    const uint64_t bd = d0 + (uint64_t)(k0 * 2);             // start address += k0 * 32 B
    ptx::mma_tf32_ts(tD, tA + k0, bd, idesc, k0 > 0 ? 1u : 0u);
    if constexpr (CF::X3) {
      ptx::mma_tf32_ts(tD, tAL + k0, bd, idesc, 1u);
      ptx::mma_tf32_ts(tD, tA + k0, bd + lo, idesc, 1u);
    }
  }
}

// ---------------------------------------------------------------------------
template <class CF>
struct Smem {
  static constexpr int OFF_CONST = 0;
  static constexpr int OFF_X = rup(CF::CONST_BYTES, 128);
  static constexpr int OFF_T = OFF_X + CF::NG * CF::XSTAGE;
  static constexpr int OFF_RES = rup(OFF_T + CF::NG * CF::TSTAGE, 1024);
  static constexpr int OFF_RING = OFF_RES + CF::RES_BYTES;
  static constexpr int OFF_XCH = OFF_RING + CF::NG * CF::NSLOT * CF::SLOT;   // 4 KB per group
  static constexpr int OFF_BAR = OFF_XCH + CF::NG * 8192;   // float4 pair-exchange buffer
  static constexpr int TOTAL = OFF_BAR + 256;
  static_assert(TOTAL <= 227 * 1024, "smem");
};

struct Bars {
  uint64_t wfull[2][4];    // per row group ring
  uint64_t xfull[2];
  uint64_t dfull[2];
  uint64_t cfull;
  uint32_t tmem_base;
};

// The weight-block sequence of one tile pair: index j in [0, GEMMS)
//   j = 0..3          : sh1, sh2, fc1_0, fc2_0
//   j = 4 + 5(s-1) + 0: att_s ; +1..+4: sh1, sh2, fc1_s, fc2_s   (s = 1..S)
// kind: 0 sh1, 1 sh2, 2 fc1, 3 fc2, 4 att
__device__ __forceinline__ void gemm_of(int j, int& kind, int& step) {
  if (j < 4) { kind = j; step = 0; return; }
  int q = j - 4;
  step = q / 5 + 1;
  int r = q % 5;
  kind = (r == 0) ? 4 : r - 1;
}

// Position u (0..NB-1) of a tile's ring sequence -> (kind, step).
template <class CF>
__device__ __forceinline__ void ring_block(int u, int& kind, int& step) {
  if constexpr (CF::RESIDENT) {
    if (u < 2) { kind = 2 + u; step = 0; return; }
    const int q = u - 2;
    step = q / 3 + 1;
    const int r = q % 3;
    kind = (r == 0) ? 4 : r + 1;
  } else {
    gemm_of(u, kind, step);
  }
}

template <class CF>
__device__ __forceinline__ uint32_t block_offset(const TcParams& p, int kind, int step) {
  switch (kind) {
    case 0: return p.off_sh1;
    case 1: return p.off_sh2;
    case 2: return p.off_fc1 + (uint32_t)step * CF::B_HID;
    case 3: return p.off_fc2 + (uint32_t)step * CF::B_HID;
    default: return p.off_att + (uint32_t)(step - 1) * CF::B_ATT;
  }
}
template <class CF>
__device__ __forceinline__ uint32_t block_bytes(int kind) {
  return kind == 0 ? CF::B_SH1 : (kind == 4 ? CF::B_ATT : CF::B_HID);
}
template <class CF>
__device__ __forceinline__ bool is_resident(int kind) {
  return CF::RESIDENT && (kind == 0 || kind == 1);
}

// ---------------------------------------------------------------------------
// Debug timeline (build with -DTBN_ENABLE_TRACE and run with TBN_TRACE=1):
// slot k of CTA 0 <- clock64.  Compiled out of production builds.
#ifdef TBN_ENABLE_TRACE
#define TBN_TRACE(k)                                                        \
  do {                                                                      \
    if (a.trace && blockIdx.x == 0 && (k) < 16384) a.trace[(k)] = clock64(); \
  } while (0)
#else
#define TBN_TRACE(k) \
  do {               \
  } while (0)
#endif

template <class CF>
__global__ void __launch_bounds__(CF::THREADS, 1)
tabnet_fused_tc(const TcParams p, const ForwardArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  using SM = Smem<CF>;
  constexpr int F = CF::F, H = CF::H, ND = CF::ND, NA = CF::NA, S = CF::S, C = CF::C, NG = CF::NG;
  constexpr int HH = CF::HH, KH = CF::KH, K1 = CF::K1;
  const float* cst = reinterpret_cast<const float*>(smem + SM::OFF_CONST);
  Bars* bars = reinterpret_cast<Bars*>(smem + SM::OFF_BAR);
#ifdef TBN_K1_PLAINWARP
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#else
  // warp index through a shuffle: provably warp-uniform, so TMEM/SMEM addresses
  // derived from it live in uniform registers (no R2UR per tcgen05 op)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
#endif
  const int64_t ntiles = (a.rows + 127) / 128;
  const int64_t npairs = (ntiles + NG - 1) / NG;
  const bool x_bulk_ok = ((reinterpret_cast<uintptr_t>(a.x) & 15u) == 0);

  // ---- setup ----
  if (threadIdx.x == 0) {
    TBN_TRACE(0);
    for (int g = 0; g < NG; ++g) {
      for (int i = 0; i < CF::NSLOT; ++i) ptx::mbar_init(&bars->wfull[g][i], 1);
      ptx::mbar_init(&bars->xfull[g], 1);
      ptx::mbar_init(&bars->dfull[g], 1);
    }
    ptx::mbar_init(&bars->cfull, 1);
    ptx::fence_mbar_init();
    ptx::mbar_arrive_expect_tx(&bars->cfull, CF::CONST_BYTES + CF::RES_BYTES);
    ptx::bulk_g2s(smem + SM::OFF_CONST, p.wimg, CF::CONST_BYTES, &bars->cfull);
    if constexpr (CF::RESIDENT) {
      ptx::bulk_g2s(smem + SM::OFF_RES, p.wimg + p.off_sh1, CF::B_SH1, &bars->cfull);
      ptx::bulk_g2s(smem + SM::OFF_RES + CF::B_SH1, p.wimg + p.off_sh2, CF::B_HID, &bars->cfull);
    }
  }
  if (warp == 0) ptx::tmem_alloc<CF::TCOLS>(&bars->tmem_base);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = bars->tmem_base;

  {
    // ======================= ROW GROUPS (thread = (row, column half)) ========
    const int g = warp >> 3;                  // row group
    const int half = (warp >> 2) & 1;         // 0: d columns, 1: a columns
    const int t = (warp & 3) * 32 + lane;     // row within tile == TMEM lane
    const uint32_t tg = tbase + (uint32_t)(g * CF::TCOLS_G) + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t tD = tg + CF::T_D, tA = tg + CF::T_A, tAL = tg + CF::T_AL;
    const uint32_t tXN = tg + CF::T_XN, tPR = tg + CF::T_PR, tAG = tg + CF::T_AG;
    const float* xs = reinterpret_cast<const float*>(smem + SM::OFF_X + g * CF::XSTAGE);
    float* ts = reinterpret_cast<float*>(smem + SM::OFF_T + g * CF::TSTAGE);
    const uint32_t bar_id = 1 + g;
    const bool issuer = ((warp & 7) == 0) && lane == 0;    // half 0, quarter 0, lane 0
    const bool flusher = ((warp & 7) == 4) && lane == 0;   // half 1, quarter 0, lane 0
    uint8_t* ring = smem + SM::OFF_RING + g * CF::NSLOT * CF::SLOT;
    // Issuer-only producer duties for this group: its own weight ring (block u
    // of the group's sequence lives in slot u % NSLOT) and its next x tile.
    auto issue_block = [&](uint32_t u) {
      const int64_t pr = (int64_t)blockIdx.x + (int64_t)(u / CF::NB) * gridDim.x;
      if (pr >= npairs || pr * NG + g >= ntiles) return;
      int kind, step;
      ring_block<CF>((int)(u % CF::NB), kind, step);
      const uint32_t bytes = block_bytes<CF>(kind);
      const int sl = (int)(u % CF::NSLOT);
      ptx::mbar_arrive_expect_tx(&bars->wfull[g][sl], bytes);
      ptx::bulk_g2s(ring + sl * CF::SLOT, p.wimg + block_offset<CF>(p, kind, step), bytes,
                    &bars->wfull[g][sl]);
    };
    auto issue_x = [&](int64_t pr) {
      if (pr >= npairs || pr * NG + g >= ntiles) return;
      const int64_t r0 = (pr * NG + g) * 128;
      const int64_t nr = a.rows - r0 < 128 ? a.rows - r0 : 128;
      const uint32_t bytes = x_bulk_ok ? (uint32_t)((nr * F * 4) & ~15ll) : 0u;
      if (bytes) {
        ptx::mbar_arrive_expect_tx(&bars->xfull[g], bytes);
        ptx::bulk_g2s(smem + SM::OFF_X + g * CF::XSTAGE, a.x + r0 * F, bytes, &bars->xfull[g]);
      } else {
        ptx::mbar_arrive(&bars->xfull[g]);
      }
    };
    uint32_t ring_used = 0;                   // issuing warp: ring blocks consumed
    uint32_t ring_issued = 0;                 // flusher: ring blocks seen (refill cursor)
    if (issuer) {
      issue_x(blockIdx.x);
      for (uint32_t u = 0; u < (uint32_t)CF::NSLOT; ++u) issue_block(u);
    }
    ptx::mbar_wait(&bars->cfull, 0);
    if (a.scale) {     // batch-statistics control: override the affine in this CTA's SMEM copy
      float* cw = reinterpret_cast<float*>(smem + SM::OFF_CONST);
      for (int f = threadIdx.x; f < F; f += blockDim.x) {
        cw[CF::C_SCALE + f] = a.scale[f];
        cw[CF::C_SHIFT + f] = a.shift[f];
      }
      ptx::named_bar_sync(13, CF::THREADS);
    }
    const float* scale = cst + CF::C_SCALE;
    const float* shift = cst + CF::C_SHIFT;
    uint32_t xphase = 0, dphase = 0;

    // Ping-pong token (FA4 style): the two row groups' CUDA-core segments (the
    // work between two GEMMs) strictly alternate, so each group's tcgen05 MMAs
    // run while the other group computes.  Named barrier 11+g = "group g may
    // run its next segment"; the other group arrives on it when its segment ends.
    // The token is held only across a segment's TMEM-load phase (released as
    // soon as the accumulator is in registers, or at the segment's end at the
    // latest), so one group's TMEM load latency overlaps the other group's math.
    bool paired = false;        // both groups have a tile in the current pair
    bool token_held = false;
    auto seg_acquire = [&](bool first_of_pair) {
      if (paired && !(g == 0 && first_of_pair)) ptx::named_bar_sync(11 + g, 512);
      token_held = paired;
    };
    auto seg_release = [&]() {
      if (token_held) ptx::named_bar_arrive(11 + (g ^ 1), 512);
      token_held = false;
    };
    // A is written (both halves) -> barrier -> one thread issues GEMM j of the
    // tile's sequence -> everyone waits for the accumulator.  `post` runs
    // between the barrier and the wait (overlaps the MMA).
    auto gemm = [&](int j, int64_t pair, auto&& post) {
      // The attentive segment (after an att GEMM, j = 4 + 5(s-1)) is latency-
      // bound (sparsemax iterations): both groups run theirs outside the token,
      // overlapping each other.  Both skip the same segment, so the alternation
      // parity is preserved.
      const bool after_att = (j >= 5) && ((j - 5) % 5 == 0);
      const bool is_att = (j >= 4) && ((j - 4) % 5 == 0);
      if (!after_att) seg_release();       // no-op if the GLU already released it
      const bool tr = (pair == blockIdx.x);
      const int gofs = g * 5000;
      if (tr && issuer) TBN_TRACE(gofs + 1000 + 4 * j);
      if (tr && flusher) TBN_TRACE(gofs + 2000 + 4 * j);
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::named_bar_sync(bar_id, 256);
      if (flusher) {
        // Producer duties, off the MMA-issue path.  Every GEMM before j has
        // completed (all threads waited on its accumulator), so the slot of
        // ring block u-1 is free: refill it with block u + NSLOT - 1.  At j == 0
        // every thread has read this tile's x: prefetch the group's next tile.
        int kind, step;
        gemm_of(j, kind, step);
        if (!is_resident<CF>(kind)) {
          const uint32_t u = ring_issued++;
          if (u >= 1) issue_block(u + CF::NSLOT - 1);
        }
        if (j == 0) issue_x(pair + gridDim.x);
      }
      if ((warp & 7) == 0) {                     // the group's issuing warp, converged
        if (tr && issuer) TBN_TRACE(gofs + 1001 + 4 * j);
        ptx::tc_fence_after();
        int kind, step;
        gemm_of(j, kind, step);
        const bool res = is_resident<CF>(kind);
        uint32_t bsm;
        uint32_t u = 0;
        if (res) {
          bsm = ptx::smem_u32(smem + SM::OFF_RES + (kind == 0 ? 0 : CF::B_SH1));
        } else {
          u = ring_used++;
          ptx::mbar_wait(&bars->wfull[g][u % CF::NSLOT], (u / CF::NSLOT) & 1u);
          bsm = ptx::smem_u32(ring + (u % CF::NSLOT) * CF::SLOT);
        }
        if (kind == 0) issue_gemm<CF, K1, CF::N2>(tD, tA, tAL, bsm);
        else if (kind == 4) issue_gemm<CF, CF::KATT, CF::FN>(tD, tA, tAL, bsm);
        else issue_gemm<CF, CF::KHID, CF::N2>(tD, tA, tAL, bsm);
        ptx::mma_commit(&bars->dfull[g]);
        if (tr && issuer) TBN_TRACE(gofs + 1002 + 4 * j);
      }
      post();
      // take the token first: while the other group computes, this group's
      // threads sleep in bar.sync instead of spinning on the mbarrier
      if (!is_att) seg_acquire(false);
      // one warp polls the accumulator barrier; the rest sleep in bar.sync
      if ((warp & 7) == 0) ptx::mbar_wait(&bars->dfull[g], dphase);
      if (tr && issuer) TBN_TRACE(gofs + 3500 + j);
      dphase ^= 1;
      ptx::named_bar_sync(bar_id, 256);
      ptx::tc_fence_after();
      if (tr && issuer) TBN_TRACE(gofs + 1003 + 4 * j);
    };
    auto nopost = [] {};

    // GLU epilogue for this half's H/2 output columns (lin | gate blocks of D).
    // Host-folded constants (tc_pack): gate columns carry -log2(e), residual
    // blocks' linear columns carry sqrt(.5); b = [b_lin' (H) | -log2e*b_gate (H)].
    //   e = 2^(gate'+nb) = exp(-u_gate);  sigma = 1/(1+e)  (one rcp per pair:
    //   q = 1/(d0 d1), sigma0 = d1 q, sigma1 = d0 q);  out = (lin'+b')*sigma [+ sqrt(.5)*prev]
    auto glu = [&](bool residual, float (&prev)[HH]) {
      constexpr int CW = HH < 32 ? HH : 32;
      const int c0 = half * HH;
#pragma unroll
      for (int j0 = 0; j0 < HH; j0 += CW) {
        float lin[CW], gate[CW];
        tmem_load_n<CW>(tD + c0 + j0, lin);
        tmem_load_n<CW>(tD + H + c0 + j0, gate);
        ptx::tmem_ld_wait();
        seg_release();
#pragma unroll
        for (int i = 0; i < CW; i += 2) {
          // D already holds lin' + b' and gate' + b' (bias row in B, ones in A)
          const float a0 = fminf(gate[i], 63.0f), a1 = fminf(gate[i + 1], 63.0f);
          const float2 d = __fadd2_rn(f2(ex2_approx(a0), ex2_approx(a1)), f2(1.0f, 1.0f));
          const float q = rcp_approx(d.x * d.y);
          const float2 sg = __fmul2_rn(f2(d.y, d.x), f2(q, q));
          float2 o;
          if (residual) {
            const float2 rp = __fmul2_rn(f2(prev[j0 + i], prev[j0 + i + 1]), f2(kR, kR));
            o = __ffma2_rn(f2(lin[i], lin[i + 1]), sg, rp);
          } else {
            o = __fmul2_rn(f2(lin[i], lin[i + 1]), sg);
          }
          prev[j0 + i] = o.x;
          prev[j0 + i + 1] = o.y;
        }
      }
    };
    // ones column of the hidden GEMMs' A (cols [H, H+8) = 1,0,..,0), rewritten
    // after each shared1 GEMM (whose A used those columns for features/ones)
    auto store_hidden_ones = [&]() {
      if (half == 1) {
        float v[CF::KG];
#pragma unroll
        for (int i = 0; i < CF::KG; ++i) v[i] = i == 0 ? 1.0f : 0.0f;
        store_a<CF, CF::KG>(tA + acol<CF>(H), tAL + acol<CF>(H), v);
      }
    };
    auto store_half = [&](const float (&v)[HH]) {     // A elements [half*H/2, +H/2)
      store_a_all<CF, HH>(tA + acol<CF>(half * HH), tAL + acol<CF>(half * HH), v);
    };
    // Row staging -> global: dense mode = TMA bulk store (+ coalesced tail),
    // transpose mode = cooperative coalesced stores.  Call after a group barrier.
    auto flush_rows = [&](float* dst, int nrows) {
      if constexpr (CF::DENSE_IO) {
        const int ne = nrows * F;
        const bool al = ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0);
        const int nb = al ? ((ne * 4) & ~15) / 4 : 0;
        if (flusher && nb > 0) {
          ptx::bulk_s2g(dst, ts, (uint32_t)nb * 4u);
          ptx::bulk_commit();
        }
        for (int e = nb + threadIdx.x % 256; e < ne; e += 256) dst[e] = ts[e];
      } else {
        for (int e = (int)(threadIdx.x % 256); e < nrows * F; e += 256) {
          const int rr = e / F, ff = e - rr * F;
          dst[e] = ts[ff * 129 + rr];
        }
      }
    };
    auto claim_ts = [&]() {      // previous readers (incl. a bulk store) done with ts
      if constexpr (CF::DENSE_IO) {
        if (flusher) ptx::bulk_wait_read0();
      }
      ptx::named_bar_sync(bar_id, 256);
    };
    // half 0 -> half 1 hand-off with the partner warp of the same lane quarter
    // (the other column half): double-buffered by parity, one 64-thread
    // barrier each.  Slot (par, 0) carries (max z, tau); slot (par, 1).x carries
    // the step's eta, written before the attentive GEMM's barrier.
    float4* xb4 = reinterpret_cast<float4*>(smem + SM::OFF_XCH) + g * 512;
    const uint32_t pair_bar = 3 + g * 4 + (warp & 3);
    uint32_t xpar = 0;
    auto send_tau = [&](float zmax, float tau) {
      xb4[(xpar * 2) * 128 + t] = make_float4(zmax, tau, 0.0f, 0.0f);
      ptx::named_bar_sync(pair_bar, 64);
      xpar ^= 1;
    };
    auto recv_tau = [&]() -> float2 {
      ptx::named_bar_sync(pair_bar, 64);
      const float4 o = xb4[(xpar * 2) * 128 + t];
      xpar ^= 1;
      return f2(o.x, o.y);
    };
    auto eta_slot = [&]() -> float& {
      return reinterpret_cast<float*>(xb4 + (xpar * 2 + 1) * 128 + t)[0];
    };
    auto ts_at = [&](int f) -> float& {
      if constexpr (CF::DENSE_IO) return ts[t * F + f];
      else return ts[f * 129 + t];
    };

    for (int64_t pair = blockIdx.x; pair < npairs; pair += gridDim.x) {
      const int64_t tile = pair * NG + g;
      if (tile >= ntiles) continue;
      const int64_t r0 = tile * 128;
      const int nrows = (int)(a.rows - r0 < 128 ? a.rows - r0 : 128);
      const bool valid = t < nrows;
      const int64_t row = r0 + t;
      int j = 0;                                 // GEMM index within the tile

      // ---- x tile (TMA-staged): xn = (x - mean) * rsqrt(var + eps) for this
      // half's features (network.py:118-120); prior = 1; agg = 0 ----
      const bool trt = (g == 0 && pair == blockIdx.x && issuer);
      if (trt) TBN_TRACE(3090);
      ptx::mbar_wait(&bars->xfull[g], xphase);
      xphase ^= 1;
      if (trt) TBN_TRACE(3091);
#ifdef TBN_NO_TOKEN       // ablation: free-running groups (measured slower)
      paired = false;
#else
      paired = (NG == 2) && (pair * NG + 1 < ntiles);
#endif
      seg_acquire(true);
      {
        const int ne = nrows * F;
        const int nbulk = x_bulk_ok ? ((ne * 4) & ~15) / 4 : 0;
        const bool full_tile = (nbulk == 128 * F);
        if constexpr (!CF::DENSE_IO) {
          claim_ts();
          for (int e = (int)(threadIdx.x % 256); e < 128 * F; e += 256) {
            float v = 0.0f;
            if (e < nbulk) v = xs[e];
            else if (e < ne) v = a.x[r0 * F + e];
            const int rr = e / F, ff = e - rr * F;
            ts[ff * 129 + rr] = v;
          }
          ptx::named_bar_sync(bar_id, 256);
        }
        if constexpr (CF::DENSE_IO) {
          if (!full_tile) {     // the last, partial tile: complete the staging tile in SMEM
            float* xw = const_cast<float*>(xs);
            for (int e = nbulk + (int)(threadIdx.x % 256); e < 128 * F; e += 256)
              xw[e] = e < ne ? __ldg(a.x + r0 * F + e) : 0.0f;
            ptx::fence_async_shared();          // generic writes before the next TMA refill
            ptx::named_bar_sync(bar_id, 256);
          }
        }
        int bad = 0;
        auto xn_half = [&](auto hc) {
          constexpr int HB = decltype(hc)::value;
          chunked<KH>([&](auto o, auto l) {
            constexpr int O = decltype(o)::value, L = decltype(l)::value;
            constexpr int FB = HB * KH + O;                          // first feature
            constexpr int LF = (FB + L <= F) ? L : (FB < F ? F - FB : 0);
            float xn[L], one[L];
#pragma unroll
            for (int i = 0; i < L; ++i) {
              const int f = FB + i;
              one[i] = 1.0f;
              if (f < F) {
                float xv;
                if constexpr (CF::DENSE_IO) xv = xs[t * F + f];
                else xv = ts[f * 129 + t];
                bad |= !isfinite(xv);
                // normalized input: (x - 0) * 1 == x exactly; no branch per element
                const float sh = a.normalized ? 0.0f : shift[f];
                const float sc = a.normalized ? 1.0f : scale[f];
                xn[i] = (xv - sh) * sc;
              } else {
                xn[i] = (f == F) ? 1.0f : 0.0f;                       // ones column (bias row)
              }
            }
            if constexpr (LF > 0) {
              tmem_store_n<LF>(tXN + FB, xn);
              tmem_store_n<LF>(tPR + FB, one);
            }
            store_a<CF, L>(tA + acol<CF>(FB), tAL + acol<CF>(FB), xn);
          });
        };
        if (half == 0) {
          xn_half(std::integral_constant<int, 0>{});
          chunked<F>([&](auto o, auto l) {                           // agg = 0 (owned by half 0)
            constexpr int O = decltype(o)::value, L = decltype(l)::value;
            float zero[L];
#pragma unroll
            for (int i = 0; i < L; ++i) zero[i] = 0.0f;
            tmem_store_n<L>(tAG + O, zero);
          });
        } else {
          xn_half(std::integral_constant<int, 1>{});
        }
        if (valid && bad && a.err_flag) raise_flag(a.err_flag);
      }
      if (trt) TBN_TRACE(3092);
      float prev[HH];
      // half 0: the head is linear, so logits = sum_s relu(d_s) @ head_W + b
      // (network.py:244, :253) accumulates per step: C registers instead of n_d
      float lacc[C];
#pragma unroll
      for (int c = 0; c < C; ++c) lacc[c] = 0.0f;
      bool all_eta_zero = true;

      // feature transformer (network.py:124-141): 4 GEMM+GLU blocks
      auto transform = [&](int step, auto&& post_first) {
        gemm(j++, pair, post_first);
        glu(false, prev);                                            // g1 = GLU(u1)
        store_half(prev);
        store_hidden_ones();
        gemm(j++, pair, nopost);
        glu(true, prev);                                             // g2
        store_half(prev);
        gemm(j++, pair, nopost);
        glu(true, prev);                                             // g3
        store_half(prev);
        gemm(j++, pair, nopost);
        glu(true, prev);                                             // g4 = f
      };

      // d = relu(f[:, :n_d]); d_sum += d; eta = sum(d); agg += eta*m
      // (network.py:241-245) for the step just finished (half 0 owns d, agg).
      // Runs in the next attentive GEMM's shadow (its post hook).
      bool agg_pending = false;
      // eta = sum(d) and d_sum (half 0, which holds d); the agg weights with the
      // importance-fallback bookkeeping: while every eta so far is 0, agg holds
      // sum_s m instead (needed only for the fallback, network.py:259-261, which
      // fires exactly then); the first eta > 0 resets it to eta*m, identical to
      // the reference's sum.  Both halves track all_eta_zero from the same eta.
      auto step_eta = [&]() -> float {
        float eta = 0.0f;
#pragma unroll
        for (int i = 0; i < HH; ++i) {
          const float d = fmaxf(prev[i], 0.0f);
#pragma unroll
          for (int c = 0; c < C; ++c) lacc[c] = fmaf(d, cst[CF::C_HW + i * C + c], lacc[c]);
          eta += d;
        }
        return eta;
      };
      auto agg_apply = [&](float eta) {
        const bool reset = all_eta_zero && eta > 0.0f;
        const float w = all_eta_zero ? (eta > 0.0f ? eta : 1.0f) : eta;
        all_eta_zero = all_eta_zero && !(eta > 0.0f);
        chunked<F>([&](auto o, auto l) {
          constexpr int O = decltype(o)::value, L = decltype(l)::value;
          float ag[L];
          tmem_load_n<L>(tAG + O, ag);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < L; ++i) ag[i] = fmaf(w, ts_at(O + i), reset ? 0.0f : ag[i]);
          tmem_store_n<L>(tAG + O, ag);
        });
      };
      // Under the attentive GEMM (its post hook): half 0 finishes the previous
      // step's d (network.py:241-244) and hands eta to half 1, which applies
      // agg += eta*m (network.py:245) while half 0 runs the tau search.
      auto agg_post = [&]() {
        if (half != 0 || !agg_pending) return;
        agg_pending = false;
        const float eta = step_eta();
        eta_slot() = eta;
        all_eta_zero = all_eta_zero && !(eta > 0.0f);
      };
      auto agg_half1 = [&]() {
        if (!agg_pending) return;
        agg_pending = false;
        agg_apply(eta_slot());
      };

      transform(0, nopost);                                           // network.py:226-227
      for (int s = 1; s <= S; ++s) {
        // A <- a = f[:, n_d:]  (half 1 owns it)
        if (half == 1) {
          float av[CF::KATT];
#pragma unroll
          for (int k = 0; k < CF::KATT; ++k) av[k] = k < NA ? prev[k] : (k == NA ? 1.0f : 0.0f);
          store_a_all<CF, CF::KATT>(tA, tAL, av);
        }
        gemm(j++, pair, agg_post);          // previous step's d/eta under the att MMA
        const bool trs = (g == 0 && pair == blockIdx.x && issuer);
        if (trs) TBN_TRACE(3000 + 8 * s);
        // attentive FC + prior + sparsemax (network.py:233-236, sparsemax.py:13-41),
        // features split between the two halves; the row's (max, sum, count)
        // reductions are combined through SMEM with the partner warp (a 64-thread
        // barrier per exchange).  a+b == b+a in IEEE, so both halves hold
        // bitwise-identical combined values and take identical decisions.
        auto attentive = [&](auto hc) {
          constexpr int HV = decltype(hc)::value;
          constexpr int HB = HV * KH;                              // first own feature
          constexpr int FE = (HB + KH < F) ? HB + KH : F;
          constexpr int NF = FE > HB ? FE - HB : 0;               // own features
          constexpr int NFA = NF > 0 ? NF : 1;
          // half 0 holds the whole row's z (it runs the tau search alone);
          // half 1 only its own features.
          constexpr int NZ = HV == 0 ? F : NF;
          constexpr int ZB = HV == 0 ? 0 : HB;                      // z[i] <-> feature ZB + i
          float z[NZ > 0 ? NZ : 1], pr[NZ > 0 ? NZ : 1], xnv[NFA];
          if constexpr (NZ > 0) {
            tmem_load_n<NZ>(tD + ZB, z);
            tmem_load_n<NZ>(tPR + ZB, pr);
            ptx::tmem_ld_wait();
          }
#pragma unroll
          for (int i = 0; i < NZ; ++i) z[i] = pr[i] * z[i];         // network.py:233-235 (bias in D)
          if constexpr (NF > 0) tmem_load_n<NF>(tXN + HB, xnv);     // lands during the search
          float zmax = -INFINITY, tau = 0.0f;
          if constexpr (HV == 0) {
            float zsum = 0.0f;
#pragma unroll
            for (int i = 0; i < F; ++i) {
              zmax = fmaxf(zmax, z[i]);
              zsum += z[i];
            }
#pragma unroll
            for (int i = 0; i < F; ++i) z[i] -= zmax;               // sparsemax.py:32
            if (trs) TBN_TRACE(3001 + 8 * s);
            // tau: Michelot's fixed point tau <- (sum_{z>tau} z - 1) / |{z > tau}|,
            // monotone from any lower bound of tau*; its support equals the
            // reference's sort/cumsum/count k (sparsemax.py:33-39).  Start from
            // max(-1, (sum z - 1)/F) (the max alone; all elements), nudged down
            // by 2^-20 relative so rounding cannot push it above tau*.
            const float bound = (zsum - (float)F * zmax - 1.0f) * (1.0f / (float)F);
            tau = fmaxf(-1.0f, bound - 9.5367431640625e-07f * fmaxf(1.0f, fabsf(bound)));
            float cnt_prev = (float)(F + 1);
            for (int it = 0; it <= F; ++it) {
              float2 sa = f2(0.0f, 0.0f), ca = f2(0.0f, 0.0f), sb = f2(0.0f, 0.0f), cb = f2(0.0f, 0.0f);
#pragma unroll
              for (int i = 0; i + 1 < F; i += 2) {
                const float2 m = f2(z[i] > tau ? 1.0f : 0.0f, z[i + 1] > tau ? 1.0f : 0.0f);
                if ((i / 2) % 2 == 0) {
                  sa = __ffma2_rn(m, f2(z[i], z[i + 1]), sa);
                  ca = __fadd2_rn(ca, m);
                } else {
                  sb = __ffma2_rn(m, f2(z[i], z[i + 1]), sb);
                  cb = __fadd2_rn(cb, m);
                }
              }
              const float2 s2 = __fadd2_rn(sa, sb), c2 = __fadd2_rn(ca, cb);
              float sm = s2.x + s2.y, c = c2.x + c2.y;
              if constexpr (F % 2) {
                const float m = z[F - 1] > tau ? 1.0f : 0.0f;
                sm = fmaf(m, z[F - 1], sm);
                c += m;
              }
              if (c >= cnt_prev) break;
              cnt_prev = c;
              tau = __fdividef(sm - 1.0f, c);                         // sparsemax.py:39
            }
            __syncwarp();                     // lanes left the search at different passes
            send_tau(zmax, tau);                                     // -> half 1
          } else {
            agg_half1();                                             // in the tau search's shadow
            const float2 o = recv_tau();
            zmax = o.x;
            tau = o.y;
#pragma unroll
            for (int i = 0; i < NZ; ++i) z[i] -= zmax;
          }
          if (trs) TBN_TRACE(3002 + 8 * s);
          ptx::tmem_ld_wait();                                       // xnv
          claim_ts();
          if (trs) TBN_TRACE(3003 + 8 * s);
          // own features: mask, prior update, xm -> A (network.py:237-238, :246);
          // A elements [HB, HB + KH) incl. the ones column and zero padding up to K1
          chunked<KH>([&](auto o, auto l) {
            constexpr int O = decltype(o)::value, L = decltype(l)::value;
            constexpr int FB = HB + O;
            constexpr int LF = (FB + L <= F) ? L : (FB < F ? F - FB : 0);
            constexpr int ZO = FB - ZB;                               // index into z / pr
            float prn[L], xm[L];
#pragma unroll
            for (int i = 0; i < L; ++i) {
              const int f = FB + i;
              if (f < F) {
                const float m = fmaxf(z[ZO + i] - tau, 0.0f);         // sparsemax.py:40
                prn[i] = pr[ZO + i] * (p.gamma - m);                  // network.py:237
                xm[i] = m * xnv[O + i];                               // network.py:238
                ts_at(f) = m;
              } else {
                prn[i] = 0.0f;
                xm[i] = (f == F) ? 1.0f : 0.0f;                       // ones column (bias row)
              }
            }
            if constexpr (LF > 0) tmem_store_n<LF>(tPR + FB, prn);
            store_a<CF, L>(tA + acol<CF>(FB), tAL + acol<CF>(FB), xm);
          });
          if (trs) TBN_TRACE(3004 + 8 * s);
        };
        if (half == 0) attentive(std::integral_constant<int, 0>{});
        else attentive(std::integral_constant<int, 1>{});
        if constexpr (CF::DENSE_IO) ptx::fence_async_shared();
        // shared1 GEMM of step s; masks[s-1] tile goes out meanwhile
        transform(s, [&] {
          if (a.masks) flush_rows(a.masks + ((int64_t)(s - 1) * a.rows + r0) * F, nrows);
        });
        agg_pending = true;
      }
      if (agg_pending && half == 0) agg_apply(step_eta());   // the last step's (no att GEMM follows)
      agg_pending = false;
      if (trt) TBN_TRACE(3100);
      // ---- head + softmax + argmax (network.py:253-256, :279), importance
      // = agg / sum(agg) or mean_s(masks) (network.py:258-261): half 0 ----
      float ag[F];
      float div = 1.0f, rdiv = 1.0f;
      if (half == 0) {
        float lg[C];
        float lmax = -INFINITY;
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
        tmem_load_n<F>(tAG, ag);
        ptx::tmem_ld_wait();
        float tot = 0.0f;
#pragma unroll
        for (int f = 0; f < F; ++f) tot += ag[f];
        div = all_eta_zero ? (float)S : tot;
        rdiv = __frcp_rn(div);
      }
      if (trt) TBN_TRACE(3101);
      claim_ts();
      if (trt) TBN_TRACE(3102);
      if (half == 0) {
#pragma unroll
        for (int f = 0; f < F; ++f) ts_at(f) = ag[f] * rdiv;
      }
      if constexpr (CF::DENSE_IO) ptx::fence_async_shared();
      ptx::named_bar_sync(bar_id, 256);
      if (a.importance) flush_rows(a.importance + r0 * F, nrows);
      if (trt) TBN_TRACE(3103);
      seg_release();
      if (paired && g == 0) ptx::named_bar_sync(11, 512);   // consume group 1's last handoff
    }
    if constexpr (CF::DENSE_IO) {
      if (flusher) ptx::bulk_wait0();
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TBN_TRACE(2);
  if (warp == 0) ptx::tmem_dealloc<CF::TCOLS>(tbase);
}

}  // namespace tc
}  // namespace tbn
