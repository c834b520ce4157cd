// kernel_simt.cu — TBN_PREC_FP32: the whole TabNet forward (network.py:195-267)
// as ONE kernel on CUDA cores, one warp per row, fp32 FFMA.  This is the
// no-tensor-core precision reference of the engine (and the first correct
// path); the production path is kernel_tc.cu (tcgen05).
//
// Per-row results depend only on the row (fixed per-lane k-ascending FFMA
// chains, fixed butterfly reductions), never on batch size, warp or block
// position: the batch-invariance contract of network.py:11-14.
#include <cstdlib>
#include "tbn_internal.h"
#include "tbn_device.cuh"

namespace tbn {

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kMaxF = 512;
constexpr int kMaxN = 256;            // 2h
constexpr int kFPerLane = kMaxF / 32; // 16

// out[n] = b[n] + sum_k in[k] * W[k*N + n]   (x @ W + b, network.py:127 etc.)
__device__ __forceinline__ void warp_gemv(const float* __restrict__ in, int K,
                                          const float* __restrict__ W,
                                          const float* __restrict__ b, int N,
                                          float* __restrict__ out, int lane) {
  for (int n0 = 0; n0 < N; n0 += 128) {
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int k = 0; k < K; ++k) {
      float a = in[k];
      const float* wr = W + (size_t)k * N;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int n = n0 + lane + 32 * j;
        if (n < N) acc[j] = fmaf(a, __ldg(wr + n), acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + lane + 32 * j;
      if (n < N) out[n] = acc[j] + __ldg(b + n);
    }
  }
}

// g = GLU(u) [+ residual]:  u[:, :h] * sigmoid(u[:, h:])   (network.py:58-61, 131-137)
__device__ __forceinline__ void warp_glu(const float* __restrict__ u, float* g, int H,
                                         bool residual, int lane) {
  for (int j = lane; j < H; j += 32) {
    float v = u[j] * sigmoid_accurate(u[H + j]);
    g[j] = residual ? (v + g[j]) * kResidualScale : v;
  }
}

// Feature transformer (network.py:124-141): shared1 -> shared2 -> fc1_s -> fc2_s.
__device__ __forceinline__ void warp_transform(const SimtParams& p, const float* xin,
                                               float* u, float* g, int step, int lane) {
  const int H = p.H, N = 2 * p.H;
  warp_gemv(xin, p.F, p.sh1_W, p.sh1_b, N, u, lane);
  __syncwarp();
  warp_glu(u, g, H, false, lane);
  __syncwarp();
  warp_gemv(g, H, p.sh2_W, p.sh2_b, N, u, lane);
  __syncwarp();
  warp_glu(u, g, H, true, lane);
  __syncwarp();
  warp_gemv(g, H, p.fc1_W + (size_t)step * H * N, p.fc1_b + (size_t)step * N, N, u, lane);
  __syncwarp();
  warp_glu(u, g, H, true, lane);
  __syncwarp();
  warp_gemv(g, H, p.fc2_W + (size_t)step * H * N, p.fc2_b + (size_t)step * N, N, u, lane);
  __syncwarp();
  warp_glu(u, g, H, true, lane);
  __syncwarp();
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
tabnet_forward_simt(SimtParams p, ForwardArgs a) {
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = p.F, H = p.H, ND = p.ND, S = p.S, C = p.C;
  const int per_warp = 5 * F + 3 * H + ND + F;   // xn, prior, agg, m, xm | u(2H), g(H) | dsum | msum
  float* base = smem + (size_t)warp * per_warp;
  float* xn = base;
  float* prior = xn + F;
  float* agg = prior + F;
  float* m = agg + F;
  float* xm = m + F;
  float* u = xm + F;
  float* g = u + 2 * H;
  float* dsum = g + H;
  float* msum = dsum + ND;
  const float* scale = a.scale ? a.scale : p.scale;
  const float* shift = a.shift ? a.shift : p.shift;

  for (int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + warp; row < a.rows;
       row += (int64_t)gridDim.x * kWarpsPerBlock) {
    // -- load + validate + normalize (network.py:207-220) --
    int bad = 0;
    for (int f = lane; f < F; f += 32) {
      float xv = a.x[row * F + f];
      bad |= !isfinite(xv);
      xn[f] = a.normalized ? xv : (xv - shift[f]) * scale[f];
      prior[f] = 1.0f;
      agg[f] = 0.0f;
      msum[f] = 0.0f;
    }
    if (__any_sync(kFull, bad) && lane == 0 && a.err_flag) raise_flag(a.err_flag);
    for (int j = lane; j < ND; j += 32) dsum[j] = 0.0f;
    __syncwarp();
    // -- step 0 transformer; a = f0[:, n_d:] (network.py:226-227) --
    warp_transform(p, xn, u, g, 0, lane);
    for (int s = 1; s <= S; ++s) {
      // att = a @ W_att + b; z = prior * att (network.py:233-235)
      const float* Wa = p.att_W + (size_t)(s - 1) * p.NA * F;
      const float* ba = p.att_b + (size_t)(s - 1) * F;
      float zs[kFPerLane];
      float zmax = -INFINITY;
#pragma unroll
      for (int i = 0; i < kFPerLane; ++i) {
        int f = lane + 32 * i;
        float z = -INFINITY;
        if (f < F) {
          float acc = 0.0f;
          for (int k = 0; k < p.NA; ++k) acc = fmaf(g[ND + k], __ldg(Wa + (size_t)k * F + f), acc);
          z = prior[f] * (acc + __ldg(ba + f));
        }
        zs[i] = z;
        zmax = fmaxf(zmax, z);
      }
      zmax = warp_max(zmax);
#pragma unroll
      for (int i = 0; i < kFPerLane; ++i) zs[i] -= zmax;   // sparsemax.py:32
      const float tau = warp_sparsemax_tau(zs, F, lane);
      float* mask_out = a.masks ? a.masks + ((size_t)(s - 1) * a.rows + row) * F : nullptr;
#pragma unroll
      for (int i = 0; i < kFPerLane; ++i) {
        int f = lane + 32 * i;
        if (f < F) {
          float mv = fmaxf(zs[i] - tau, 0.0f);             // sparsemax.py:40
          m[f] = mv;
          prior[f] = prior[f] * (p.gamma - mv);            // network.py:237
          xm[f] = mv * xn[f];                              // network.py:238
          if (mask_out) mask_out[f] = mv;                  // network.py:246
          msum[f] += mv;
        }
      }
      __syncwarp();
      warp_transform(p, xm, u, g, s, lane);
      // d = relu(f[:, :n_d]); d_sum += d; eta = sum(d); agg += eta * m (network.py:241-245)
      float eta = 0.0f;
      for (int j = lane; j < ND; j += 32) {
        float d = fmaxf(g[j], 0.0f);
        dsum[j] += d;
        eta += d;
      }
      eta = warp_sum(eta);
      for (int f = lane; f < F; f += 32) agg[f] = fmaf(eta, m[f], agg[f]);
      __syncwarp();
    }
    // -- head + softmax (network.py:253-256) --
    float logit = -INFINITY;
    if (lane < C) {
      float acc = 0.0f;
      for (int k = 0; k < ND; ++k) acc = fmaf(dsum[k], __ldg(p.head_W + (size_t)k * C + lane), acc);
      logit = acc + __ldg(p.head_b + lane);
    }
    float lmax = warp_max(logit);
    float e = (lane < C) ? expf(logit - lmax) : 0.0f;
    float esum = warp_sum(e);
    float prob = e / esum;
    if (lane < C) {
      if (a.logits) a.logits[row * C + lane] = logit;
      if (a.probs) a.probs[row * C + lane] = prob;
    }
    // argmax, lowest index on ties
    float bv = (lane < C) ? prob : -INFINITY;
    int bi = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(kFull, bv, o);
      int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0 && a.pred) a.pred[row] = bi;
    // -- importance (network.py:258-261) --
    float tot = 0.0f;
    for (int f = lane; f < F; f += 32) tot += agg[f];
    tot = warp_sum(tot);
    if (a.importance) {
      for (int f = lane; f < F; f += 32)
        a.importance[row * F + f] = (tot > 0.0f) ? agg[f] / tot : msum[f] / (float)S;
    }
    __syncwarp();
  }
}

// ---- row-blocked variant: kBR rows per block in lockstep ------------------
// The GEMVs are done by the whole block for its 8 rows at once: a thread owns
// output column(s) n and accumulates them for several rows, so each weight
// element it loads feeds several rows' FFMA chains (the per-row kernel above
// reloads every weight for every row and is L1-bound).  Each output is still ONE
// fp32 FFMA chain over k ascending, then + bias: bit-for-bit the per-row
// kernel's arithmetic, so outputs are identical (batch invariance holds).
#ifndef TBN_SIMT_BR
#define TBN_SIMT_BR 16
#endif
constexpr int kBR = TBN_SIMT_BR;                       // rows per block == warps
constexpr int kBT = 32 * kBR;                          // threads per block

__device__ __forceinline__ int rup4(int v) { return (v + 3) & ~3; }

struct BlkLayout {   // per-row SMEM buffers, each 16-byte aligned
  int F4, H4, N4, ND4;
  int xn, prior, agg, m, msum, in, u, g, dsum, per_row;
  __device__ __forceinline__ BlkLayout(int F, int H, int ND) {
    F4 = rup4(F); H4 = rup4(H); N4 = rup4(2 * H); ND4 = rup4(ND);
    xn = 0; prior = xn + F4; agg = prior + F4; m = agg + F4; msum = m + F4; in = msum + F4;
    u = in + F4; g = u + N4; dsum = g + H4; per_row = dsum + ND4;
  }
};

// out_r[n] = b[n] + sum_k in_r[k] W[k*N + n] for the block's kBR rows.
// N >= kBT: thread t owns columns t + kBT j (NC of them) for all rows (RR = kBR);
// N <  kBT: thread t owns column t % N for rows t / N + (kBT / N) i (RR of them).
template <int NC, int RR>
__device__ __forceinline__ void blk_gemv_p2(float* smem_rows, int per_row, int in_off, int out_off,
                                         int K, const float* __restrict__ W,
                                         const float* __restrict__ b, int N) {
  const int t = threadIdx.x;
  const bool wide_n = N >= kBT;
  int col[NC], row[RR];
#pragma unroll
  for (int j = 0; j < NC; ++j) col[j] = wide_n ? t + kBT * j : t % N;
#pragma unroll
  for (int i = 0; i < RR; ++i) row[i] = wide_n ? i : t / N + (kBT / N) * i;
  float acc[NC][RR];
#pragma unroll
  for (int j = 0; j < NC; ++j)
#pragma unroll
    for (int i = 0; i < RR; ++i) acc[j][i] = 0.0f;
  const int K4 = K & ~3;
  for (int k = 0; k < K4; k += 4) {
    float w[4][NC];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int j = 0; j < NC; ++j) w[kk][j] = __ldg(W + (size_t)(k + kk) * N + col[j]);
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      const float4 a = *reinterpret_cast<const float4*>(smem_rows + row[i] * per_row + in_off + k);
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        acc[j][i] = fmaf(a.x, w[0][j], acc[j][i]);
        acc[j][i] = fmaf(a.y, w[1][j], acc[j][i]);
        acc[j][i] = fmaf(a.z, w[2][j], acc[j][i]);
        acc[j][i] = fmaf(a.w, w[3][j], acc[j][i]);
      }
    }
  }
  for (int k = K4; k < K; ++k) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const float wv = __ldg(W + (size_t)k * N + col[j]);
#pragma unroll
      for (int i = 0; i < RR; ++i) acc[j][i] = fmaf(smem_rows[row[i] * per_row + in_off + k], wv, acc[j][i]);
    }
  }
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const float bv = __ldg(b + col[j]);
#pragma unroll
    for (int i = 0; i < RR; ++i) smem_rows[row[i] * per_row + out_off + col[j]] = acc[j][i] + bv;
  }
}

// dispatch on N (2H for the transformer GEMVs, F for the attentive one)
template <int T>
struct GemvShape {
  __host__ __device__ static constexpr int nc(int n) { return n >= T ? n / T : 1; }
  __host__ __device__ static constexpr int rr(int n) { return n >= T ? kBR : kBR * n / T; }
};
__device__ __forceinline__ bool blk_gemv_pow2(float* sm, int per_row, int in_off, int out_off, int K,
                                           const float* W, const float* b, int N) {
  using G = GemvShape<kBT>;
  switch (N) {
    case 32: blk_gemv_p2<G::nc(32), G::rr(32)>(sm, per_row, in_off, out_off, K, W, b, N); return true;
    case 64: blk_gemv_p2<G::nc(64), G::rr(64)>(sm, per_row, in_off, out_off, K, W, b, N); return true;
    case 128: blk_gemv_p2<G::nc(128), G::rr(128)>(sm, per_row, in_off, out_off, K, W, b, N); return true;
    case 256: blk_gemv_p2<G::nc(256), G::rr(256)>(sm, per_row, in_off, out_off, K, W, b, N); return true;
    case 512: blk_gemv_p2<G::nc(512), G::rr(512)>(sm, per_row, in_off, out_off, K, W, b, N); return true;
    default: return false;
  }
}

// out_r[n] = b[n] + sum_k in_r[k] W[k*N + n] for the block's kBR rows (N <= kBT).
// The block's threads form G = kBT / N groups of N: thread t owns column t % N
// for rows t / N + G i (i < RR = ceil(kBR / G); rows past kBR are skipped).
template <int RR>
__device__ __forceinline__ void blk_gemv_any(float* smem_rows, int per_row, int in_off, int out_off,
                                         int K, const float* __restrict__ W,
                                         const float* __restrict__ b, int N) {
  const int t = threadIdx.x;
  const int G = kBT / N;
  if (t >= G * N) return;
  const int col = t % N, rg = t / N;
  int row[RR];
  bool ok[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) {
    row[i] = rg + G * i;
    ok[i] = row[i] < kBR;
    if (!ok[i]) row[i] = 0;
  }
  float acc[RR];
#pragma unroll
  for (int i = 0; i < RR; ++i) acc[i] = 0.0f;
  const int K4 = K & ~3;
  for (int k = 0; k < K4; k += 4) {
    float w[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) w[kk] = __ldg(W + (size_t)(k + kk) * N + col);
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      if (RR > 1 && !ok[i]) continue;
      const float4 a = *reinterpret_cast<const float4*>(smem_rows + row[i] * per_row + in_off + k);
      acc[i] = fmaf(a.x, w[0], acc[i]);
      acc[i] = fmaf(a.y, w[1], acc[i]);
      acc[i] = fmaf(a.z, w[2], acc[i]);
      acc[i] = fmaf(a.w, w[3], acc[i]);
    }
  }
  for (int k = K4; k < K; ++k) {
    const float wv = __ldg(W + (size_t)k * N + col);
#pragma unroll
    for (int i = 0; i < RR; ++i)
      if (ok[i]) acc[i] = fmaf(smem_rows[row[i] * per_row + in_off + k], wv, acc[i]);
  }
  const float bv = __ldg(b + col);
#pragma unroll
  for (int i = 0; i < RR; ++i)
    if (ok[i]) smem_rows[row[i] * per_row + out_off + col] = acc[i] + bv;
}

// N: 2H for the transformer GEMVs, F for the attentive one.  Powers of two take
// the compile-time mapping above (no predicates); other widths the general one.
__device__ __forceinline__ void blk_gemv_n(float* sm, int per_row, int in_off, int out_off, int K,
                                           const float* W, const float* b, int N) {
  if (blk_gemv_pow2(sm, per_row, in_off, out_off, K, W, b, N)) return;
  const int G = kBT / N;
  const int rr = (kBR + G - 1) / G;
  if (rr <= 1) blk_gemv_any<1>(sm, per_row, in_off, out_off, K, W, b, N);
  else if (rr <= 2) blk_gemv_any<2>(sm, per_row, in_off, out_off, K, W, b, N);
  else if (rr <= 4) blk_gemv_any<4>(sm, per_row, in_off, out_off, K, W, b, N);
  else if (rr <= 8) blk_gemv_any<8>(sm, per_row, in_off, out_off, K, W, b, N);
  else blk_gemv_any<16>(sm, per_row, in_off, out_off, K, W, b, N);
}

__device__ __forceinline__ void blk_glu(float* r, const BlkLayout& L, int H, bool residual, int lane) {
  for (int j = lane; j < H; j += 32) {
    float v = r[L.u + j] * sigmoid_accurate(r[L.u + H + j]);
    r[L.g + j] = residual ? (v + r[L.g + j]) * kResidualScale : v;
  }
}

// the feature transformer for the block's rows: in (per row at L.in, or xn) -> g
__device__ __forceinline__ void blk_transform(const SimtParams& p, float* sm, const BlkLayout& L,
                                              int in_off, int step, float* r, int lane) {
  const int H = p.H, N = 2 * H;
  blk_gemv_n(sm, L.per_row, in_off, L.u, p.F, p.sh1_W, p.sh1_b, N);
  __syncthreads();
  blk_glu(r, L, H, false, lane);
  __syncthreads();
  blk_gemv_n(sm, L.per_row, L.g, L.u, H, p.sh2_W, p.sh2_b, N);
  __syncthreads();
  blk_glu(r, L, H, true, lane);
  __syncthreads();
  blk_gemv_n(sm, L.per_row, L.g, L.u, H, p.fc1_W + (size_t)step * H * N, p.fc1_b + (size_t)step * N, N);
  __syncthreads();
  blk_glu(r, L, H, true, lane);
  __syncthreads();
  blk_gemv_n(sm, L.per_row, L.g, L.u, H, p.fc2_W + (size_t)step * H * N, p.fc2_b + (size_t)step * N, N);
  __syncthreads();
  blk_glu(r, L, H, true, lane);
  __syncthreads();
}

// MINB = 2 (two blocks per SM, registers capped at 64 with some spills) when the
// rows' SMEM allows it: +8-10% for HR/BLS; wide's 225 KB blocks run one per SM
template <int MINB>
__global__ void __launch_bounds__(kBT, MINB)
tabnet_forward_simt_blk(SimtParams p, ForwardArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = p.F, ND = p.ND, S = p.S, C = p.C;
  const BlkLayout L(F, p.H, ND);
  float* r = smem + warp * L.per_row;                  // this warp's row
  const float* scale = a.scale ? a.scale : p.scale;
  const float* shift = a.shift ? a.shift : p.shift;

  for (int64_t r0 = (int64_t)blockIdx.x * kBR; r0 < a.rows; r0 += (int64_t)gridDim.x * kBR) {
    const int64_t row = r0 + warp;
    const bool valid = row < a.rows;
    int bad = 0;
    for (int f = lane; f < L.F4; f += 32) {
      float xv = (valid && f < F) ? a.x[row * F + f] : 0.0f;
      if (valid && f < F) bad |= !isfinite(xv);
      r[L.xn + f] = (f < F && !a.normalized) ? (xv - shift[f]) * scale[f] : xv;
      r[L.prior + f] = 1.0f;
      r[L.agg + f] = 0.0f;
      r[L.msum + f] = 0.0f;
      r[L.in + f] = 0.0f;
    }
    if (__any_sync(kFull, bad) && lane == 0 && a.err_flag) raise_flag(a.err_flag);
    for (int j = lane; j < ND; j += 32) r[L.dsum + j] = 0.0f;
    __syncthreads();
    blk_transform(p, smem, L, L.xn, 0, r, lane);
    for (int s = 1; s <= S; ++s) {
      // att = a @ W_att + b for the block's rows (into m), z = prior * att
      blk_gemv_n(smem, L.per_row, L.g + ND, L.m, p.NA, p.att_W + (size_t)(s - 1) * p.NA * F,
                 p.att_b + (size_t)(s - 1) * F, F);
      __syncthreads();
      float zs[kFPerLane];
      float zmax = -INFINITY;
#pragma unroll
      for (int i = 0; i < kFPerLane; ++i) {
        const int f = lane + 32 * i;
        float z = -INFINITY;
        if (f < F) z = r[L.prior + f] * r[L.m + f];
        zs[i] = z;
        zmax = fmaxf(zmax, z);
      }
      zmax = warp_max(zmax);
#pragma unroll
      for (int i = 0; i < kFPerLane; ++i) zs[i] -= zmax;   // sparsemax.py:32
      const float tau = warp_sparsemax_tau(zs, F, lane);
      float* mask_out = (a.masks && valid) ? a.masks + ((size_t)(s - 1) * a.rows + row) * F : nullptr;
#pragma unroll
      for (int i = 0; i < kFPerLane; ++i) {
        const int f = lane + 32 * i;
        if (f < F) {
          const float mv = fmaxf(zs[i] - tau, 0.0f);             // sparsemax.py:40
          r[L.m + f] = mv;
          r[L.prior + f] = r[L.prior + f] * (p.gamma - mv);      // network.py:237
          r[L.in + f] = mv * r[L.xn + f];                        // network.py:238
          if (mask_out) mask_out[f] = mv;                        // network.py:246
          r[L.msum + f] += mv;
        }
      }
      __syncthreads();
      blk_transform(p, smem, L, L.in, s, r, lane);
      float eta = 0.0f;
      for (int j = lane; j < ND; j += 32) {
        const float d = fmaxf(r[L.g + j], 0.0f);
        r[L.dsum + j] += d;
        eta += d;
      }
      eta = warp_sum(eta);
      for (int f = lane; f < F; f += 32) r[L.agg + f] = fmaf(eta, r[L.m + f], r[L.agg + f]);
      __syncthreads();
    }
    float logit = -INFINITY;
    if (lane < C) {
      float acc = 0.0f;
      for (int k = 0; k < ND; ++k) acc = fmaf(r[L.dsum + k], __ldg(p.head_W + (size_t)k * C + lane), acc);
      logit = acc + __ldg(p.head_b + lane);
    }
    const float lmax = warp_max(logit);
    const float e = (lane < C) ? expf(logit - lmax) : 0.0f;
    const float esum = warp_sum(e);
    const float prob = e / esum;
    if (valid && lane < C) {
      if (a.logits) a.logits[row * C + lane] = logit;
      if (a.probs) a.probs[row * C + lane] = prob;
    }
    float bv = (lane < C) ? prob : -INFINITY;
    int bi = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(kFull, bv, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (valid && lane == 0 && a.pred) a.pred[row] = bi;
    float tot = 0.0f;
    for (int f = lane; f < F; f += 32) tot += r[L.agg + f];
    tot = warp_sum(tot);
    if (valid && a.importance) {
      for (int f = lane; f < F; f += 32)
        a.importance[row * F + f] = (tot > 0.0f) ? r[L.agg + f] / tot : r[L.msum + f] / (float)S;
    }
    __syncthreads();
  }
}

}  // namespace

static int rup4_host(int v) { return (v + 3) & ~3; }

size_t simt_smem_bytes(const SimtParams& p) {
  return (size_t)kWarpsPerBlock * (5 * p.F + 3 * p.H + p.ND + p.F) * sizeof(float);
}

bool simt_supported(int F, int H, int C) { return F <= kMaxF && 2 * H <= kMaxN && C <= 32; }

cudaError_t launch_simt(const SimtParams& p, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  if (!simt_supported(p.F, p.H, p.C)) return cudaErrorInvalidValue;
  size_t smem = simt_smem_bytes(p);
  struct SimtTag {};
  cudaError_t ce = smem_attr_once<SimtTag>((const void*)tabnet_forward_simt, 200 * 1024);
  if (ce != cudaSuccess) return ce;
  int64_t blocks_needed = (a.rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int64_t max_blocks = (int64_t)num_sms * 8;
  int grid = (int)(blocks_needed < max_blocks ? blocks_needed : max_blocks);
  if (grid < 1) grid = 1;
  static const bool per_row = getenv("TBN_SIMT_PER_ROW") != nullptr;   // A/B: the first kernel
  const int n2 = 2 * p.H;
  const int per_row_floats = 6 * rup4_host(p.F) + rup4_host(n2) + rup4_host(p.H) + rup4_host(p.ND);
  const size_t bsmem = (size_t)kBR * per_row_floats * sizeof(float);
  // (F < 32, Adult: the per-row kernel measured slightly faster)
  const bool blk_ok = !per_row && n2 <= kBT && p.F >= 32 && p.F <= kBT && p.ND % 4 == 0 &&
                      bsmem <= 227 * 1024;
  if (blk_ok) {
    const bool two = 2 * bsmem <= 227 * 1024;
    auto kern = two ? tabnet_forward_simt_blk<2> : tabnet_forward_simt_blk<1>;
    struct Blk1Tag {};
    struct Blk2Tag {};
    ce = smem_attr_once<Blk1Tag>((const void*)tabnet_forward_simt_blk<1>, 227 * 1024);
    if (ce == cudaSuccess) ce = smem_attr_once<Blk2Tag>((const void*)tabnet_forward_simt_blk<2>, 227 * 1024);
    if (ce != cudaSuccess) return ce;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBT, bsmem);
    const int64_t nb = (a.rows + kBR - 1) / kBR;
    const int64_t cap = (int64_t)num_sms * (per_sm > 0 ? per_sm : 1);
    const int bgrid = (int)(nb < cap ? nb : cap);
    kern<<<bgrid < 1 ? 1 : bgrid, kBT, bsmem, stream>>>(p, a);
    return cudaGetLastError();
  }
  tabnet_forward_simt<<<grid, kWarpsPerBlock * 32, smem, stream>>>(p, a);
  return cudaGetLastError();
}

// ---- standalone sparsemax (sparsemax.py:13-41), warp per row ----
namespace {
__global__ void sparsemax_rows_kernel(const float* __restrict__ z, int64_t rows, int n,
                                      float* __restrict__ out, int32_t* err_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    float zs[kFPerLane];
    float zmax = -INFINITY;
    int bad = 0;
#pragma unroll
    for (int i = 0; i < kFPerLane; ++i) {
      int f = lane + 32 * i;
      float v = (f < n) ? z[r * n + f] : -INFINITY;
      if (f < n) bad |= !isfinite(v);
      zs[i] = v;
      zmax = fmaxf(zmax, v);
    }
    if (__any_sync(kFull, bad) && lane == 0 && err_flag) raise_flag(err_flag);
    zmax = warp_max(zmax);
#pragma unroll
    for (int i = 0; i < kFPerLane; ++i) zs[i] -= zmax;
    float tau = warp_sparsemax_tau(zs, n, lane);
#pragma unroll
    for (int i = 0; i < kFPerLane; ++i) {
      int f = lane + 32 * i;
      if (f < n) out[r * n + f] = fmaxf(zs[i] - tau, 0.0f);
    }
  }
}
}  // namespace

// ---- standalone float64 sparsemax for the host helper API (any width) ----
// The reference helper (sparsemax.py:13-41) is float64 for any length; the
// public sparsemax() keeps that: warp per row, the row re-read from L1/L2 on
// every pass, Michelot's fixed point tau <- (sum_{z>tau} z - 1)/|{z>tau}| in
// float64 from the lower bound max(-1, (sum z - 1)/n) (its support equals the
// reference's sort/cumsum/count k; tau differs only by summation order).
namespace {
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__global__ void sparsemax_rows_f64_kernel(const double* __restrict__ z, int64_t rows, int n,
                                          double* __restrict__ out, int32_t* err_flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const double* zr = z + r * n;
    double zmax = -INFINITY, zsum = 0.0;
    int bad = 0;
    for (int f = lane; f < n; f += 32) {
      const double v = zr[f];
      bad |= !isfinite(v);
      zmax = fmax(zmax, v);
      zsum += v;
    }
    if (__any_sync(0xffffffffu, bad)) {
      if (lane == 0 && err_flag) raise_flag(err_flag);
      continue;
    }
    zmax = warp_max_d(zmax);                                   // sparsemax.py:32
    zsum = warp_sum_d(zsum) - (double)n * zmax;
    double tau = fmax(-1.0, (zsum - 1.0) / (double)n);
    tau -= 0x1p-40 * fmax(1.0, fabs(tau));
    double cnt_prev = (double)n + 1.0;
    for (int it = 0; it <= n; ++it) {
      double sm = 0.0, cn = 0.0;
      for (int f = lane; f < n; f += 32) {
        const double v = zr[f] - zmax;
        if (v > tau) { sm += v; cn += 1.0; }
      }
      sm = warp_sum_d(sm);
      cn = warp_sum_d(cn);
      if (cn >= cnt_prev) break;
      cnt_prev = cn;
      tau = (sm - 1.0) / cn;                                   // sparsemax.py:39
    }
    for (int f = lane; f < n; f += 32) out[r * n + f] = fmax(zr[f] - zmax - tau, 0.0);   // :40
  }
}
}  // namespace

cudaError_t launch_sparsemax_f64(const double* z, int64_t rows, int n, double* out, int32_t* err_flag,
                                 int num_sms, cudaStream_t stream) {
  int64_t blocks = (rows + 7) / 8;
  int64_t cap = (int64_t)num_sms * 16;
  int grid = (int)(blocks < cap ? blocks : cap);
  if (grid < 1) grid = 1;
  sparsemax_rows_f64_kernel<<<grid, 256, 0, stream>>>(z, rows, n, out, err_flag);
  return cudaGetLastError();
}

cudaError_t launch_sparsemax(const float* z, int64_t rows, int n, float* out, int32_t* err_flag,
                             int num_sms, cudaStream_t stream) {
  if (n > kMaxF) return cudaErrorInvalidValue;
  int64_t blocks = (rows + 7) / 8;
  int64_t cap = (int64_t)num_sms * 16;
  int grid = (int)(blocks < cap ? blocks : cap);
  if (grid < 1) grid = 1;
  sparsemax_rows_kernel<<<grid, 256, 0, stream>>>(z, rows, n, out, err_flag);
  return cudaGetLastError();
}

}  // namespace tbn
