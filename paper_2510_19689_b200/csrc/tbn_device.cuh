// tbn_device.cuh — device helpers shared by the TabNet kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tbn {

constexpr float kResidualScale = 0.70710678118654752440f;  // sqrt(0.5), network.py:29
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Accurate fp32 logistic: 1/(1+exp(-x)) (network.py:60) with full-precision expf.
__device__ __forceinline__ float sigmoid_accurate(float x) { return 1.0f / (1.0f + expf(-x)); }

// Sort-free sparsemax threshold for one row held by a warp (lane owns
// elements lane, lane+32, ...).  Mirrors sparsemax.py:13-41: shift by the row
// max (:32), then find tau with |support| = k and tau = (sum_support - 1)/k
// (:37-39).  Instead of sorting, Michelot's fixed point tau <- (sum_{z>tau} z - 1)/|{z>tau}|
// is iterated from tau0 = -1 (a lower bound: the max element alone); it is
// monotone and stops when the support no longer shrinks.  In exact arithmetic
// its support equals the reference's count-based k.
template <int kMaxPerLane>
__device__ __forceinline__ float warp_sparsemax_tau(const float (&zs)[kMaxPerLane], int n, int lane) {
  float tau = -1.0f;
  int cnt_prev = n + 1;
  for (int it = 0; it <= n; ++it) {
    float s = 0.f;
    int c = 0;
#pragma unroll
    for (int i = 0; i < kMaxPerLane; ++i) {
      int f = lane + 32 * i;
      if (f < n && zs[i] > tau) { s += zs[i]; ++c; }
    }
    s = warp_sum(s);
    c = warp_sum_i(c);
    if (c >= cnt_prev) break;
    cnt_prev = c;
    tau = (s - 1.0f) / (float)c;
  }
  return tau;
}

}  // namespace tbn
