// kernel_aux.cu — the use_batch_stats negative control (network.py:212-216):
// per-column mean and population variance of THIS batch, in float64, turned
// into the same (scale, shift) affine the frozen-stats path uses.  It exists so
// that load_invariance_check's negative control (invariance.py:59,67-71) has a
// batch-dependent model to catch; production paths never set it.
#include "tbn_internal.h"

namespace tbn {
namespace {

__global__ void batch_stats_kernel(const float* __restrict__ x, int64_t rows, int F,
                                   float* __restrict__ scale, float* __restrict__ shift) {
  __shared__ double red[256];
  const int f = blockIdx.x;
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) s += (double)x[r * F + f];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double mean = red[0] / (double)rows;
  __syncthreads();
  double q = 0.0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
    double d = (double)x[r * F + f] - mean;
    q += d * d;
  }
  red[threadIdx.x] = q;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double var = red[0] / (double)rows;
    scale[f] = (float)(1.0 / sqrt(var + 1e-8));   // _NORM_EPS, network.py:27
    shift[f] = (float)mean;
  }
}

// Per-partition column means (stability.py:103-106: each partition's
// importance.mean(axis=0)): values (P*per, W) fp32 row-major, out (P, W) f64.
// Block = 32 columns x 8 row lanes; a warp reads 128 contiguous bytes of one
// row; float64 accumulation, fixed summation order (deterministic).
__global__ void partition_mean_kernel(const float* __restrict__ v, int64_t per, int W,
                                      double* __restrict__ out) {
  __shared__ double red[8][33];
  const int p = blockIdx.x, f = blockIdx.y * 32 + threadIdx.x;
  const float* base = v + (int64_t)p * per * W;
  double s = 0.0;
  if (f < W)
    for (int64_t r = threadIdx.y; r < per; r += 8) s += (double)base[r * W + f];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && f < W) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    out[(int64_t)p * W + f] = t / (double)per;
  }
}

}  // namespace

cudaError_t launch_partition_mean(const float* v, int64_t per, int partitions, int W, double* out,
                                  cudaStream_t stream) {
  partition_mean_kernel<<<dim3(partitions, (W + 31) / 32), dim3(32, 8), 0, stream>>>(v, per, W, out);
  return cudaGetLastError();
}

cudaError_t launch_batch_stats(const float* x, int64_t rows, int F, float* scale, float* shift,
                               cudaStream_t stream) {
  batch_stats_kernel<<<F, 256, 0, stream>>>(x, rows, F, scale, shift);
  return cudaGetLastError();
}

}  // namespace tbn
