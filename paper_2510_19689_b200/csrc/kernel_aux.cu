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

}  // namespace

cudaError_t launch_batch_stats(const float* x, int64_t rows, int F, float* scale, float* shift,
                               cudaStream_t stream) {
  batch_stats_kernel<<<F, 256, 0, stream>>>(x, rows, F, scale, shift);
  return cudaGetLastError();
}

}  // namespace tbn
