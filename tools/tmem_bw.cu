// tmem_bw.cu — TMEM load/store throughput microbenchmark (tcgen05.ld/st 32x32b).
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace tbn::ptx;

template <int NCOL>
__global__ void tmem_ld_bench(int iters, unsigned long long* cyc, float* sink, int mode) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&tb);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = tb + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64 % 512);
  float acc = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (mode == 0) {
      uint32_t r[16];
#pragma unroll
      for (int c = 0; c < NCOL; c += 16) {
        TBN_TMEM_LD16(base + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += __uint_as_float(r[i]);
      }
    } else if (mode == 1) {   // all loads then one wait
      uint32_t r[NCOL];
#pragma unroll
      for (int c = 0; c < NCOL; c += 16) {
        uint32_t* rr = r + c;
        TBN_TMEM_LD16(base + c, rr);
      }
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < NCOL; ++i) acc += __uint_as_float(r[i]);
    } else {                  // stores
      uint32_t r[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(acc + i);
#pragma unroll
      for (int c = 0; c < NCOL; c += 16) TBN_TMEM_ST16(base + c, r);
      tmem_st_wait();
      acc += 1.0f;
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  unsigned long long* d_cyc; float* sink;
  cudaMalloc(&d_cyc, 1024 * 8); cudaMalloc(&sink, 1024 * 1024 * 4);
  const int iters = 2000;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      tmem_ld_bench<64><<<1, warps * 32>>>(iters, d_cyc, sink, mode);
      cudaDeviceSynchronize();
      tmem_ld_bench<64><<<1, warps * 32>>>(iters, d_cyc, sink, mode);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c; cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
      double bytes = (double)iters * warps * 32 * 64 * 4;
      printf("mode=%s warps=%2d  cycles/iter=%.1f  bytes/cycle/SM=%.1f  %s\n",
             mode == 0 ? "ld16+wait" : mode == 1 ? "ld64,1wait" : "st16x4", warps,
             (double)c / iters, bytes / c, cudaGetErrorString(e));
    }
  return 0;
}
