// synccheck_probe.cu — does compute-sanitizer synccheck accept named barriers
// with a thread count below blockDim while other warps wait at __syncthreads?
// mode 0: warps 0-3 loop on bar.sync 1,128; warps 4-15 go to __syncthreads.
// mode 1: every group of 4 warps loops on its own barrier (1 + g, 128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 synccheck_probe.cu -o synccheck_probe
#include <cstdio>
__global__ void k(int mode, int* out) {
  const int warp = threadIdx.x >> 5, g = warp >> 2;
  int acc = 0;
  if (mode == 1 || g == 0) {
    for (int i = 0; i < 8; ++i) {
      __syncwarp();
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(128) : "memory");
      acc += i;
    }
  }
  __syncthreads();
  out[threadIdx.x] = acc;
}
int main() {
  int* d;
  cudaMalloc(&d, 512 * 4);
  for (int mode = 0; mode < 2; ++mode) {
    k<<<1, 512>>>(mode, d);
    printf("mode %d: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  return 0;
}
