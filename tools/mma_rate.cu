// Dev probe: tcgen05.mma kind::f16 issue rate for one CTA, M=128 x N x K=16,
// B in SMEM with SWIZZLE_NONE (canonical, LBO 128 B) vs SWIZZLE_128B (K-major,
// SBO 1024 B), A from TMEM (ts) or SMEM (ss).  Values are garbage (zeros):
// only the cycles per MMA are measured.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_19689_b200/csrc \
//        tools/mma_rate.cu -o /tmp/mma_rate && /tmp/mma_rate
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"
using namespace tbn;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;             // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

template <int N, bool SW, bool TS, int LAG = 0, bool LOAD = false>
__global__ void probe(long long* out, int iters, const uint8_t* g) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, cb[4], lb[2];
  // B: N rows x 64 K bf16 = N*128 B; A: 128 x 64 bf16 = 16 KB
  uint8_t* B = smem;
  uint8_t* A = smem + N * 128;
  for (int i = threadIdx.x; i < (N * 128 + 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) ptx::mbar_init(&cb[i], 1); ptx::mbar_init(&lb[0], 1); ptx::mbar_init(&lb[1], 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tbase);
  ptx::fence_async_shared();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tD = tbase, tA = tbase + 256;
  const uint32_t sB = ptx::smem_u32(B), sA = ptx::smem_u32(A);
  constexpr uint32_t idesc = ptx::idesc_f32acc(ptx::kFmtBF16, 128, N);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int k0 = 0; k0 < 64; k0 += 16) {
        const uint64_t bd = SW ? desc_sw128(sB + k0 * 2) : ptx::smem_desc(sB + k0 / 8 * 128, 128u, 8u * 128u);
        if (TS) {
          ptx::mma_f16_ts(tD, tA + k0 / 2, bd, idesc, 1u);
        } else {
          const uint64_t ad = SW ? desc_sw128(sA + k0 * 2) : ptx::smem_desc(sA + k0 / 8 * 128, 128u, 8u * 128u);
          if (ptx::elect_one()) ptx::mma_f16_ss(tD, ad, bd, idesc, 1u);
          __syncwarp();
        }
      }
      if (LOAD) {      // a 32 KB ring refill per chunk (TMA bulk, L2-resident source)
        if (threadIdx.x == 0) {
          if (it >= 2) ptx::mbar_wait(&lb[it & 1], ((it - 2) >> 1) & 1u);
          ptx::mbar_arrive_expect_tx(&lb[it & 1], 32768);
          ptx::bulk_g2s(smem + N * 128 + 16384 + (it & 1) * 32768, g + (size_t)(it % 64) * 32768, 32768, &lb[it & 1]);
        }
        __syncwarp();
      }
      if (LAG > 0) {   // the K3 issue pattern: commit per chunk, wait for chunk it-LAG
        ptx::mma_commit(&cb[it & 3]);
        if (it >= LAG) ptx::mbar_wait(&cb[(it - LAG) & 3], ((it - LAG) >> 2) & 1u);
      }
    }
    ptx::mma_commit(&bar);
    ptx::mbar_wait(&bar, 0);
    t1 = clock64();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tbase);
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

template <int N, bool SW, bool TS, int LAG = 0, bool LOAD = false>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = N * 128 + 16384 + 65536;
  uint8_t* g;
  cudaMalloc(&g, 64 << 15);
  cudaMemset(g, 0, 64 << 15);
  cudaFuncSetAttribute(probe<N, SW, TS, LAG, LOAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  probe<N, SW, TS, LAG, LOAD><<<1, 128, smem>>>(d, 10, g);
  probe<N, SW, TS, LAG, LOAD><<<1, 128, smem>>>(d, iters, g);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%-22s N=%3d cycles/MMA %.1f (floor %d)  %s\n", name, N, (double)h / (iters * 4), 128 * N / 256,
         cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(g);
}

int main() {
  run<256, false, true>("noswizzle ts");
  run<256, false, true, 1>("noswizzle ts lag1");
  run<256, false, true, 2>("noswizzle ts lag2");
  run<256, false, false, 1>("noswizzle ss lag1");
  run<256, false, true, 1, true>("noswizzle ts lag1 +tma");
  run<256, false, false, 1, true>("noswizzle ss lag1 +tma");
  run<256, true, true>("sw128 ts");
  run<256, false, false>("noswizzle ss");
  run<256, true, false>("sw128 ss");
  run<128, false, true>("noswizzle ts");
  run<128, true, true>("sw128 ts");
  run<64, false, true>("noswizzle ts");
  run<64, true, true>("sw128 ts");
  return 0;
}
