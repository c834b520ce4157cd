// ws_probe.cu — tcgen05.mma.ws (weight-stationary) with M=32 on sm_100a:
// (1) where do the 32 accumulator rows land in TMEM, and does the D / A lane
//     field select the warp quarter (so each warp can own an independent
//     32-row MMA chain in its own lanes)?
// (2) issue->completion latency of a K=48 chain (3 MMAs) + commit, for
//     M=128 (A in TMEM) against ws M=32 issued by 1 or 4 warps at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2510_19689_b200/csrc ws_probe.cu -o ws_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
using namespace tbn::ptx;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int K = 16, N = 64;

__device__ __forceinline__ void mma_ws_f16_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.ws.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ws_f16_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

// layout probe: A[r][k] = (r+1) if k == 0 else 0; B[n][k] = (n+1) if k == 0 else 0
// so D[r][n] = (r+1)(n+1).  mode 0: ws M=32 SS; 1: ws M=32 TS; 2: ws M=64 TS.
// Each warp q issues its own MMA with D / A lane field 32q (mode 0/1); mode 2
// only warp 0 issues with lane field 0.
__global__ void layout(float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  uint8_t* sA = smem;                 // 32 rows x K bf16, canonical, per warp 1 KB
  uint8_t* sB = smem + 4096;          // N rows x K bf16
  auto off = [&](int r, int k) -> uint32_t { return (r / 8) * ((K / 8) * 128) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2; };
  for (int k = 0; k < K; ++k) *(__nv_bfloat16*)(sA + warp * 1024 + off(lane, k)) = __float2bfloat16(k == 0 ? (float)(lane + 1) : 0.f);
  for (int idx = t; idx < N * K; idx += 128) { int n = idx / K, k = idx % K; *(__nv_bfloat16*)(sB + off(n, k)) = __float2bfloat16(k == 0 ? (float)(n + 1) : 0.f); }
  if (warp == 0) tmem_alloc<256>(&tbase);
  if (t < 4) { mbar_init(&bar[t], 1); }
  if (t == 0) fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t tq = tb + ((uint32_t)(warp * 32) << 16);
  {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(-7.0f);
    for (int c = 0; c < 256; c += 16) TBN_TMEM_ST16(tq + c, r);
    // A in TMEM cols [128, 136): row = lane (+32 * warp for M=64 probing)
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) {
      const float rv = (float)(lane + 1 + (mode == 2 ? 32 * warp : 0));
      __nv_bfloat162 b = __floats2bfloat162_rn(i == 0 ? rv : 0.f, 0.f);
      a[i] = *(uint32_t*)&b;
    }
    TBN_TMEM_ST8(tq + 128, a);
    tmem_st_wait();
  }
  fence_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t M = mode == 2 ? 64 : 32;
  const uint32_t idesc = idesc_f32acc(kFmtBF16, M, N);
  const uint64_t bd = smem_desc(smem_u32(sB), 128u, (K / 8) * 128u);
  bool issuer = (mode == 2) ? (warp == 0) : true;
  if (issuer) {
    const uint32_t dq = (mode == 2) ? tb : tq;
    if (mode == 0) {
      const uint64_t ad = smem_desc(smem_u32(sA + warp * 1024), 128u, (K / 8) * 128u);
      mma_ws_f16_ss(dq, ad, bd, idesc, 0u);
    } else {
      mma_ws_f16_ts(dq, dq + 128, bd, idesc, 0u);
    }
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  {
    uint32_t r[16];
    for (int c = 0; c < 128; c += 16) {
      TBN_TMEM_LD16(tq + c, r);
      tmem_ld_wait();
      for (int i = 0; i < 16; ++i) D[t * 128 + c + i] = __uint_as_float(r[i]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tb);
}

// latency: nw warps each issue `reps` rounds of [3 MMAs (K = 48) -> commit ->
// wait] on their own D; M=128 (warp 0 only, A in TMEM) or ws M=32 per warp.
__global__ void latency(long long* out, int ws, int nw, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 16384; i += blockDim.x) smem[i] = 0;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (t < 4) mbar_init(&bar[t], 1);
  if (t == 0) fence_mbar_init();
  fence_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t tq = tb + ((uint32_t)(warp * 32) << 16);
  constexpr int KK = 48;
  const uint64_t bd = smem_desc(smem_u32(smem), 128u, (KK / 8) * 128u);
  long long t0 = clock64();
  if (ws ? (warp < nw) : (warp == 0)) {
    const uint32_t idesc = idesc_f32acc(kFmtBF16, ws ? 32 : 128, 64);
    const uint32_t d = ws ? tq : tb;
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      for (int k0 = 0; k0 < KK; k0 += 16) {
        if (ws) mma_ws_f16_ts(d, d + 128 + k0 / 2, bd + (uint64_t)k0, idesc, k0 > 0);
        else mma_f16_ts(d, d + 128 + k0 / 2, bd + (uint64_t)k0, idesc, k0 > 0);
      }
      mma_commit(&bar[warp]);
      mbar_wait(&bar[warp], ph);
      ph ^= 1;
    }
  }
  long long t1 = clock64();
  if ((t & 31) == 0) out[warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  float* dD;
  long long* dL;
  CK(cudaMalloc(&dD, 128 * 128 * 4));
  CK(cudaMalloc(&dL, 64));
  CK(cudaFuncSetAttribute(layout, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  CK(cudaFuncSetAttribute(latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  const char* names[3] = {"ws M=32 SS, per-warp lane field", "ws M=32 TS, per-warp lane field", "ws M=64 TS, warp 0 only"};
  for (int mode = 0; mode < 3; ++mode) {
    layout<<<1, 128, 65536>>>(dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    std::vector<float> D(128 * 128);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    printf("%s:\n", names[mode]);
    for (int lane = 0; lane < 128; lane += 8) {
      printf("  lane %3d:", lane);
      for (int c = 0; c < 128; c += 16) {
        const float v = D[lane * 128 + c + 1];   // column c+1: (r+1)(n+1) with n = c+1 -> r
        if (v == -7.0f) printf("    .   ");
        else printf(" %7.1f", v);
      }
      printf("\n");
    }
  }
  for (int ws = 0; ws < 2; ++ws)
    for (int nw = 1; nw <= 4; nw *= (ws ? 4 : 8)) {
      const int reps = 2000;
      latency<<<1, 128, 65536>>>(dL, ws, nw, reps);
      CK(cudaDeviceSynchronize());
      long long L[4];
      CK(cudaMemcpy(L, dL, sizeof(L), cudaMemcpyDeviceToHost));
      printf("latency %s nw=%d: %.1f cycles per K=48 round trip (warp 0)\n", ws ? "ws M=32" : "M=128 ", nw,
             (double)L[0] / reps);
    }
  return 0;
}
