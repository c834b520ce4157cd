// m64_probe.cu — where does a cta_group::1 M=64 tcgen05.mma (kind::f16) put
// its accumulator in TMEM, and can the D / A lane field select lanes 64..127?
// Measured on B200: rows 16j..16j+15 land in lanes 32j..32j+15 (the first 16
// lanes of each warp quarter) and the D lane field is ignored, so two M=64
// halves of a 128-row tile need twice the TMEM columns of one M=128 MMA — no
// use for K2's intra-group ping-pong idea.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2510_19689_b200/csrc m64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
using namespace tbn::ptx;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int K = 16, N = 64;
// mode 0: SS, D lane base 0; 1: SS, D lane base 64; 2: TS (A in TMEM lanes 64.., D lanes 64..)
__global__ void probe(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  uint8_t* sA = smem;                 // 64 rows x K bf16, canonical
  uint8_t* sB = smem + 64 * K * 2;    // N rows x K bf16
  auto off = [&](int r, int k) -> uint32_t { return (r / 8) * ((K / 8) * 128) + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2; };
  if (t < 64) for (int k = 0; k < K; ++k) *(__nv_bfloat16*)(sA + off(t, k)) = __float2bfloat16(A[t * K + k]);
  for (int idx = t; idx < N * K; idx += 128) { int n = idx / K, k = idx % K; *(__nv_bfloat16*)(sB + off(n, k)) = __float2bfloat16(B[k * N + n]); }
  if (warp == 0) tmem_alloc<128>(&tbase);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t tq = tb + ((uint32_t)(warp * 32) << 16);
  // sentinel everywhere in cols [0, 128)
  {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(-7.0f);
    for (int c = 0; c < 128; c += 16) TBN_TMEM_ST16(tq + c, r);
    if (mode == 2 && t >= 64) {   // A (TS) for rows t-64 at lanes 64.., cols [64, 72): bf16 pairs
      uint32_t a[8];
      for (int i = 0; i < 8; ++i) {
        __nv_bfloat162 b = __floats2bfloat162_rn(A[(t - 64) * K + 2 * i], A[(t - 64) * K + 2 * i + 1]);
        a[i] = *(uint32_t*)&b;
      }
      TBN_TMEM_ST8(tq + 64, a);
    }
    tmem_st_wait();
  }
  fence_async_shared();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t idesc = idesc_f32acc(kFmtBF16, 64, N);
    const uint64_t ad = smem_desc(smem_u32(sA), 128u, (K / 8) * 128u);
    const uint64_t bd = smem_desc(smem_u32(sB), 128u, (K / 8) * 128u);
    const uint32_t dlane = (mode == 0) ? 0u : (64u << 16);
    if (mode == 2) {
      mma_f16_ts(tb + dlane, tb + (64u << 16) + 64, bd, idesc, 0u);
    } else if (elect_one()) {
      mma_f16_ss(tb + dlane, ad, bd, idesc, 0u);
    }
    __syncwarp();
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[64];
  {
    uint32_t r[16];
    for (int c = 0; c < 64; c += 16) {
      TBN_TMEM_LD16(tq + c, r);
      tmem_ld_wait();
      for (int i = 0; i < 16; ++i) v[c + i] = __uint_as_float(r[i]);
    }
  }
  for (int c = 0; c < 64; ++c) D[t * 64 + c] = v[c];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tb);
}

int main() {
  std::vector<float> A(64 * K), B(K * N);
  for (int i = 0; i < 64 * K; ++i) A[i] = (float)((i * 7) % 13 - 6) * 0.25f;
  for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 5) % 11 - 5) * 0.125f;
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, 128 * 64 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for (int mode = 0; mode < 3; ++mode) {
    probe<<<1, 128, 65536>>>(dA, dB, dD, mode);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(128 * 64);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    // which lanes got which row's result?
    int hits = 0, sent = 0, other = 0;
    printf("mode %d:", mode);
    for (int lane = 0; lane < 128; ++lane) {
      int match = -1;
      for (int row = 0; row < 64 && match < 0; ++row) {
        bool ok = true;
        for (int n = 0; n < N && ok; ++n) {
          double ref = 0;
          for (int k = 0; k < K; ++k) ref += (double)A[row * K + k] * B[k * N + n];
          ok = fabs(D[lane * 64 + n] - ref) < 1e-2;
        }
        if (ok) match = row;
      }
      if (match >= 0) { ++hits; if (lane % 16 == 0) printf(" L%d<-r%d", lane, match); }
      else if (D[lane * 64] == -7.0f) ++sent; else ++other;
    }
    printf("  | lanes with a row result %d, untouched %d, other %d\n", hits, sent, other);
  }
  return 0;
}
