// umma_probe.cu — hardware check of the tcgen05 operand layouts the fused
// kernel relies on (SS and TS kind::tf32, SS kind::f16/bf16, 3xTF32 split,
// N in {16,48,64,128}, K in {8,16,32,40,64}).  Standalone executable:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2510_19689_b200/csrc umma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"

using namespace tbn::ptx;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

// mode 0: SS tf32, 1: TS tf32, 2: SS tf32 3x (hi/lo), 3: SS bf16
__global__ void probe(const float* A, const float* B, float* D, int N, int K, int mode, int layout) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  const bool bf = (mode >= 3);
  const int esz = bf ? 2 : 4, T = 16 / esz;            // elements per 16-byte core-matrix row
  const uint32_t sboA = (K / T) * 128, sboB = (K / T) * 128;
  uint8_t* sA = smem;
  uint8_t* sAlo = sA + 128 * K * 4;
  uint8_t* sB = sAlo + 128 * K * 4;
  uint8_t* sBlo = sB + N * K * 4;
  // layout 0/2: 8-row groups at SBO=(K/T)*128, K core matrices at +128
  // layout 1   : K core-matrix columns outer (LBO=(rows/8)*128), 8-row groups at SBO=128
  auto offr = [&](int r, int k, int rows) -> uint32_t {
    if (layout == 1) return (k / T) * (uint32_t)(rows / 8 * 128) + (r / 8) * 128 + (r % 8) * 16 + (k % T) * esz;
    return (r / 8) * ((K / T) * 128) + (k / T) * 128 + (r % 8) * 16 + (k % T) * esz;
  };
  // stage A (row t) and B
  for (int k = 0; k < K; ++k) {
    float a = A[t * K + k];
    if (bf) {
      *(__nv_bfloat16*)(sA + offr(t, k, 128)) = __float2bfloat16(a);
    } else {
      *(float*)(sA + offr(t, k, 128)) = a;
      float hi = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
      *(float*)(sAlo + offr(t, k, 128)) = a - hi;
    }
  }
  for (int idx = t; idx < N * K; idx += 128) {
    int n = idx / K, k = idx % K;
    float b = B[k * N + n];   // W[k][n]
    if (bf) {
      *(__nv_bfloat16*)(sB + offr(n, k, N)) = __float2bfloat16(b);
    } else {
      *(float*)(sB + offr(n, k, N)) = b;
      float hi = __uint_as_float(__float_as_uint(b) & 0xFFFFE000u);
      *(float*)(sBlo + offr(n, k, N)) = b - hi;
    }
  }
  if (warp == 0) tmem_alloc<256>(&tbase);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d_t = tbase;          // D at col 0
  const uint32_t a_t = tbase + 128;    // A (TS mode) at col 128
  if (mode == 4) {
    // bf16 A in TMEM: hypothesis column c packs k = 2c (low half), 2c+1 (high half)
    uint32_t lane_base = a_t + ((uint32_t)(warp * 32) << 16);
    for (int k0 = 0; k0 < K; k0 += 16) {
      uint32_t r[8];
      for (int j = 0; j < 8; ++j) {
        __nv_bfloat162 v = __floats2bfloat162_rn(A[t * K + k0 + 2 * j], A[t * K + k0 + 2 * j + 1]);
        r[j] = *reinterpret_cast<uint32_t*>(&v);
      }
      TBN_TMEM_ST8(lane_base + k0 / 2, r);
    }
    tmem_st_wait();
  }
  if (mode == 1) {
    // lane t = row t, column k = A[t][k]
    uint32_t lane_base = a_t + ((uint32_t)(warp * 32) << 16);
    for (int k0 = 0; k0 < K; k0 += 8) {
      uint32_t r[8];
      for (int j = 0; j < 8; ++j) r[j] = __float_as_uint(A[t * K + k0 + j]);
      TBN_TMEM_ST8(lane_base + k0, r);
    }
    tmem_st_wait();
  }
  fence_async_shared();
  tc_fence_before();
  __syncthreads();
  if (t == 0) {
    tc_fence_after();
    const uint32_t fmt = bf ? kFmtBF16 : kFmtTF32;
    const uint32_t idesc = idesc_f32acc(fmt, 128, N);
    const int kstep = bf ? 16 : 8;
    int first = 1;
    for (int k0 = 0; k0 < K; k0 += kstep) {
      uint64_t da, db;
      if (layout == 1) {
        const uint32_t kA = (k0 / T) * (128 / 8 * 128), kB = (k0 / T) * (uint32_t)(N / 8 * 128);
        da = smem_desc(smem_u32(sA) + kA, 128 / 8 * 128, 128);
        db = smem_desc(smem_u32(sB) + kB, (uint32_t)(N / 8 * 128), 128);
      } else if (layout == 2) {
        const uint32_t koff = (k0 / T) * 128;
        da = smem_desc(smem_u32(sA) + koff, sboA, 128);
        db = smem_desc(smem_u32(sB) + koff, sboB, 128);
      } else {
        const uint32_t koff = (k0 / T) * 128;          // two core matrices per instruction
        da = smem_desc(smem_u32(sA) + koff, 128, sboA);
        db = smem_desc(smem_u32(sB) + koff, 128, sboB);
      }
      if (mode == 1) {
        mma_tf32_ts(d_t, a_t + k0, db, idesc, first ? 0u : 1u);
      } else if (mode == 3) {
        mma_f16_ss(d_t, da, db, idesc, first ? 0u : 1u);
      } else if (mode == 4) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     :: "r"(d_t), "r"(a_t + k0 / 2), "l"(db), "r"(idesc), "r"(first ? 0u : 1u) : "memory");
      } else {
        mma_tf32_ss(d_t, da, db, idesc, first ? 0u : 1u);
        if (mode == 2) {
          const uint32_t koff = (k0 / T) * 128;
          uint64_t dalo = smem_desc(smem_u32(sAlo) + koff, 128, sboA);
          uint64_t dblo = smem_desc(smem_u32(sBlo) + koff, 128, sboB);
          mma_tf32_ss(d_t, dalo, db, idesc, 1u);
          mma_tf32_ss(d_t, da, dblo, idesc, 1u);
        }
      }
      first = 0;
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t lane_d = d_t + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    TBN_TMEM_LD16(lane_d + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[t * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tbase);
}

static float trunc_tf32(float x) {
  uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float y; memcpy(&y, &u, 4); return y;
}
static float rn_bf16(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  int fails = 0;
  const int Ns[] = {16, 48, 64, 128};
  const int Ks[] = {8, 16, 32, 40, 64};
  for (int mode = 0; mode < 5; ++mode)
   for (int layout = 0; layout < 3; ++layout)
    for (int N : Ns)
      for (int K : Ks) {
        if (mode >= 3 && K % 16) continue;
        if (layout > 0 && !(mode == 3 || (mode == 0 && layout == 1))) continue;
        std::vector<float> A(128 * K), B(K * N), D(128 * N);
        srand(1234 + N * 7 + K);
        for (auto& v : A) v = (rand() / (float)RAND_MAX - 0.5f) * 4.f;
        for (auto& v : B) v = (rand() / (float)RAND_MAX - 0.5f) * 4.f;
        float *dA, *dB, *dD;
        CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
        CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(dD, 0, D.size() * 4));
        size_t smem = 128 * K * 8 + N * K * 8 + 1024;
        CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        probe<<<1, 128, smem>>>(dA, dB, dD, N, K, mode, layout);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0, maxref = 0;
        for (int r = 0; r < 128; ++r)
          for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k) {
              float a = A[r * K + k], b = B[k * N + n];
              if (mode >= 3) { a = rn_bf16(a); b = rn_bf16(b); }
              else if (mode != 2) { a = trunc_tf32(a); b = trunc_tf32(b); }
              ref += (double)a * (double)b;
            }
            maxerr = fmax(maxerr, fabs(ref - D[r * N + n]));
            maxref = fmax(maxref, fabs(ref));
          }
        double rel = maxerr / maxref;
        bool ok = rel < (mode == 2 ? 2e-6 : 1e-5);
        if (!ok) fails += 0;
        if (!ok) ++fails;
        printf("mode=%d(%s) layout=%d N=%3d K=%2d  max|err|=%.3e rel=%.3e %s\n", mode,
               mode == 0 ? "ss_tf32" : mode == 1 ? "ts_tf32" : mode == 2 ? "ss_3xtf32" : mode == 3 ? "ss_bf16" : "ts_bf16",
               layout, N, K, maxerr, rel, ok ? "OK" : "FAIL");
        cudaFree(dA); cudaFree(dB); cudaFree(dD);
      }
  printf("probe: %d failures\n", fails);
  return fails ? 1 : 0;
}
