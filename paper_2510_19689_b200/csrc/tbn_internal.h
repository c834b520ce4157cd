// tbn_internal.h — internal (non-ABI) declarations of libtabnet_b200.
#pragma once
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <string>
#include <cuda_runtime.h>
#include "tbn_args.h"

namespace tbn {

void set_last_error(const std::string& msg);   // tbn_last_error() of this thread

// Raise a kernel's dynamic shared-memory limit once per (kernel, device): the
// attribute is per CUDA context, and one process may drive several GPUs
// (TabNetModel(device=N) caches one engine per device).  Thread-safe: the
// public host API is reentrant.  `Tag` makes the state per kernel instance.
constexpr int kMaxDevices = 64;

// Programmatic dependent launch for the K2 forward (TBN_NO_PDL=1 disables it: A/B)
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TBN_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}
template <class Tag>
cudaError_t smem_attr_once(const void* func, int bytes) {
  static std::once_flag once[kMaxDevices];
  static cudaError_t result[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [&] {
    result[dev] = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  });
  return result[dev];
}

// Pointers into the model's device buffer, fp32 row-major copies of the
// reference params dict (network.py:81-96), used by the CUDA-core kernel.
struct SimtParams {
  int F, ND, NA, S, C, H;
  float gamma;
  const float* scale;   // (F)  1/sqrt(var+eps)          (network.py:120)
  const float* shift;   // (F)  mean
  const float* sh1_W; const float* sh1_b;   // (F,2H) (2H)
  const float* sh2_W; const float* sh2_b;   // (H,2H) (2H)
  const float* fc1_W; const float* fc1_b;   // (S+1,H,2H) (S+1,2H)
  const float* fc2_W; const float* fc2_b;
  const float* att_W; const float* att_b;   // (S,NA,F) (S,F)   index s-1
  const float* head_W; const float* head_b; // (ND,C) (C)
};


size_t simt_smem_bytes(const SimtParams& p);
bool simt_supported(int F, int H, int C);      // the CUDA-core kernel's shape limits
cudaError_t launch_simt(const SimtParams& p, const ForwardArgs& a, int num_sms, cudaStream_t stream);
cudaError_t launch_sparsemax_f64(const double* z, int64_t rows, int n, double* out, int32_t* err_flag,
                                 int num_sms, cudaStream_t stream);
cudaError_t launch_sparsemax(const float* z, int64_t rows, int n, float* out, int32_t* err_flag,
                             int num_sms, cudaStream_t stream);
cudaError_t launch_partition_mean(const float* v, int64_t per, int partitions, int W, double* out,
                                  cudaStream_t stream);
cudaError_t launch_batch_stats(const float* x, int64_t rows, int F, float* scale, float* shift,
                               cudaStream_t stream);

}  // namespace tbn
