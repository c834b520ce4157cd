// tbn_args.h — the launch-argument block every fused forward kernel takes.
// Device-safe (no host headers), so the kernels also build under NVRTC
// (kernel_k2_jit.cu compiles K2 for model shapes without a prebuilt instance).
#pragma once
#include "tbn_rtc.h"

namespace tbn {

struct ForwardArgs {
  const float* x;
  int64_t rows;
  int normalized;
  const float* scale;   // per-call override (batch-stats control); null = model's
  const float* shift;
  float* logits;
  float* probs;
  float* masks;
  float* importance;
  int32_t* pred;
  int32_t* err_flag;
  float* scratch;              // K3: per-CTA row-tile state in the workspace
  unsigned long long* trace;   // debug timeline (TBN_TRACE env); null in production
  int packed;                  // TBN_FLAG_PACKED: host-side launch geometry only
};

// Raise the non-finite-input flag.  A plain (idempotent) store, not an
// atomic: the flag may live in device-mapped page-locked host memory (the
// zero-copy host path), where PCIe atomics are not guaranteed.
#ifdef __CUDACC__
__device__ __forceinline__ void raise_flag(int32_t* f) { *(volatile int32_t*)f = 1; }
#endif

}  // namespace tbn
