// tbn_tc.h — the tcgen05 fused forward (kernel_tc.cu): host-side packing (K0)
// and launch interface.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "tbn_internal.h"

namespace tbn {

// Borrowed views of the reference params dict (float64, row-major, x @ W).
struct HostParams {
  int F = 0, ND = 0, NA = 0, S = 0, C = 0;
  double gamma = 1.3;
  const double* sh1_W = nullptr; const double* sh1_b = nullptr;
  const double* sh2_W = nullptr; const double* sh2_b = nullptr;
  std::vector<const double*> fc1_W, fc1_b, fc2_W, fc2_b;   // index s = 0..S
  std::vector<const double*> att_W, att_b;                 // index s = 1..S (0 unused)
  const double* head_W = nullptr; const double* head_b = nullptr;
  const double* norm_mean = nullptr; const double* norm_var = nullptr;
};

struct TcModel {
  int kernel = 1;          // 1: K1 (tc_kernel.cuh), 2: K2 (k2_kernel.cuh), 3: K3 (k3_kernel.cuh)
  int shape_id = -1;       // which compiled instance
  int precision = 0;
  void* d_buf = nullptr;   // packed operands + epilogue constants
  size_t bytes = 0;
  size_t scratch_per_cta = 0;   // K3: global per-CTA row-tile state (prior, agg, mask)
  void* params = nullptr;  // host copy of the kernel's parameter block
  const void* jit = nullptr;    // K2 compiled at run time (kernel_k2_jit.cu), else null
};

// A K2 shape's image/launch layout (k2_kernel.cuh Cfg constants, at run time).
struct K2Layout {
  int F = 0, ND = 0, NA = 0, S = 0, C = 0;
  bool X3 = false, BF = false;
  int H = 0, N2 = 0, NP = 0, K1 = 0, KHID = 0, KATT = 0, FN = 0;
  int C_SCALE = 0, C_SHIFT = 0, C_HW = 0, C_HB = 0;
  int O_SH1 = 0, O_SH2 = 0, O_FC1 = 0, O_FC2 = 0, O_ATT = 0, HBR = 0, ABR = 0;
  int IMG_BYTES = 0, SMEM_BYTES = 0, THREADS = 0;
};
bool k2_pack_layout(const K2Layout& L, const HostParams& hp, TcModel* out, std::string* err);

bool tc_supported(const HostParams& hp, int precision);
bool tc_pack(const HostParams& hp, int precision, TcModel* out, std::string* err);
void tc_free(TcModel* m);
cudaError_t launch_tc(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream);

// K2, the thread-per-row design for the single-pass modes (kernel_k2.cu)
bool k2_supported(const HostParams& hp, int precision);
bool k2_pack(const HostParams& hp, int precision, TcModel* out, std::string* err);
void k2_free(TcModel* m);
cudaError_t k2_launch(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream);

// K2 compiled for the model's shape at run time with NVRTC (kernel_k2_jit.cu):
// any shape the kernel's static limits admit, cubins cached in memory and on disk
bool k2_jit_available();
bool k2_jit_pack(const HostParams& hp, int precision, TcModel* out, std::string* err);
cudaError_t k2_jit_launch(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream);

// K3, the wide-model design (kernel_k3.cu)
bool k3_supported(const HostParams& hp, int precision);
bool k3_pack(const HostParams& hp, int precision, TcModel* out, std::string* err);
void k3_free(TcModel* m);
cudaError_t k3_launch(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream);

}  // namespace tbn
