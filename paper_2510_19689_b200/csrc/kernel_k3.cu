// kernel_k3.cu — host side of K3 (k3_kernel.cuh), the wide-model kernel: its
// weight packer and instance.  Every B operand is cut into K-chunks of at most
// 32 KB, each a standalone N x Kc K-major canonical block (bf16, round to
// nearest even from the float64 weight), stored back to back in the order the
// kernel streams them.  GLU constants are folded as in K2 (tanh form).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include "tbn_tc.h"
#include "k3_kernel.cuh"
#include "k3x_kernel.cuh"
#include "pack_util.h"

namespace tbn {

namespace {

// The device's persisting-L2 set-aside for K3's row-state scratch: reserved
// once per device at model creation (cudaDeviceSetLimit is not allowed while
// a stream captures, and the host path captures its launches as graphs);
// launches only read it.  TBN_K3_PERSIST_MB overrides (0 disables).
std::once_flag g_persist_once[kMaxDevices];
size_t g_persist_bytes[kMaxDevices];

void l2_persist_setup(size_t want) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return;
  std::call_once(g_persist_once[dev], [&] {
    g_persist_bytes[dev] = 0;
    int maxp = 0;
    if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess) return;
    size_t lim = want;
    if (const char* e = std::getenv("TBN_K3_PERSIST_MB")) lim = (size_t)std::atol(e) << 20;
    if (lim > (size_t)maxp) lim = (size_t)maxp;
    if (lim > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim) == cudaSuccess)
      g_persist_bytes[dev] = lim;
    cudaGetLastError();
  });
}

// the largest access-policy window the device accepts (cudaDevAttrMaxAccessPolicyWindowSize)
size_t max_window_bytes() {
  static std::once_flag once[kMaxDevices];
  static size_t v[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  std::call_once(once[dev], [&] {
    int w = 0;
    v[dev] = cudaDeviceGetAttribute(&w, cudaDevAttrMaxAccessPolicyWindowSize, dev) == cudaSuccess ? (size_t)w : 0;
    cudaGetLastError();
  });
  return v[dev];
}

size_t l2_persist_bytes() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
  return g_persist_bytes[dev];
}

// W (Kin x N row-major, x @ W) -> chunks of kc rows of K (last may be short),
// element (n, k) of a chunk at (n/8)*(kc*8) + (k/8)*64 + (n%8)*8 + k%8.
// Row k == Kin carries the bias (when given); rows beyond are zero.
void pack_chunked(std::vector<uint16_t>& img, size_t off_bytes, const double* W, int Kin, int N,
                  int Ktot, int kc_max, const std::vector<double>* colscale, const double* bias) {
  size_t base = off_bytes / 2;
  for (int k0 = 0; k0 < Ktot; k0 += kc_max) {
    const int kc = Ktot - k0 < kc_max ? Ktot - k0 : kc_max;
    for (int n = 0; n < N; ++n)
      for (int kl = 0; kl < kc; ++kl) {
        const int k = k0 + kl;
        double w = k < Kin ? W[(size_t)k * N + n] : (bias && k == Kin ? bias[n] : 0.0);
        if (colscale) w *= (*colscale)[n];
        img[base + (size_t)(n / 8) * (kc * 8) + (kl / 8) * 64 + (n % 8) * 8 + (kl % 8)] =
            pack::bf16_rn_host((float)w);
      }
    base += (size_t)N * kc;
  }
}

template <class CF>
bool pack_k3(const HostParams& hp, TcModel* out, std::string* err) {
  constexpr int F = CF::F, H = CF::H, N2 = CF::N2, S = CF::S, ND = CF::ND, NA = CF::NA, C = CF::C;
  std::vector<uint16_t> img(CF::IMG_BYTES / 2, 0);
  float* cst = reinterpret_cast<float*>(img.data());
  const double kR = 0.70710678118654752440;
  for (int f = 0; f < F; ++f) {
    cst[CF::C_SCALE + f] = (float)(1.0 / std::sqrt(hp.norm_var[f] + 1e-8));   // network.py:120
    cst[CF::C_SHIFT + f] = (float)hp.norm_mean[f];
  }
  for (int n = 0; n < N2; ++n) cst[CF::C_B1 + n] = (float)(hp.sh1_b[n] * 0.5);  // shared1 bias, tanh-folded
  for (int i = 0; i < ND * C; ++i) cst[CF::C_HW + i] = (float)hp.head_W[i];
  for (int i = 0; i < C; ++i) cst[CF::C_HB + i] = (float)hp.head_b[i];
  std::vector<double> cs_first(N2, 0.5), cs_res(N2);
  for (int n = 0; n < N2; ++n) cs_res[n] = n < H ? 0.5 * kR : 0.5;
  pack_chunked(img, CF::O_SH1, hp.sh1_W, F, N2, CF::K1, CF::KC_N2, &cs_first, nullptr);
  pack_chunked(img, CF::O_SH2, hp.sh2_W, H, N2, CF::KHID, CF::KC_N2, &cs_res, hp.sh2_b);
  for (int s = 0; s <= S; ++s) {
    pack_chunked(img, CF::O_FC1 + (size_t)s * CF::BLK_HID, hp.fc1_W[s], H, N2, CF::KHID, CF::KC_N2,
                 &cs_res, hp.fc1_b[s]);
    pack_chunked(img, CF::O_FC2 + (size_t)s * CF::BLK_HID, hp.fc2_W[s], H, N2, CF::KHID, CF::KC_N2,
                 &cs_res, hp.fc2_b[s]);
  }
  for (int s = 1; s <= S; ++s)
    pack_chunked(img, CF::O_ATT + (size_t)(s - 1) * CF::BLK_ATT, hp.att_W[s], NA, F, CF::KATT,
                 CF::KC_ATT, nullptr, hp.att_b[s]);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, CF::IMG_BYTES);
  if (e == cudaSuccess) e = cudaMemcpy(d, img.data(), CF::IMG_BYTES, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (d) cudaFree(d);
    if (err) *err = cudaGetErrorString(e);
    return false;
  }
  out->d_buf = d;
  out->bytes = CF::IMG_BYTES;
  out->scratch_per_cta = CF::SCRATCH_PER_CTA;
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      l2_persist_setup((size_t)sms * CF::SCRATCH_PER_CTA);
  }
  out->params = new k3::Params{(const uint8_t*)d, (float)hp.gamma};
  return true;
}

template <class CF>
cudaError_t launch_k3_impl(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  cudaError_t e = smem_attr_once<CF>((const void*)k3::tabnet_wide<CF>, CF::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  if (!a.scratch) return cudaErrorInvalidValue;
  const int64_t ntiles = (a.rows + 127) / 128;
  int cap = num_sms;
  if (const char* e = std::getenv("TBN_K3_GRID")) cap = std::atoi(e) > 0 ? std::atoi(e) : num_sms;   // dev A/B
  const int grid = (int)(ntiles < cap ? ntiles : cap);
  // The per-CTA row-state scratch is re-read every step: pin it in L2 with a
  // persisting access-policy window over exactly the scratch this launch uses
  // (the evict_last hints inside the kernel only take effect within the
  // device's persisting set-aside, which defaults to 0).
  const size_t scratch_bytes = (size_t)grid * CF::SCRATCH_PER_CTA;
  const size_t persist = l2_persist_bytes();
  const size_t window = scratch_bytes < max_window_bytes() ? scratch_bytes : max_window_bytes();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = CF::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (persist > 0 && window > 0) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = a.scratch;
    attr[0].val.accessPolicyWindow.num_bytes = window;
    attr[0].val.accessPolicyWindow.hitRatio = (float)((double)persist / (double)window > 1.0
                                                          ? 1.0 : (double)persist / (double)window);
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, k3::tabnet_wide<CF>, *(const k3::Params*)m.params, a);
}

// ---- K3X (k3x_kernel.cuh): the 3xTF32 wide kernel -------------------------
// B chunks of kc K-rows: hi block (N x kc, K-major canonical tf32: element
// (n, k) at (n/8)*(kc*8) + (k/4)*32 + (n%8)*4 + k%4) then the lo block;
// hi = rna_tf32(w'), lo = rna_tf32(w' - hi) from the float64 w' = w * colscale.
void pack_chunked_tf32(std::vector<float>& img, size_t off_bytes, const double* W, int Kin, int N, int kc,
                       const std::vector<double>* colscale) {
  size_t base = off_bytes / 4;
  for (int k0 = 0; k0 < Kin; k0 += kc) {
    for (int n = 0; n < N; ++n)
      for (int kl = 0; kl < kc; ++kl) {
        const int k = k0 + kl;
        double w = k < Kin ? W[(size_t)k * N + n] : 0.0;
        if (colscale) w *= (*colscale)[n];
        const size_t idx = (size_t)(n / 8) * (kc * 8) + (kl / 4) * 32 + (n % 8) * 4 + (kl % 4);
        const float h = pack::tf32_rna_host((float)w);
        img[base + idx] = h;
        img[base + (size_t)N * kc + idx] = pack::tf32_rna_host((float)(w - (double)h));
      }
    base += (size_t)2 * N * kc;
  }
}

template <class CF>
bool pack_k3x(const HostParams& hp, TcModel* out, std::string* err) {
  constexpr int F = CF::F, H = CF::H, N2 = CF::N2, S = CF::S, ND = CF::ND, NA = CF::NA, C = CF::C;
  std::vector<float> img(CF::IMG_BYTES / 4, 0.0f);
  for (int f = 0; f < F; ++f) {
    img[CF::C_SCALE + f] = (float)(1.0 / std::sqrt(hp.norm_var[f] + 1e-8));   // network.py:120
    img[CF::C_SHIFT + f] = (float)hp.norm_mean[f];
  }
  for (int i = 0; i < ND * C; ++i) img[CF::C_HW + i] = (float)hp.head_W[i];
  for (int i = 0; i < C; ++i) img[CF::C_HB + i] = (float)hp.head_b[i];
  // exact sigmoid (as K1/K2 3xTF32): gate columns x -log2(e); residual blocks'
  // linear columns x sqrt(1/2) (network.py:131-137)
  const double kR = 0.70710678118654752440, kLog2e = 1.4426950408889634;
  std::vector<double> cs_first(N2), cs_res(N2);
  for (int n = 0; n < N2; ++n) {
    cs_first[n] = n < H ? 1.0 : -kLog2e;
    cs_res[n] = n < H ? kR : -kLog2e;
  }
  float* b = img.data() + CF::O_BIAS / 4;
  for (int n = 0; n < N2; ++n) {
    b[CF::B_SH1 + n] = (float)(hp.sh1_b[n] * cs_first[n]);
    b[CF::B_SH2 + n] = (float)(hp.sh2_b[n] * cs_res[n]);
    for (int s = 0; s <= S; ++s) {
      b[CF::B_FC1 + s * N2 + n] = (float)(hp.fc1_b[s][n] * cs_res[n]);
      b[CF::B_FC2 + s * N2 + n] = (float)(hp.fc2_b[s][n] * cs_res[n]);
    }
  }
  for (int s = 1; s <= S; ++s)
    for (int f = 0; f < F; ++f) b[CF::B_ATT + (s - 1) * F + f] = (float)hp.att_b[s][f];
  pack_chunked_tf32(img, CF::O_SH1, hp.sh1_W, F, N2, CF::KC_N2, &cs_first);
  pack_chunked_tf32(img, CF::O_SH2, hp.sh2_W, H, N2, CF::KC_N2, &cs_res);
  for (int s = 0; s <= S; ++s) {
    pack_chunked_tf32(img, CF::O_FC1 + (size_t)s * CF::BLK_HID, hp.fc1_W[s], H, N2, CF::KC_N2, &cs_res);
    pack_chunked_tf32(img, CF::O_FC2 + (size_t)s * CF::BLK_HID, hp.fc2_W[s], H, N2, CF::KC_N2, &cs_res);
  }
  for (int s = 1; s <= S; ++s)
    pack_chunked_tf32(img, CF::O_ATT + (size_t)(s - 1) * CF::BLK_ATT, hp.att_W[s], NA, F, CF::KC_ATT, nullptr);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, CF::IMG_BYTES);
  if (e == cudaSuccess) e = cudaMemcpy(d, img.data(), CF::IMG_BYTES, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (d) cudaFree(d);
    if (err) *err = cudaGetErrorString(e);
    return false;
  }
  out->d_buf = d;
  out->bytes = CF::IMG_BYTES;
  out->scratch_per_cta = CF::SCRATCH_PER_CTA;
  // (k3_free deletes params as k3::Params: the layouts are identical)
  static_assert(sizeof(k3x::Params) == sizeof(k3::Params), "params layout");
  out->params = new k3::Params{(const uint8_t*)d, (float)hp.gamma};
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      l2_persist_setup((size_t)sms * CF::SCRATCH_PER_CTA);
  }
  return true;
}

template <class CF>
cudaError_t launch_k3x_impl(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  cudaError_t e = smem_attr_once<CF>((const void*)k3x::tabnet_wide_x3<CF>, CF::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  if (!a.scratch) return cudaErrorInvalidValue;
  const int64_t ntiles = (a.rows + 127) / 128;
  int cap = num_sms;
  if (const char* e = std::getenv("TBN_K3_GRID")) cap = std::atoi(e) > 0 ? std::atoi(e) : num_sms;   // dev A/B
  const int grid = (int)(ntiles < cap ? ntiles : cap);
  const size_t scratch_bytes = (size_t)grid * CF::SCRATCH_PER_CTA;
  const size_t persist = l2_persist_bytes();
  const size_t window = scratch_bytes < max_window_bytes() ? scratch_bytes : max_window_bytes();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = CF::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (persist > 0 && window > 0) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = a.scratch;
    attr[0].val.accessPolicyWindow.num_bytes = window;
    attr[0].val.accessPolicyWindow.hitRatio = (float)((double)persist / (double)window > 1.0
                                                          ? 1.0 : (double)persist / (double)window);
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  k3x::Params prm{((const k3::Params*)m.params)->wimg, ((const k3::Params*)m.params)->gamma};
  return cudaLaunchKernelEx(&cfg, k3x::tabnet_wide_x3<CF>, prm, a);
}

struct K3Instance {
  int F, ND, NA, S, C, prec;
  bool (*pack)(const HostParams&, TcModel*, std::string*);
  cudaError_t (*launch)(const TcModel&, const ForwardArgs&, int, cudaStream_t);
};

#define TBN_K3(F, ND, NA, S, C) \
  K3Instance{F, ND, NA, S, C, 2, &pack_k3<k3::Cfg<F, ND, NA, S, C>>, &launch_k3_impl<k3::Cfg<F, ND, NA, S, C>>}
#define TBN_K3X(F, ND, NA, S, C) \
  K3Instance{F, ND, NA, S, C, 0, &pack_k3x<k3x::Cfg<F, ND, NA, S, C>>, &launch_k3x_impl<k3x::Cfg<F, ND, NA, S, C>>}

const K3Instance kK3[] = {
    TBN_K3(512, 64, 64, 8, 10),   // wide (BASELINE config 5), bf16
    TBN_K3X(512, 64, 64, 8, 10),  // wide, 3xTF32 (the parity mode)
};

const K3Instance* find_k3(const HostParams& hp, int precision) {
  if (std::getenv("TBN_NO_K3X") && precision == 0) return nullptr;   // dev A/B: the CUDA-core fp32 path
  for (const K3Instance& in : kK3)
    if (in.prec == precision && in.F == hp.F && in.ND == hp.ND && in.NA == hp.NA && in.S == hp.S && in.C == hp.C)
      return &in;
  return nullptr;
}

}  // namespace

bool k3_supported(const HostParams& hp, int precision) { return find_k3(hp, precision) != nullptr; }

bool k3_pack(const HostParams& hp, int precision, TcModel* out, std::string* err) {
  const K3Instance* in = find_k3(hp, precision);
  if (!in) {
    if (err) *err = "no K3 instance";
    return false;
  }
  out->shape_id = (int)(in - kK3);
  return in->pack(hp, out, err);
}

void k3_free(TcModel* m) {
  if (m->d_buf) cudaFree(m->d_buf);
  delete (k3::Params*)m->params;
  m->d_buf = nullptr;
  m->params = nullptr;
}

cudaError_t k3_launch(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  if (m.shape_id < 0) return cudaErrorInvalidValue;
  return kK3[m.shape_id].launch(m, a, num_sms, stream);
}

}  // namespace tbn
