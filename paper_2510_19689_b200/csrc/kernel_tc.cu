// kernel_tc.cu — host side of K1 (tc_kernel.cuh): the weight packer K0 and the
// per-shape kernel instances.  K0 turns the reference's float64 params dict
// (network.py:81-96, used as x @ W) into the device weight image: a constant
// block (affine, biases, head) and one B operand block per GEMM, stored N x K
// K-major in the UMMA canonical no-swizzle layout, split hi/lo for 3xTF32:
// hi = rna_tf32(w), lo = rna_tf32(w - hi), both computed from the float64 weight.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "tbn_tc.h"
#include "tc_kernel.cuh"
#include "pack_util.h"

namespace tbn {

namespace {

using pack::pack_block;

struct Instance {
  int F, ND, NA, S, C, prec;
  bool (*pack)(const HostParams&, TcModel*, std::string*);
  cudaError_t (*launch)(const TcModel&, const ForwardArgs&, int, cudaStream_t);
};

template <class CF>
bool pack_impl(const HostParams& hp, TcModel* out, std::string* err) {
  constexpr int F = CF::F, H = CF::H, N2 = CF::N2, S = CF::S, ND = CF::ND, NA = CF::NA, C = CF::C;
  std::vector<float> c(CF::C_END, 0.0f);
  for (int f = 0; f < F; ++f) {
    c[CF::C_SCALE + f] = (float)(1.0 / std::sqrt(hp.norm_var[f] + 1e-8));   // network.py:120
    c[CF::C_SHIFT + f] = (float)hp.norm_mean[f];
  }
  // Folded GLU constants (the epilogue in tc_kernel.cuh relies on them):
  // gate columns x -log2(e) so exp(-u_gate) = 2^(D_gate + b'); the linear
  // columns of the residual blocks (shared2, fc1, fc2) x sqrt(.5), so
  // (lin*sigma + prev)*sqrt(.5) = lin'*sigma + sqrt(.5)*prev (network.py:131-137).
  const double kLog2e = 1.4426950408889634, kR = 0.70710678118654752440;
  std::vector<double> cs_first(N2), cs_res(N2);
  for (int n = 0; n < N2; ++n) {
    cs_first[n] = n < H ? 1.0 : -kLog2e;
    cs_res[n] = n < H ? kR : -kLog2e;
  }
  for (int n = 0; n < N2; ++n) {
    c[CF::C_BSH1 + n] = (float)(hp.sh1_b[n] * cs_first[n]);
    c[CF::C_BSH2 + n] = (float)(hp.sh2_b[n] * cs_res[n]);
    for (int s = 0; s <= S; ++s) {
      c[CF::C_BFC1 + s * N2 + n] = (float)(hp.fc1_b[s][n] * cs_res[n]);
      c[CF::C_BFC2 + s * N2 + n] = (float)(hp.fc2_b[s][n] * cs_res[n]);
    }
  }
  for (int s = 1; s <= S; ++s)
    for (int f = 0; f < F; ++f) c[CF::C_BATT + (s - 1) * CF::FN + f] = (float)hp.att_b[s][f];
  for (int i = 0; i < ND * C; ++i) c[CF::C_HW + i] = (float)hp.head_W[i];
  for (int i = 0; i < C; ++i) c[CF::C_HB + i] = (float)hp.head_b[i];

  const size_t a16 = 16;
  auto al = [&](size_t v) { return (v + a16 - 1) / a16 * a16; };
  size_t off = al(CF::CONST_BYTES);
  tc::TcParams tp{};
  tp.off_sh1 = (uint32_t)off; off = al(off + CF::B_SH1);
  tp.off_sh2 = (uint32_t)off; off = al(off + CF::B_HID);
  tp.off_fc1 = (uint32_t)off; off = al(off + (size_t)(S + 1) * CF::B_HID);
  tp.off_fc2 = (uint32_t)off; off = al(off + (size_t)(S + 1) * CF::B_HID);
  tp.off_att = (uint32_t)off; off = al(off + (size_t)S * CF::B_ATT);
  tp.gamma = (float)hp.gamma;
  const size_t bytes = off;
  std::vector<float> img(bytes / 4, 0.0f);
  std::memcpy(img.data(), c.data(), c.size() * 4);
  pack_block(img, tp.off_sh1 / 4, hp.sh1_W, F, N2, N2, CF::K1, CF::X3, N2, &cs_first, hp.sh1_b, CF::BF);
  pack_block(img, tp.off_sh2 / 4, hp.sh2_W, H, N2, N2, CF::KHID, CF::X3, N2, &cs_res, hp.sh2_b, CF::BF);
  for (int s = 0; s <= S; ++s) {
    pack_block(img, (tp.off_fc1 + (size_t)s * CF::B_HID) / 4, hp.fc1_W[s], H, N2, N2, CF::KHID, CF::X3, N2,
               &cs_res, hp.fc1_b[s], CF::BF);
    pack_block(img, (tp.off_fc2 + (size_t)s * CF::B_HID) / 4, hp.fc2_W[s], H, N2, N2, CF::KHID, CF::X3, N2,
               &cs_res, hp.fc2_b[s], CF::BF);
  }
  for (int s = 1; s <= S; ++s)
    pack_block(img, (tp.off_att + (size_t)(s - 1) * CF::B_ATT) / 4, hp.att_W[s], NA, F, CF::FN, CF::KATT,
               CF::X3, F, nullptr, hp.att_b[s], CF::BF);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(d, img.data(), bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (d) cudaFree(d);
    if (err) *err = cudaGetErrorString(e);
    return false;
  }
  tp.wimg = (const uint8_t*)d;
  out->d_buf = d;
  out->bytes = bytes;
  out->params = new tc::TcParams(tp);
  return true;
}

template <class CF>
cudaError_t launch_impl(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  constexpr int smem = tc::Smem<CF>::TOTAL;
  cudaError_t e = smem_attr_once<CF>((const void*)tc::tabnet_fused_tc<CF>, smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (a.rows + 127) / 128;
  const int64_t npairs = (ntiles + CF::NG - 1) / CF::NG;
  const int grid = (int)(npairs < num_sms ? npairs : num_sms);
  tc::tabnet_fused_tc<CF><<<grid, CF::THREADS, smem, stream>>>(*(const tc::TcParams*)m.params, a);
  return cudaGetLastError();
}

#define TBN_INSTANCE(F, ND, NA, S, C, P)                                             \
  Instance{F, ND, NA, S, C, P, &pack_impl<tc::Cfg<F, ND, NA, S, C, P>>,             \
           &launch_impl<tc::Cfg<F, ND, NA, S, C, P>>}

// Compiled model shapes (BASELINE.json configs; BLS as its 2-class reference model).
const Instance kInstances[] = {
    TBN_INSTANCE(14, 8, 8, 3, 2, tc::kPrecTF32x3),   // Adult
    TBN_INSTANCE(14, 8, 8, 3, 2, tc::kPrecTF32),
    TBN_INSTANCE(14, 8, 8, 3, 2, tc::kPrecBF16),
    TBN_INSTANCE(35, 16, 16, 5, 2, tc::kPrecTF32x3), // HR
    TBN_INSTANCE(35, 16, 16, 5, 2, tc::kPrecTF32),
    TBN_INSTANCE(35, 16, 16, 5, 2, tc::kPrecBF16),
    TBN_INSTANCE(64, 32, 32, 5, 2, tc::kPrecTF32x3), // BLS
    TBN_INSTANCE(64, 32, 32, 5, 2, tc::kPrecTF32),
    TBN_INSTANCE(64, 32, 32, 5, 2, tc::kPrecBF16),
    TBN_INSTANCE(64, 32, 32, 5, 1, tc::kPrecTF32x3), // BLS regression head (TBN_CFG_REGRESSION)
    TBN_INSTANCE(64, 32, 32, 5, 1, tc::kPrecTF32),
};

const Instance* find(const HostParams& hp, int precision) {
  int prec = precision == 0 ? tc::kPrecTF32x3
             : precision == 1 ? tc::kPrecTF32
             : precision == 2 ? tc::kPrecBF16 : -1;
  for (const Instance& in : kInstances)
    if (in.F == hp.F && in.ND == hp.ND && in.NA == hp.NA && in.S == hp.S && in.C == hp.C && in.prec == prec)
      return &in;
  return nullptr;
}

}  // namespace

bool tc_supported(const HostParams& hp, int precision) {
  // prebuilt instances, else K2 compiled for the shape at model creation
  // (whether that compile succeeds is only known then: tc_pack reports it)
  return k3_supported(hp, precision) || k2_supported(hp, precision) || find(hp, precision) != nullptr ||
         (k2_jit_available() && precision >= 0 && precision <= 2);
}

// K2 (k2_kernel.cuh) serves the single-pass modes wherever an instance exists;
// TBN_KERNEL=k1 pins the K1 design, TBN_KERNEL=jit prefers the runtime-compiled
// K2 over K1 (development A/B only).
static bool k2_allowed() {
  const char* e = std::getenv("TBN_KERNEL");
  return !(e && std::strcmp(e, "k1") == 0);
}
static bool jit_preferred() {
  const char* e = std::getenv("TBN_KERNEL");
  return e && std::strcmp(e, "jit") == 0;
}

bool tc_pack(const HostParams& hp, int precision, TcModel* out, std::string* err) {
  if (k3_supported(hp, precision)) {
    out->kernel = 3;
    out->precision = precision;
    return k3_pack(hp, precision, out, err);
  }
  if (k2_allowed() && k2_supported(hp, precision)) {
    out->kernel = 2;
    out->precision = precision;
    return k2_pack(hp, precision, out, err);
  }
  const Instance* in = jit_preferred() ? nullptr : find(hp, precision);
  if (!in) {
    if (k2_allowed() && k2_jit_available()) return k2_jit_pack(hp, precision, out, err);
    if (err) *err = "unsupported: no kernel instance for this shape";
    return false;
  }
  out->kernel = 1;
  out->shape_id = (int)(in - kInstances);
  out->precision = precision;
  return in->pack(hp, out, err);
}

void tc_free(TcModel* m) {
  if (m->kernel == 3) {
    k3_free(m);
    return;
  }
  if (m->kernel == 2) {
    k2_free(m);
    return;
  }
  if (m->d_buf) cudaFree(m->d_buf);
  delete (tc::TcParams*)m->params;
  m->d_buf = nullptr;
  m->params = nullptr;
}

cudaError_t launch_tc(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  if (m.kernel == 3) return k3_launch(m, a, num_sms, stream);
  if (m.kernel == 2) return k2_launch(m, a, num_sms, stream);
  if (m.shape_id < 0) return cudaErrorInvalidValue;
  return kInstances[m.shape_id].launch(m, a, num_sms, stream);
}

}  // namespace tbn
