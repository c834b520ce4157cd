// kernel_k2.cu — host side of K2 (k2_kernel.cuh): its weight packer and the
// per-shape instances.  The image is the reference's float64 params dict
// (network.py:81-96, used as x @ W) as B operands (N x K K-major canonical,
// TF32 = rna(w) or BF16 = rne(w)) with the bias as an extra K row, and the GLU
// constants folded in for the tanh form of the sigmoid:
//   sigma(u) = (1 + tanh(u/2)) / 2   =>  gate columns x 1/2,
//   linear columns x 1/2 (shared1) or x sqrt(1/2)/2 (the residual blocks
//   shared2/fc1/fc2, network.py:131-137: (lin sigma + prev) sqrt(.5)).
#include <type_traits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "tbn_tc.h"
#include "k2_kernel.cuh"
#include "pack_util.h"

#ifndef TBN_K2_ROWQ
#define TBN_K2_ROWQ 128
#endif

namespace tbn {

// The K2 weight image for one shape (layout L): constants, then every B
// operand block (pack_util.h: N x K K-major canonical, bias hi/lo rows 0/1).
bool k2_pack_layout(const K2Layout& L, const HostParams& hp, TcModel* out, std::string* err) {
  const int F = L.F, H = L.H, N2 = L.N2, S = L.S, ND = L.ND, NA = L.NA, C = L.C;
  std::vector<float> img(L.IMG_BYTES / 4, 0.0f);
  for (int f = 0; f < F; ++f) {
    img[L.C_SCALE + f] = (float)(1.0 / std::sqrt(hp.norm_var[f] + 1e-8));   // network.py:120
    img[L.C_SHIFT + f] = (float)hp.norm_mean[f];
  }
  for (int i = 0; i < ND * C; ++i) img[L.C_HW + i] = (float)hp.head_W[i];
  for (int i = 0; i < C; ++i) img[L.C_HB + i] = (float)hp.head_b[i];
  const double kR = 0.70710678118654752440, kLog2e = 1.4426950408889634;
  std::vector<double> cs_first(N2), cs_res(N2);
  for (int n = 0; n < N2; ++n) {
    if (L.X3) {              // exact sigmoid: gate x -log2(e); residual linear x sqrt(.5)
      cs_first[n] = n < H ? 1.0 : -kLog2e;
      cs_res[n] = n < H ? kR : -kLog2e;
    } else {                 // tanh form: everything x 1/2, residual linear x sqrt(.5)/2
      cs_first[n] = 0.5;
      cs_res[n] = n < H ? 0.5 * kR : 0.5;
    }
  }
  using pack::pack_block_k2;
  pack_block_k2(img, L.O_SH1 / 4, hp.sh1_W, F, N2, L.NP, L.K1, L.X3, N2, &cs_first, hp.sh1_b, L.BF);
  pack_block_k2(img, L.O_SH2 / 4, hp.sh2_W, H, N2, L.NP, L.KHID, L.X3, N2, &cs_res, hp.sh2_b, L.BF);
  for (int s = 0; s <= S; ++s) {
    pack_block_k2(img, (L.O_FC1 + s * L.HBR) / 4, hp.fc1_W[s], H, N2, L.NP, L.KHID, L.X3, N2, &cs_res,
                  hp.fc1_b[s], L.BF);
    pack_block_k2(img, (L.O_FC2 + s * L.HBR) / 4, hp.fc2_W[s], H, N2, L.NP, L.KHID, L.X3, N2, &cs_res,
                  hp.fc2_b[s], L.BF);
  }
  for (int s = 1; s <= S; ++s)
    pack_block_k2(img, (L.O_ATT + (s - 1) * L.ABR) / 4, hp.att_W[s], NA, F, L.FN, L.KATT, L.X3, F, nullptr,
                  hp.att_b[s], L.BF);
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, L.IMG_BYTES);
  if (e == cudaSuccess) e = cudaMemcpy(d, img.data(), L.IMG_BYTES, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (d) cudaFree(d);
    if (err) *err = cudaGetErrorString(e);
    return false;
  }
  out->d_buf = d;
  out->bytes = L.IMG_BYTES;
  out->params = new k2::Params{(const uint8_t*)d, (float)hp.gamma};
  return true;
}

namespace {

struct K2Instance {
  int F, ND, NA, S, C, prec;
  bool (*pack)(const HostParams&, TcModel*, std::string*);
  cudaError_t (*launch)(const TcModel&, const ForwardArgs&, int, cudaStream_t);
};

// Everything the packer and the launcher need to know about one K2 shape;
// built from the compile-time Cfg for the prebuilt instances and read back
// from a query kernel for NVRTC-compiled ones (kernel_k2_jit.cu).
template <class CF>
K2Layout layout_of() {
  K2Layout L;
  L.F = CF::F; L.ND = CF::ND; L.NA = CF::NA; L.S = CF::S; L.C = CF::C;
  L.X3 = CF::X3; L.BF = CF::BF; L.H = CF::H; L.N2 = CF::N2; L.NP = CF::NP;
  L.K1 = CF::K1; L.KHID = CF::KHID; L.KATT = CF::KATT; L.FN = CF::FN;
  L.C_SCALE = CF::C_SCALE; L.C_SHIFT = CF::C_SHIFT; L.C_HW = CF::C_HW; L.C_HB = CF::C_HB;
  L.O_SH1 = CF::O_SH1; L.O_SH2 = CF::O_SH2; L.O_FC1 = CF::O_FC1; L.O_FC2 = CF::O_FC2; L.O_ATT = CF::O_ATT;
  L.HBR = tc::rup(CF::B_HID, 128); L.ABR = tc::rup(CF::B_ATT, 128);
  L.IMG_BYTES = CF::IMG_BYTES; L.SMEM_BYTES = CF::SMEM_BYTES; L.THREADS = CF::THREADS;
  return L;
}

template <class CF>
bool pack_k2(const HostParams& hp, TcModel* out, std::string* err) {
  return k2_pack_layout(layout_of<CF>(), hp, out, err);
}

// rows of the batch -> CTAs: one CTA per SM, each with a contiguous, equal
// block of rows (k2_kernel.cuh); small batches: one CTA per TBN_K2_ROWQ rows
// (spreading them thinner, 32 rows per CTA, measured no faster).
// TBN_FLAG_PACKED: NG full tiles per CTA on as few SMs as the batch needs.
inline int k2_grid(const ForwardArgs& a, int num_sms, int ng) {
  const int64_t nq = a.packed ? (a.rows + 128 * ng - 1) / (128 * ng) : (a.rows + TBN_K2_ROWQ - 1) / TBN_K2_ROWQ;
  return (int)(nq < num_sms ? nq : num_sms);
}

template <class CF>
cudaError_t launch_k2_cfg(const TcModel& m, const ForwardArgs& a, int grid, cudaStream_t stream) {
  cudaError_t e = smem_attr_once<CF>((const void*)k2::tabnet_rowthread<CF>, CF::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = CF::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (k2_kernel.cuh)
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k2::tabnet_rowthread<CF>, *(const k2::Params*)m.params, a);
}

// The split latency instance of a shape (k2_kernel.cuh, Cfg::SPLIT) where its
// one 8-warp group fits with every weight block resident; else none (the
// 2-group latency instance stands in).
template <int F, int ND, int NA, int S, int C, int P>
struct SplitOf {
  static constexpr bool ok = ND % 2 == 0 && NA % 2 == 0 &&
                             (!k2::Cfg<F, ND, NA, S, C, P, 1>::RING || P == tc::kPrecTF32x3);
  using type = std::conditional_t<ok, k2::Cfg<F, ND, NA, S, C, P, 1, true>, k2::Cfg<F, ND, NA, S, C, P, 2>>;
};

// CF: the throughput instance; CL: the latency instance of the same shape
// (at most 2 row groups), launched when no CTA gets more than CL::NG tiles;
// CS: the split latency instance, launched when every CTA gets one tile.
// All read the same weight image and give bitwise identical rows.
template <class CF, class CL, class CS>
cudaError_t launch_k2_impl(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  static_assert(CF::IMG_BYTES == CL::IMG_BYTES && CF::O_ATT == CL::O_ATT && CF::O_FC2 == CL::O_FC2 &&
                CF::C_HB == CL::C_HB, "the latency instance must read the same weight image");
  static_assert(CF::IMG_BYTES == CS::IMG_BYTES && CF::O_ATT == CS::O_ATT && CF::O_FC2 == CS::O_FC2 &&
                CF::C_HB == CS::C_HB, "the split instance must read the same weight image");
  if constexpr (CS::SPLIT || CL::NG < CF::NG) {
    static const bool off = std::getenv("TBN_K2_NO_LATENCY") != nullptr;   // development A/B only
    static const bool nosplit = std::getenv("TBN_K2_NO_SPLIT") != nullptr;  // development A/B only
    if (!a.packed && !off) {
      const int grid = k2_grid(a, num_sms, CL::NG);
      const int64_t rpc = (((a.rows + grid - 1) / grid) + 3) & ~(int64_t)3;
      if constexpr (CS::SPLIT) {
        if (rpc <= 128 && !nosplit) return launch_k2_cfg<CS>(m, a, grid, stream);
      }
      if constexpr (CL::NG < CF::NG) {
        if ((rpc + 127) / 128 <= CL::NG) return launch_k2_cfg<CL>(m, a, grid, stream);
      }
    }
  }
  return launch_k2_cfg<CF>(m, a, k2_grid(a, num_sms, CF::NG), stream);
}

#define TBN_K2(F, ND, NA, S, C, P)                                                  \
  K2Instance{F, ND, NA, S, C, P, &pack_k2<k2::Cfg<F, ND, NA, S, C, P>>,            \
             &launch_k2_impl<k2::Cfg<F, ND, NA, S, C, P>, k2::Cfg<F, ND, NA, S, C, P, 2>, \
                             typename SplitOf<F, ND, NA, S, C, P>::type>}

#ifdef TBN_K2_SINGLE   // dev A/B builds: one instance only, e.g. -DTBN_K2_SINGLE=K2_HR_BF16
#define K2_HR_BF16 35, 16, 16, 5, 2, tc::kPrecBF16
#define K2_HR_TF32 35, 16, 16, 5, 2, tc::kPrecTF32
#define K2_HR_X3 35, 16, 16, 5, 2, tc::kPrecTF32x3
#define K2_BLS_BF16 64, 32, 32, 5, 1, tc::kPrecBF16
#define TBN_K2_EXPAND(...) TBN_K2(__VA_ARGS__)
const K2Instance kK2[] = {TBN_K2_EXPAND(TBN_K2_SINGLE)};
#else
const K2Instance kK2[] = {
    TBN_K2(14, 8, 8, 3, 2, tc::kPrecTF32x3),   // Adult, 3xTF32 parity mode
    TBN_K2(35, 16, 16, 5, 2, tc::kPrecTF32x3), // HR, 3xTF32 parity mode
    TBN_K2(14, 8, 8, 3, 2, tc::kPrecTF32),     // Adult
    TBN_K2(14, 8, 8, 3, 2, tc::kPrecBF16),
    TBN_K2(35, 16, 16, 5, 2, tc::kPrecTF32),   // HR
    TBN_K2(35, 16, 16, 5, 2, tc::kPrecBF16),
    TBN_K2(64, 32, 32, 5, 2, tc::kPrecBF16),   // BLS (its 2-class reference model)
    TBN_K2(64, 32, 32, 5, 1, tc::kPrecBF16),   // BLS regression head (TBN_CFG_REGRESSION)
};
#endif

const K2Instance* find_k2(const HostParams& hp, int precision) {
  const int prec = precision == 0 ? tc::kPrecTF32x3 : precision == 1 ? tc::kPrecTF32
                 : precision == 2 ? tc::kPrecBF16 : -1;
  for (const K2Instance& in : kK2)
    if (in.F == hp.F && in.ND == hp.ND && in.NA == hp.NA && in.S == hp.S && in.C == hp.C && in.prec == prec)
      return &in;
  return nullptr;
}

}  // namespace

bool k2_supported(const HostParams& hp, int precision) { return find_k2(hp, precision) != nullptr; }

bool k2_pack(const HostParams& hp, int precision, TcModel* out, std::string* err) {
  const K2Instance* in = find_k2(hp, precision);
  if (!in) {
    if (err) *err = "no K2 instance";
    return false;
  }
  out->shape_id = (int)(in - kK2);
  out->jit = nullptr;
  return in->pack(hp, out, err);
}

void k2_free(TcModel* m) {
  if (m->d_buf) cudaFree(m->d_buf);
  delete (k2::Params*)m->params;
  m->d_buf = nullptr;
  m->params = nullptr;
}

cudaError_t k2_launch(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  if (m.jit) return k2_jit_launch(m, a, num_sms, stream);
  if (m.shape_id < 0) return cudaErrorInvalidValue;
  return kK2[m.shape_id].launch(m, a, num_sms, stream);
}

}  // namespace tbn
