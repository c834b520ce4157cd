// kernel_prep.cu — device preprocessing: the numeric tail
// of the reference's PreprocessPlan.transform (data/preprocess.py:68-122) on
// the GPU, ahead of the forward.
//
// The host keeps what only the host can do — the string -> level lookups on
// Python objects — and hands over one float64 code per raw column and row:
//   standardize / passthrough : the value, NaN when the cell was missing (None)
//   ordinal                   : the level's integer (the plan's mapping), -1 unseen
//   onehot                    : the category index, -1 when absent from the plan
// The kernel expands that (rows x ncols) code matrix into the model's input
// matrix (rows x F) in float32: median imputation, (v - mean) / std in float64
// then one rounding (so the result equals the reference's float64 matrix cast
// to float32 bit for bit), ordinal codes as values, one-hot blocks.  One thread
// per output element, so the F-wide rows are written fully coalesced; the
// per-feature descriptor (source column, kind, level, constants) is a small
// device table built once per plan.
#include <cmath>
#include <cstdint>
#include <vector>

#include "tabnet_b200.h"
#include "tbn_internal.h"

struct tbn_prep {
  int device = 0;
  int ncols = 0;
  int width = 0;            // output features F
  int* d_src = nullptr;     // per output feature: source column
  int* d_kind = nullptr;    //                     kind
  int* d_level = nullptr;   //                     one-hot level index
  double* d_k = nullptr;    //                     median, mean, std (3 per feature)
};

namespace {

__global__ void prep_kernel(const double* __restrict__ codes, int64_t rows, int ncols, int F,
                            const int* __restrict__ src, const int* __restrict__ kind,
                            const int* __restrict__ level, const double* __restrict__ kc,
                            float* __restrict__ out) {
  const int64_t total = rows * (int64_t)F;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F;
    const int f = (int)(i - r * F);
    const double v = __ldg(codes + r * ncols + __ldg(src + f));
    const int k = __ldg(kind + f);
    double o;
    if (k == TBN_PREP_STANDARDIZE || k == TBN_PREP_PASSTHROUGH) {
      const double x = isnan(v) ? __ldg(kc + 3 * f) : v;                   // impute the median
      o = (k == TBN_PREP_STANDARDIZE) ? (x - __ldg(kc + 3 * f + 1)) / __ldg(kc + 3 * f + 2) : x;
    } else if (k == TBN_PREP_ORDINAL) {
      o = v;                                                               // level index, -1 unseen
    } else {
      o = (v == (double)__ldg(level + f)) ? 1.0 : 0.0;                     // one-hot
    }
    out[i] = __double2float_rn(o);
  }
}

}  // namespace

extern "C" {

tbn_status tbn_prep_create(const tbn_prep_column* cols, int32_t ncols, int32_t device, tbn_prep** out) {
  if (!out || !cols || ncols < 1) {
    tbn::set_last_error("tbn_prep_create: need >= 1 column");
    return TBN_ERR_CONFIG;
  }
  *out = nullptr;
  std::vector<int> src, kind, level;
  std::vector<double> kc;
  for (int c = 0; c < ncols; ++c) {
    const tbn_prep_column& d = cols[c];
    if (d.kind < TBN_PREP_STANDARDIZE || d.kind > TBN_PREP_ONEHOT) {
      tbn::set_last_error("tbn_prep_create: unknown column kind");
      return TBN_ERR_CONFIG;
    }
    if (d.kind == TBN_PREP_STANDARDIZE && !(d.std != 0.0)) {
      tbn::set_last_error("tbn_prep_create: standardize column with zero std");
      return TBN_ERR_CONFIG;
    }
    const int w = d.kind == TBN_PREP_ONEHOT ? d.width : 1;
    if (w < 1) {
      tbn::set_last_error("tbn_prep_create: one-hot column with no levels");
      return TBN_ERR_CONFIG;
    }
    for (int j = 0; j < w; ++j) {
      src.push_back(c);
      kind.push_back(d.kind);
      level.push_back(j);
      kc.push_back(d.median);
      kc.push_back(d.mean);
      kc.push_back(d.std);
    }
  }
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    tbn::set_last_error("tbn_prep_create: bad device");
    return TBN_ERR_CUDA;
  }
  tbn_prep* p = new tbn_prep();
  p->device = device;
  p->ncols = ncols;
  p->width = (int)src.size();
  const size_t F = src.size();
  cudaError_t e = cudaMalloc(&p->d_src, F * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_kind, F * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_level, F * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_k, 3 * F * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(p->d_src, src.data(), F * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_kind, kind.data(), F * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_level, level.data(), F * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(p->d_k, kc.data(), 3 * F * sizeof(double), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    tbn::set_last_error(std::string("tbn_prep_create: ") + cudaGetErrorString(e));
    tbn_prep_destroy(p);
    return TBN_ERR_CUDA;
  }
  *out = p;
  return TBN_OK;
}

void tbn_prep_destroy(tbn_prep* p) {
  if (!p) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaFree(p->d_src);
  cudaFree(p->d_kind);
  cudaFree(p->d_level);
  cudaFree(p->d_k);
  cudaSetDevice(prev);
  delete p;
}

int32_t tbn_prep_width(const tbn_prep* p) { return p ? p->width : 0; }

tbn_status tbn_preprocess(const tbn_prep* p, const double* codes, int64_t rows, float* out, void* stream) {
  if (!p || rows < 0 || (rows > 0 && (!codes || !out))) {
    tbn::set_last_error("tbn_preprocess: bad arguments");
    return TBN_ERR_INVALID_INPUT;
  }
  if (rows == 0) return TBN_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  const int64_t total = rows * (int64_t)p->width;
  const int64_t want = (total + 255) / 256;
  const int grid = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
  prep_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(codes, rows, p->ncols, p->width, p->d_src, p->d_kind,
                                                      p->d_level, p->d_k, out);
  const cudaError_t e = cudaGetLastError();
  if (prev != p->device) cudaSetDevice(prev);
  if (e != cudaSuccess) {
    tbn::set_last_error(std::string("tbn_preprocess: ") + cudaGetErrorString(e));
    return TBN_ERR_CUDA;
  }
  return TBN_OK;
}

}  // extern "C"
