// pack_util.h — host-side helpers of the weight packers (K0): rounding to
// TF32/BF16 and the UMMA canonical K-major no-swizzle block layout.
#pragma once
#include <cstdint>
#include <cstring>
#include <vector>

namespace tbn {
namespace pack {

inline float tf32_rna_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

inline uint16_t bf16_rn_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);       // round to nearest even (finite inputs)
  return (uint16_t)(u >> 16);
}

inline float bf16_to_float(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float y;
  std::memcpy(&y, &u, 4);
  return y;
}

// bf16 variant: 16-bit elements, 8 per 16-byte core-matrix row:
// element index (n/8)*(Kp*8) + (k/8)*64 + (n%8)*8 + (k%8).
inline void pack_block_bf16(std::vector<float>& img, size_t off_floats, const double* W, int Kin, int Nvalid,
                     int N, int Kp, int col_stride, const std::vector<double>* colscale,
                     const double* bias) {
  uint16_t* b = reinterpret_cast<uint16_t*>(img.data() + off_floats);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < Kp; ++k) {
      const size_t idx = (size_t)(n / 8) * (Kp * 8) + (k / 8) * 64 + (n % 8) * 8 + (k % 8);
      double w = (n < Nvalid && k < Kin) ? W[(size_t)k * col_stride + n] : 0.0;
      if (bias && n < Nvalid && k == Kin) w = bias[n];
      if (colscale) w *= (*colscale)[n];
      b[idx] = bf16_rn_host((float)w);
    }
}

// Pack W (Kin x N, row-major, x @ W) into B = W^T as N x Kp K-major canonical
// blocks: float index (n/8)*(Kp*8) + (k/4)*32 + (n%8)*4 + (k%4).  Rows n >= Nvalid
// and columns k >= Kin are zero.
inline void pack_block(std::vector<float>& img, size_t off_floats, const double* W, int Kin, int Nvalid,
                int N, int Kp, bool x3, int col_stride, const std::vector<double>* colscale = nullptr,
                const double* bias = nullptr, bool bf16 = false) {
  if (bf16) {
    pack_block_bf16(img, off_floats, W, Kin, Nvalid, N, Kp, col_stride, colscale, bias);
    return;
  }
  float* hi = img.data() + off_floats;
  float* lo = hi + (size_t)N * Kp;
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < Kp; ++k) {
      const size_t idx = (size_t)(n / 8) * (Kp * 8) + (k / 4) * 32 + (n % 8) * 4 + (k % 4);
      double w = (n < Nvalid && k < Kin) ? W[(size_t)k * col_stride + n] : 0.0;
      if (bias && n < Nvalid && k == Kin) w = bias[n];     // bias row (ones column in A)
      if (colscale) w *= (*colscale)[n];
      float h = tf32_rna_host((float)w);
      hi[idx] = h;
      if (x3) lo[idx] = tf32_rna_host((float)(w - (double)h));
    }
}

// K2 layout: the bias rides in B rows 0 (hi) and 1 (lo) against two ones
// columns at the START of every A operand, so all GEMMs share the ones (written
// once per row tile) and the weight rows follow at k = 2 .. Kin+1; the rest of
// the Kp rows are zero (the A elements there may hold any finite stale value).
// hi = round(b), lo = round(b - hi) in the operand format: the bias reaches
// the fp32 accumulator with ~2^-17 (bf16) / 2^-22 (tf32) relative error
// instead of one rounding.  3xTF32 splits every B element hi/lo already
// (separate lo block), so its row 1 stays zero.
inline void pack_block_k2(std::vector<float>& img, size_t off_floats, const double* W, int Kin, int Nvalid,
                          int N, int Kp, bool x3, int col_stride, const std::vector<double>* colscale,
                          const double* bias, bool bf16) {
  auto val = [&](int n, int k) -> double {     // B[n][k] before the operand rounding
    if (n >= Nvalid) return 0.0;
    const double cs = colscale ? (*colscale)[n] : 1.0;
    if (k >= 2 && k < Kin + 2) return W[(size_t)(k - 2) * col_stride + n] * cs;
    if (k >= 2 || !bias) return 0.0;
    const double b = bias[n] * cs;
    if (x3) return k == 0 ? b : 0.0;             // the 3xTF32 block split carries b's low part
    const double hi = bf16 ? (double)bf16_to_float(bf16_rn_host((float)b)) : (double)tf32_rna_host((float)b);
    return k == 0 ? hi : b - hi;
  };
  if (bf16) {
    uint16_t* b = reinterpret_cast<uint16_t*>(img.data() + off_floats);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < Kp; ++k)
        b[(size_t)(n / 8) * (Kp * 8) + (k / 8) * 64 + (n % 8) * 8 + (k % 8)] = bf16_rn_host((float)val(n, k));
    return;
  }
  float* hi = img.data() + off_floats;
  float* lo = hi + (size_t)N * Kp;
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < Kp; ++k) {
      const size_t idx = (size_t)(n / 8) * (Kp * 8) + (k / 4) * 32 + (n % 8) * 4 + (k % 4);
      const double w = val(n, k);
      const float h = tf32_rna_host((float)w);
      hi[idx] = h;
      if (x3) lo[idx] = tf32_rna_host((float)(w - (double)h));
    }
}

}  // namespace pack
}  // namespace tbn
