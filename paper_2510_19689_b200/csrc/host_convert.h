// host_convert.h — host-side f64 <-> f32 conversion for the float64 drop-in
// call, on a persistent worker pool (host_convert.cpp).
#pragma once
#include <cstddef>
#include <functional>

namespace tbn {

// dst[i] = (D)src[i], i < n (AVX2 when available; f64 outputs with streaming stores)
void convert_span(double* dst, const float* src, size_t n);
void convert_span(float* dst, const double* src, size_t n);
void convert_span(float* dst, const float* src, size_t n);

// fn(lo, hi) over [0, n) split across the pool (inline below min_parallel, or
// when another host thread holds the pool)
void host_parallel_for(size_t n, size_t min_parallel, const std::function<void(size_t, size_t)>& fn);

}  // namespace tbn
