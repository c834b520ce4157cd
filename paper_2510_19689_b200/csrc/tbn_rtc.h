// tbn_rtc.h — the few standard names the kernel headers use, from the host
// C++ library under nvcc and from libcu++ (cuda/std) under NVRTC, which has
// no host standard library.
#pragma once
#ifdef __CUDACC_RTC__
#include <cuda/std/cstdint>
#include <cuda/std/type_traits>
#include <cuda/std/limits>
using cuda::std::int32_t;
using cuda::std::int64_t;
using cuda::std::uint8_t;
using cuda::std::uint16_t;
using cuda::std::uint32_t;
using cuda::std::uint64_t;
using cuda::std::uintptr_t;
namespace std {
using cuda::std::integral_constant;
using cuda::std::is_same;
}  // namespace std
#ifndef INFINITY
#define INFINITY (__int_as_float(0x7f800000))
#endif
#else
#include <cmath>
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#endif
