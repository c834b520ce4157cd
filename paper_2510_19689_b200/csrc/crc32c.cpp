// crc32c.cpp — CRC-32C (Castagnoli, reflected poly 0x82F63B78) for the .tbnt
// trailer (reference io.py:22-36, a pure-Python table loop that takes 0.89 s on
// the 8.2 MB wide model).  SSE4.2's crc32 instruction computes exactly this
// polynomial; a slicing table is the fallback.
#include <cstddef>
#include <cstdint>
#include <cstring>
#include "tabnet_b200.h"

#if defined(__x86_64__)
#include <nmmintrin.h>
#endif

namespace {
struct Table {
  uint32_t t[256];
  Table() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ 0x82F63B78u : c >> 1;
      t[i] = c;
    }
  }
};
const Table& table() {
  static Table tb;
  return tb;
}
uint32_t crc_sw(const uint8_t* p, size_t n, uint32_t c) {
  const Table& tb = table();
  for (size_t i = 0; i < n; ++i) c = (c >> 8) ^ tb.t[(c ^ p[i]) & 0xFF];
  return c;
}
#if defined(__x86_64__)
__attribute__((target("sse4.2"))) uint32_t crc_hw(const uint8_t* p, size_t n, uint32_t c) {
  uint64_t c64 = c;
  while (n >= 8) {
    uint64_t v;
    std::memcpy(&v, p, 8);
    c64 = _mm_crc32_u64(c64, v);
    p += 8;
    n -= 8;
  }
  uint32_t c32 = (uint32_t)c64;
  while (n--) c32 = _mm_crc32_u8(c32, *p++);
  return c32;
}
#endif
}  // namespace

extern "C" uint32_t tbn_crc32c(const uint8_t* data, size_t n, uint32_t crc) {
  uint32_t c = crc ^ 0xFFFFFFFFu;
#if defined(__x86_64__)
  if (__builtin_cpu_supports("sse4.2")) return crc_hw(data, n, c) ^ 0xFFFFFFFFu;
#endif
  return crc_sw(data, n, c) ^ 0xFFFFFFFFu;
}
