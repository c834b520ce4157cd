// host_convert.cpp — the host side of the float64 drop-in call
// (TabNetModel.apply, network.py:195-267, returns float64 arrays): element-wise
// f64 <-> f32 conversion between the caller's numpy arrays and the pinned
// staging, spread over a persistent worker pool.
//
// HR @ 65,536 moves 9.2 MB of x in and 56 MB of outputs out per call; as f64
// the host side reads 74 MB and writes 121 MB.  The f64 outputs are written
// with non-temporal stores (no read-for-ownership of the destination lines:
// ~1/3 less memory traffic) when the CPU has AVX2.  The pool is created on
// first use and kept: starting 16 threads per chunk cost ~0.1-0.3 ms per call.
#include "host_convert.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <mutex>
#include <thread>
#include <vector>

namespace tbn {
namespace {

bool have_avx2() {
  static const bool v = __builtin_cpu_supports("avx2");
  return v;
}

__attribute__((target("avx2"))) void f32_to_f64_nt(double* dst, const float* src, size_t n) {
  size_t i = 0;
  // scalar head up to a 32-byte aligned destination
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u)) {
    dst[i] = (double)src[i];
    ++i;
  }
  for (; i + 8 <= n; i += 8) {
    const __m256 v = _mm256_loadu_ps(src + i);
    _mm256_stream_pd(dst + i, _mm256_cvtps_pd(_mm256_castps256_ps128(v)));
    _mm256_stream_pd(dst + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(v, 1)));
  }
  for (; i < n; ++i) dst[i] = (double)src[i];
  _mm_sfence();
}

__attribute__((target("avx2"))) void f64_to_f32_avx(float* dst, const double* src, size_t n) {
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const __m128 lo = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i));
    const __m128 hi = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i + 4));
    _mm256_storeu_ps(dst + i, _mm256_set_m128(hi, lo));
  }
  for (; i < n; ++i) dst[i] = (float)src[i];
}

// A fixed set of workers that run one parallel-for at a time; a caller that
// finds the pool busy (another host thread's apply) runs its range inline.
class Pool {
 public:
  Pool() {
    unsigned hw = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("TBN_HOST_THREADS"))      // cap (1 = no workers)
      if (std::atoi(e) > 0 && (unsigned)std::atoi(e) < hw) hw = (unsigned)std::atoi(e);
    nworkers_ = hw > 16 ? 15 : (hw > 1 ? hw - 1 : 0);
    for (unsigned t = 0; t < nworkers_; ++t) th_.emplace_back([this, t] { loop(t + 1); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  unsigned workers() const { return nworkers_; }
  bool try_run(size_t n, const std::function<void(size_t, size_t)>& fn) {
    std::unique_lock<std::mutex> busy(run_m_, std::try_to_lock);
    if (!busy.owns_lock() || nworkers_ == 0) return false;
    const unsigned parts = nworkers_ + 1;
    {
      std::lock_guard<std::mutex> lk(m_);
      fn_ = &fn;
      n_ = n;
      parts_ = parts;
      pending_ = nworkers_;
      ++gen_;
    }
    cv_.notify_all();
    part(0, fn);                                   // the caller takes part 0
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
    return true;
  }

 private:
  void part(unsigned k, const std::function<void(size_t, size_t)>& fn) {
    const size_t per = (n_ + parts_ - 1) / parts_;
    const size_t lo = std::min(n_, (size_t)k * per), hi = std::min(n_, lo + per);
    if (lo < hi) fn(lo, hi);
  }
  void loop(unsigned k) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(size_t, size_t)>* fn;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        fn = fn_;
      }
      part(k, *fn);
      {
        std::lock_guard<std::mutex> lk(m_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::mutex run_m_;                 // one parallel-for at a time
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> th_;
  const std::function<void(size_t, size_t)>* fn_ = nullptr;
  size_t n_ = 0;
  unsigned parts_ = 1, nworkers_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

Pool& pool() {
  // leaked on purpose: worker threads must not be joined from a static
  // destructor after the runtime started tearing down
  static Pool* p = new Pool();
  return *p;
}

}  // namespace

void convert_span(double* dst, const float* src, size_t n) {
  if (have_avx2()) {
    f32_to_f64_nt(dst, src, n);
    return;
  }
  for (size_t i = 0; i < n; ++i) dst[i] = (double)src[i];
}

void convert_span(float* dst, const double* src, size_t n) {
  if (have_avx2()) {
    f64_to_f32_avx(dst, src, n);
    return;
  }
  for (size_t i = 0; i < n; ++i) dst[i] = (float)src[i];
}

void convert_span(float* dst, const float* src, size_t n) { std::copy(src, src + n, dst); }

void host_parallel_for(size_t n, size_t min_parallel, const std::function<void(size_t, size_t)>& fn) {
  if (n == 0) return;
  if (n < min_parallel || !pool().try_run(n, fn)) fn(0, n);
}

}  // namespace tbn
