// capi.cu — the C ABI of libtabnet_b200.so (include/tabnet_b200.h).
//
// Owns: parameter validation mirroring ModelConfig/TabNetModel (config.py:29-41,
// network.py:110-114, network.py:207-211), the weight packer K0 (f64 params
// dict -> device layouts), the dispatch to the fused forward kernels, and the
// host-buffer path (pinned staging on a per-thread stream) that the
// reference-facing Python apply() and bench.py's e2e leg use.
#include "tabnet_b200.h"
#include "tbn_internal.h"
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <thread>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: free when no profiler is attached

namespace {
// NVTX range for nsys/ncu timelines: forward, H2D, D2H of the host path
// TBN_HOST_TIMING=<ms>: report host-path phases slower than that to stderr
// (development aid for latency tails; off by default)
double host_timing_ms() {
  static const double v = [] {
    const char* e = std::getenv("TBN_HOST_TIMING");
    return e ? std::atof(e) : -1.0;
  }();
  return v;
}
struct NvtxRange {
  explicit NvtxRange(const char* name) : name_(name) {
    nvtxRangePushA(name);
    if (host_timing_ms() >= 0) t0_ = std::chrono::steady_clock::now();
  }
  ~NvtxRange() {
    nvtxRangePop();
    if (host_timing_ms() >= 0) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
      if (ms >= host_timing_ms())
        std::fprintf(stderr, "[tbn host] %s: %.3f ms (thread %zu)\n", name_, ms,
                     std::hash<std::thread::id>()(std::this_thread::get_id()) % 100000);
    }
  }
  const char* name_;
  std::chrono::steady_clock::time_point t0_;
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace
#include "tbn_tc.h"
#include "host_convert.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

namespace {

thread_local std::string g_last_error;

tbn_status fail(tbn_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}
tbn_status cuda_fail(cudaError_t e, const char* where) {
  return fail(TBN_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TBN_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

void tbn::set_last_error(const std::string& msg) { g_last_error = msg; }

struct tbn_model {
  uint64_t id = 0;             // unique per created model (keys the host path's graph cache)
  tbn_config cfg{};
  bool regression = false;     // TBN_CFG_REGRESSION: identity head, logits only
  int precision = TBN_PREC_TF32X3;
  int device = 0;
  int num_sms = 148;
  float* d_simt = nullptr;     // fp32 copies for the CUDA-core kernel
  tbn::SimtParams simt{};
  tbn::TcModel tc{};           // packed tcgen05 operands (kernel_tc.cu)
};

extern "C" {

int32_t tbn_abi_version(void) { return TBN_ABI_VERSION; }
const char* tbn_last_error(void) { return g_last_error.c_str(); }

int32_t tbn_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

tbn_status tbn_device_init(int32_t device) {
  if (device < 0 || device >= tbn_device_count()) return fail(TBN_ERR_CUDA, "no such CUDA device");
  DeviceGuard guard(device);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaFree(nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "context init");
  return TBN_OK;
}

tbn_status tbn_model_create(const tbn_config* cfg, const char* const* names,
                            const double* const* values, const int64_t* sizes,
                            int32_t n_params, const double* norm_mean,
                            const double* norm_var, int32_t precision,
                            int32_t device, tbn_model** out) {
  if (!cfg || !out || (!names && n_params > 0) || !norm_mean || !norm_var)
    return fail(TBN_ERR_CONFIG, "null argument");
  *out = nullptr;
  const tbn_config c = *cfg;
  // ModelConfig.__post_init__ (config.py:29-41)
  if (c.feature_count < 1) return fail(TBN_ERR_CONFIG, "feature_count must be >= 1");
  const bool regression = (c.flags & TBN_CFG_REGRESSION) != 0;
  if (c.flags & ~TBN_CFG_REGRESSION) return fail(TBN_ERR_CONFIG, "unknown config flags");
  if (regression ? c.n_classes != 1 : c.n_classes < 2)
    return fail(TBN_ERR_CONFIG, regression ? "a regression head has n_classes == 1"
                                           : "n_classes must be >= 2");
  if (c.n_d < 1 || c.n_a < 1) return fail(TBN_ERR_CONFIG, "n_d and n_a must be >= 1");
  if (c.n_steps < 1) return fail(TBN_ERR_CONFIG, "n_steps must be >= 1");
  if (!(c.gamma >= 1.0)) return fail(TBN_ERR_CONFIG, "gamma must be >= 1");
  if (precision < TBN_PREC_TF32X3 || precision > TBN_PREC_FP32)
    return fail(TBN_ERR_CONFIG, "unknown precision");
  const int F = c.feature_count, ND = c.n_d, NA = c.n_a, S = c.n_steps, C = c.n_classes;
  const int H = ND + NA, N2 = 2 * H;
  // TabNetModel.__post_init__ (network.py:113-114)
  for (int f = 0; f < F; ++f)
    if (!(norm_var[f] > 0.0)) return fail(TBN_ERR_CONFIG, "normalization variances must be > 0");

  // params dict by name (init_parameters, network.py:81-96)
  std::map<std::string, std::pair<const double*, int64_t>> pm;
  for (int i = 0; i < n_params; ++i) {
    if (!names[i] || !values[i]) return fail(TBN_ERR_CONFIG, "null param entry");
    pm[names[i]] = {values[i], sizes[i]};
  }
  auto need = [&](const std::string& k, int64_t n, const double** p) -> tbn_status {
    auto it = pm.find(k);
    if (it == pm.end()) return fail(TBN_ERR_CONFIG, "missing parameter " + k);
    if (it->second.second != n)
      return fail(TBN_ERR_CONFIG, "parameter " + k + " has " + std::to_string(it->second.second) +
                                      " elements, expected " + std::to_string(n));
    *p = it->second.first;
    return TBN_OK;
  };
  tbn::HostParams hp;
  hp.F = F; hp.ND = ND; hp.NA = NA; hp.S = S; hp.C = C; hp.gamma = c.gamma;
  tbn_status st;
  if ((st = need("shared1_W", (int64_t)F * N2, &hp.sh1_W)) != TBN_OK) return st;
  if ((st = need("shared1_b", N2, &hp.sh1_b)) != TBN_OK) return st;
  if ((st = need("shared2_W", (int64_t)H * N2, &hp.sh2_W)) != TBN_OK) return st;
  if ((st = need("shared2_b", N2, &hp.sh2_b)) != TBN_OK) return st;
  if ((st = need("head_W", (int64_t)ND * C, &hp.head_W)) != TBN_OK) return st;
  if ((st = need("head_b", C, &hp.head_b)) != TBN_OK) return st;
  hp.fc1_W.resize(S + 1); hp.fc1_b.resize(S + 1); hp.fc2_W.resize(S + 1); hp.fc2_b.resize(S + 1);
  hp.att_W.resize(S + 1, nullptr); hp.att_b.resize(S + 1, nullptr);
  for (int s = 0; s <= S; ++s) {
    std::string p = "step" + std::to_string(s) + "_";
    if ((st = need(p + "fc1_W", (int64_t)H * N2, &hp.fc1_W[s])) != TBN_OK) return st;
    if ((st = need(p + "fc1_b", N2, &hp.fc1_b[s])) != TBN_OK) return st;
    if ((st = need(p + "fc2_W", (int64_t)H * N2, &hp.fc2_W[s])) != TBN_OK) return st;
    if ((st = need(p + "fc2_b", N2, &hp.fc2_b[s])) != TBN_OK) return st;
    if (s >= 1) {
      if ((st = need(p + "att_W", (int64_t)NA * F, &hp.att_W[s])) != TBN_OK) return st;
      if ((st = need(p + "att_b", F, &hp.att_b[s])) != TBN_OK) return st;
    }
  }
  hp.norm_mean = norm_mean;
  hp.norm_var = norm_var;

  int ndev = tbn_device_count();
  if (ndev <= 0) return fail(TBN_ERR_CUDA, "no CUDA device available (this engine has no CPU fallback)");
  if (device < 0 || device >= ndev) return fail(TBN_ERR_CONFIG, "device index out of range");
  if (precision != TBN_PREC_FP32 && !tbn::tc_supported(hp, precision))
    return fail(TBN_ERR_UNSUPPORTED, "no tcgen05 kernel instance for this model shape/precision");
  if (precision == TBN_PREC_FP32 && !tbn::simt_supported(F, H, C))
    return fail(TBN_ERR_UNSUPPORTED, "fp32 CUDA-core kernel supports feature_count <= 512, "
                                     "2*(n_d+n_a) <= 256, n_classes <= 32");

  DeviceGuard guard(device);
  tbn_model* m = new tbn_model();
  m->cfg = c;
  m->precision = precision;
  m->regression = regression;
  static std::atomic<uint64_t> next_id{1};
  m->id = next_id++;
  m->device = device;
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);

  // ---- fp32 copies (scale/shift + all params) for the CUDA-core kernel ----
  std::vector<float> buf;
  auto put = [&](const double* src, size_t n) -> size_t {
    size_t off = align_up(buf.size(), 32);
    buf.resize(off + n, 0.0f);
    for (size_t i = 0; i < n; ++i) buf[off + i] = (float)src[i];
    return off;
  };
  std::vector<double> scale(F), shift(F);
  for (int f = 0; f < F; ++f) {
    scale[f] = 1.0 / std::sqrt(norm_var[f] + 1e-8);   // network.py:120
    shift[f] = norm_mean[f];
  }
  size_t o_scale = put(scale.data(), F), o_shift = put(shift.data(), F);
  size_t o_sh1W = put(hp.sh1_W, (size_t)F * N2), o_sh1b = put(hp.sh1_b, N2);
  size_t o_sh2W = put(hp.sh2_W, (size_t)H * N2), o_sh2b = put(hp.sh2_b, N2);
  size_t o_fc1W = 0, o_fc1b = 0, o_fc2W = 0, o_fc2b = 0, o_attW = 0, o_attb = 0;
  size_t o_hW = put(hp.head_W, (size_t)ND * C), o_hb = put(hp.head_b, C);
  // Per-step tensors are stacked densely, (s * H * N2) indexing in the kernel.
  {
    std::vector<float> dense;
    auto dput = [&](const std::vector<const double*>& v, int s0, int s1, size_t n) -> size_t {
      size_t off = align_up(dense.size(), 32);
      dense.resize(off + n * (s1 - s0 + 1), 0.0f);
      for (int s = s0; s <= s1; ++s)
        for (size_t i = 0; i < n; ++i) dense[off + (size_t)(s - s0) * n + i] = (float)v[s][i];
      return off;
    };
    size_t base = align_up(buf.size(), 32);
    o_fc1W = base + dput(hp.fc1_W, 0, S, (size_t)H * N2);
    o_fc1b = base + dput(hp.fc1_b, 0, S, N2);
    o_fc2W = base + dput(hp.fc2_W, 0, S, (size_t)H * N2);
    o_fc2b = base + dput(hp.fc2_b, 0, S, N2);
    o_attW = base + dput(hp.att_W, 1, S, (size_t)NA * F);
    o_attb = base + dput(hp.att_b, 1, S, F);
    buf.resize(base + dense.size());
    std::memcpy(buf.data() + base, dense.data(), dense.size() * sizeof(float));
  }
  cudaError_t e = cudaMalloc(&m->d_simt, buf.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(m->d_simt, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(m->d_simt);
    delete m;
    return cuda_fail(e, "uploading model");
  }
  float* d = m->d_simt;
  tbn::SimtParams& sp = m->simt;
  sp.F = F; sp.ND = ND; sp.NA = NA; sp.S = S; sp.C = C; sp.H = H; sp.gamma = (float)c.gamma;
  sp.scale = d + o_scale; sp.shift = d + o_shift;
  sp.sh1_W = d + o_sh1W; sp.sh1_b = d + o_sh1b; sp.sh2_W = d + o_sh2W; sp.sh2_b = d + o_sh2b;
  sp.fc1_W = d + o_fc1W; sp.fc1_b = d + o_fc1b; sp.fc2_W = d + o_fc2W; sp.fc2_b = d + o_fc2b;
  sp.att_W = d + o_attW; sp.att_b = d + o_attb; sp.head_W = d + o_hW; sp.head_b = d + o_hb;

  // ---- tcgen05 operand packing (K0) ----
  if (precision != TBN_PREC_FP32) {
    std::string err;
    if (!tbn::tc_pack(hp, precision, &m->tc, &err)) {
      cudaFree(m->d_simt);
      delete m;
      if (err.rfind("unsupported:", 0) == 0) return fail(TBN_ERR_UNSUPPORTED, err);
      return fail(TBN_ERR_CUDA, "tcgen05 weight packing failed: " + err);
    }
  }
  *out = m;
  return TBN_OK;
}

void tbn_model_destroy(tbn_model* m) {
  if (!m) return;
  DeviceGuard guard(m->device);
  cudaFree(m->d_simt);
  tbn::tc_free(&m->tc);
  delete m;
}

tbn_status tbn_model_info(const tbn_model* m, tbn_config* cfg, int32_t* precision, int32_t* device) {
  if (!m) return fail(TBN_ERR_CONFIG, "null model");
  if (cfg) *cfg = m->cfg;
  if (precision) *precision = m->precision;
  if (device) *device = m->device;
  return TBN_OK;
}

size_t tbn_workspace_bytes(const tbn_model* m, int64_t rows, uint32_t flags) {
  size_t b = 256;
  if (m && (flags & TBN_FLAG_BATCH_STATS)) b += align_up(2 * (size_t)m->cfg.feature_count * sizeof(float), 256);
  if (m && m->tc.scratch_per_cta) {      // K3 row-tile state: one slice per CTA of the grid
    const int64_t tiles = (rows + 127) / 128;
    const int64_t grid = tiles < m->num_sms ? tiles : m->num_sms;
    b += (size_t)(grid > 0 ? grid : 1) * m->tc.scratch_per_cta;
  }
  return b;
}

tbn_status tbn_forward(const tbn_model* m, const float* x, int64_t rows, uint32_t flags,
                       const tbn_outputs* out, int32_t* err_flag, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!m) return fail(TBN_ERR_CONFIG, "null model");
  if (rows < 0) return fail(TBN_ERR_INVALID_INPUT, "rows must be >= 0");
  if (rows == 0) return TBN_OK;
  if (!x) return fail(TBN_ERR_INVALID_INPUT, "null input");
  NvtxRange nv("tbn_forward");
  if ((flags & TBN_FLAG_NORMALIZED) && (flags & TBN_FLAG_BATCH_STATS)) flags &= ~TBN_FLAG_BATCH_STATS;
  if (workspace_bytes < tbn_workspace_bytes(m, rows, flags) || !workspace)
    return fail(TBN_ERR_CONFIG, "workspace too small");
  DeviceGuard guard(m->device);
  cudaStream_t s = (cudaStream_t)stream;
  tbn::ForwardArgs a{};
  a.x = x;
  a.rows = rows;
  a.normalized = (flags & TBN_FLAG_NORMALIZED) ? 1 : 0;
  a.packed = (flags & TBN_FLAG_PACKED) ? 1 : 0;
  if (out) {
    a.logits = out->logits; a.probs = out->probabilities; a.masks = out->masks;
    a.importance = out->importance; a.pred = out->predicted_class;
    if (m->regression) {        // identity head: the kernels write the logits only
      if (!a.logits) a.logits = a.probs;
      a.probs = nullptr;
      a.pred = nullptr;
    }
  }
  a.err_flag = err_flag;
  if (m->tc.kernel == 3) {               // K3 moves rows with 128-bit accesses
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    if (!al16(a.x) || !al16(a.masks) || !al16(a.importance))
      return fail(TBN_ERR_INVALID_INPUT, "wide-model kernel needs 16-byte aligned x/masks/importance");
  }
  if (m->tc.scratch_per_cta)             // K3 scratch after the batch-stats block
    a.scratch = (float*)((char*)workspace + 256 +
                         ((flags & TBN_FLAG_BATCH_STATS)
                              ? align_up(2 * (size_t)m->cfg.feature_count * sizeof(float), 256) : 0));
  if (flags & TBN_FLAG_BATCH_STATS) {
    float* ss = (float*)((char*)workspace + 256);
    a.scale = ss;
    a.shift = ss + m->cfg.feature_count;
    TBN_CUDA(tbn::launch_batch_stats(x, rows, m->cfg.feature_count, ss, ss + m->cfg.feature_count, s));
  }
  // Development aid: TBN_TRACE=1 records a clock64 timeline of CTA 0 and
  // prints it to stderr after a synchronizing copy (never set in production).
  static const bool trace_on = getenv("TBN_TRACE") != nullptr;
  // TBN_TRACE_MAPPED: the timeline lives in mapped host memory and the host
  // polls it while the kernel runs, so a hung kernel still shows how far it got
  static const bool trace_mapped = getenv("TBN_TRACE_MAPPED") != nullptr;
  static unsigned long long* d_trace = nullptr;
  static unsigned long long* h_trace = nullptr;
  if (trace_mapped && m->precision != TBN_PREC_FP32) {
    if (!h_trace) {
      cudaHostAlloc((void**)&h_trace, 16384 * sizeof(unsigned long long), cudaHostAllocMapped);
      cudaHostGetDevicePointer((void**)&d_trace, h_trace, 0);
    }
    std::memset(h_trace, 0, 16384 * sizeof(unsigned long long));
    a.trace = d_trace;
  } else if (trace_on && m->precision != TBN_PREC_FP32) {
    if (!d_trace) cudaMalloc(&d_trace, 16384 * sizeof(unsigned long long));
    cudaMemsetAsync(d_trace, 0, 16384 * sizeof(unsigned long long), s);
    a.trace = d_trace;
  }
  cudaError_t e;
  if (m->precision == TBN_PREC_FP32)
    e = tbn::launch_simt(m->simt, a, m->num_sms, s);
  else
    e = tbn::launch_tc(m->tc, a, m->num_sms, s);
  if (e != cudaSuccess) return cuda_fail(e, "forward kernel launch");
  if (a.trace && trace_mapped) {
    for (int i = 0; i < 200 && cudaStreamQuery(s) == cudaErrorNotReady; ++i) usleep(50000);
    const bool hung = cudaStreamQuery(s) == cudaErrorNotReady;
    fprintf(stderr, "TRACE rows=%lld %s\n", (long long)rows, hung ? "HUNG" : "done");
    for (int k = 0; k < 16384; ++k)
      if (((volatile unsigned long long*)h_trace)[k]) fprintf(stderr, "TRACE %d %llu\n", k, ((volatile unsigned long long*)h_trace)[k]);
    if (hung) _exit(3);
  } else if (a.trace) {
    std::vector<unsigned long long> h(16384);
    cudaMemcpyAsync(h.data(), d_trace, 16384 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const unsigned long long t0 = h[0];
    fprintf(stderr, "TRACE rows=%lld\n", (long long)rows);
    for (int k = 0; k < 16384; ++k)
      if (h[k]) fprintf(stderr, "TRACE %d %lld\n", k, (long long)(h[k] - t0));
  }
  return TBN_OK;
}

}  // extern "C"

// ------------------------- host-buffer path -------------------------------
// Reference-facing synchronous call with HOST buffers.  Batches up to
// kZeroCopyMax rows (kZeroCopyMaxStaged through the staging) run as ONE kernel
// that reads x from and writes the outputs and the error flag straight into
// page-locked host memory over PCIe (zero-copy: one launch and one
// synchronize, the latency path).  Larger batches are cut into row chunks that
// flow through kNumStreams streams, so chunk i's H2D, chunk i-1's kernel and
// chunk i-2's D2H overlap (PCIe is full duplex).  Page-locked caller buffers
// (cudaHostAlloc / torch pin_memory) are used in place; other buffers (and the
// float64 numpy path) are staged through per-stream pinned memory with the
// f64<->f32 conversion fused into the staging copy.
// Per-row results are bitwise independent of the chunking (invariance contract).
namespace {

constexpr int kNumStreams = 3;
constexpr int64_t kMinChunk = 8192;
// zero-copy up to here: HR end-to-end 2,048 / 8,192 / 32,768 rows 79 / 180 /
// 633 us vs 117 / 253 / 666 us through copy-engine transfers; at 65,536 rows
// the copy engines win (1.22 vs 1.25 ms)
constexpr int64_t kZeroCopyMax = 32768;
// through the staging (float64 apply): HR 8,192 rows 0.66 vs 1.45 ms; above
// 2 * kMinChunk the chunked pipeline overlaps the host conversions with the
// transfers and wins (32,768 rows: 0.95 vs 1.55 ms)
constexpr int64_t kZeroCopyMaxStaged = 2 * kMinChunk;

struct StreamCtx {
  cudaStream_t stream = nullptr;
  void* pin = nullptr;  size_t pin_bytes = 0;
  void* dev = nullptr;  size_t dev_bytes = 0;
  int64_t pending_r0 = -1, pending_rows = 0;   // chunk whose staged outputs await copy-out
};

struct HostCtx {
  StreamCtx s[kNumStreams];
};

void free_host_ctx(int device, HostCtx* c) {
  if (cudaSetDevice(device) != cudaSuccess) {   // runtime already torn down: nothing to free
    cudaGetLastError();
    return;
  }
  for (auto& sc : c->s)
    if (sc.stream) cudaStreamSynchronize(sc.stream);
  for (auto& sc : c->s) {
    if (sc.pin) cudaFreeHost(sc.pin);
    if (sc.dev) cudaFree(sc.dev);
    if (sc.stream) cudaStreamDestroy(sc.stream);
  }
  cudaGetLastError();
  delete c;
}

// Host-path contexts (streams + pinned/device staging) are leased per call
// from a process-wide pool per device: apply() is reentrant and
// concurrent callers never share one, but callers' threads come and go (the
// serving workers of each InferenceService, invariance.py:40-41's fresh
// 32-thread pool per check) while the contexts and their staging stay
// allocated and warm.  Creating a context and growing its staging cost
// 25-330 ms under concurrent traffic (stream creation and cudaFree serialise
// against other threads' work), which per-thread contexts paid on every new
// thread.  The pool holds at most the peak number of concurrent calls.
struct CtxPool {
  std::mutex mu;
  std::vector<HostCtx*> free[tbn::kMaxDevices];
};
CtxPool& ctx_pool() {
  static CtxPool* p = new CtxPool();      // never destroyed: calls may run during exit
  return *p;
}

HostCtx* lease_host_ctx(int device) {
  if (device < 0 || device >= tbn::kMaxDevices) return nullptr;
  {
    std::lock_guard<std::mutex> lk(ctx_pool().mu);
    auto& f = ctx_pool().free[device];
    if (!f.empty()) {
      HostCtx* c = f.back();
      f.pop_back();
      return c;
    }
  }
  NvtxRange nv("tbn_host: context creation");
  HostCtx* c = new HostCtx();
  for (auto& sc : c->s)
    if (cudaStreamCreateWithFlags(&sc.stream, cudaStreamNonBlocking) != cudaSuccess) {
      free_host_ctx(device, c);
      return nullptr;
    }
  return c;
}

void return_host_ctx(int device, HostCtx* c) {
  std::lock_guard<std::mutex> lk(ctx_pool().mu);
  ctx_pool().free[device].push_back(c);
}

struct CtxLease {
  int device;
  HostCtx* hc;
  explicit CtxLease(int d) : device(d), hc(lease_host_ctx(d)) {}
  ~CtxLease() {
    if (hc) return_host_ctx(device, hc);
  }
  CtxLease(const CtxLease&) = delete;
  CtxLease& operator=(const CtxLease&) = delete;
};

// On any early error return from the host path, wait for the chunks already
// queued (their DMAs read/write the per-thread pinned staging) before the
// next call may reuse that staging.
struct DrainOnError {
  HostCtx* hc;
  bool armed = true;
  ~DrainOnError() {
    if (!armed) return;
    for (auto& sc : hc->s) {
      if (sc.stream) cudaStreamSynchronize(sc.stream);
      sc.pending_r0 = -1;
    }
    cudaGetLastError();
  }
};

// Staging grows in steps of 4x from 8 MB (HR: ~7,000 rows) to 128 MB, then in
// 128 MB steps: page-locking
// costs ~2-4 ms per call to cudaMallocHost alone (tools/pin_cost.py) and
// 50-180 ms when it contends with other threads' work inside a serving
// process, so it should happen about once per context.  Requests of a few
// bytes (the error-flag slot of the direct path) stay small.
size_t staging_size(size_t need) {
  if (need <= 4096) return 4096;
  const size_t big = (size_t)128 << 20;        // above: the next multiple of 128 MB (no 4x overshoot)
  if (need > big) return (need + big - 1) / big * big;
  size_t v = (size_t)8 << 20;
  while (v < need) v <<= 2;
  return v;
}
cudaError_t ensure(StreamCtx* c, size_t pin_bytes, size_t dev_bytes) {
  if (c->pin_bytes < pin_bytes) {
    if (c->pin) cudaFreeHost(c->pin);
    c->pin = nullptr; c->pin_bytes = 0;
    const size_t sz = staging_size(pin_bytes);
    cudaError_t e = cudaMallocHost(&c->pin, sz);
    if (e != cudaSuccess) return e;
    c->pin_bytes = sz;
  }
  if (c->dev_bytes < dev_bytes) {
    if (c->dev) cudaFree(c->dev);
    c->dev = nullptr; c->dev_bytes = 0;
    const size_t sz = staging_size(dev_bytes);
    cudaError_t e = cudaMalloc(&c->dev, sz);
    if (e != cudaSuccess) return e;
    c->dev_bytes = sz;
  }
  return cudaSuccess;
}

// the device-side address of page-locked host memory (the same address under
// unified addressing); nullptr for null or unmapped pointers
void* mapped(const void* p) {
  if (!p) return nullptr;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, const_cast<void*>(p), 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return d;
}

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

struct Layout {
  size_t x, logits, probs, masks, imp, pred, err, ws, total;
};

Layout layout_for(const tbn_model* m, int64_t rows, uint32_t flags) {
  const size_t F = m->cfg.feature_count, C = m->cfg.n_classes, S = m->cfg.n_steps, R = rows;
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  // x | err | outputs: a small batch moves [x, err] in one H2D copy (err
  // zeroed in the pinned staging) and [err, outputs] in one D2H copy
  L.x = take(R * F * 4);
  L.err = take(4);
  L.logits = take(R * C * 4);
  L.probs = take(R * C * 4);
  L.masks = take(S * R * F * 4);
  L.imp = take(R * F * 4);
  L.pred = take(R * 4);
  L.ws = take(tbn_workspace_bytes(m, rows, flags));
  L.total = o;
  return L;
}

// A batch of element-wise conversions (dst[i] = (D)src[i]) spread over the
// host worker pool (host_convert.cpp) when large: the float64 apply() path
// converts every output of every chunk (HR @ 65,536: 14 M values).
template <typename D, typename S_>
struct ConvertJob {
  D* dst;
  const S_* src;
  size_t n;
};
template <typename D, typename S_>
void convert_all(const std::vector<ConvertJob<D, S_>>& jobs) {
  size_t total = 0;
  for (const auto& j : jobs) total += j.n;
  // (the pool's wake-up costs more than it saves below ~1 MB: measured on the
  // staged small-batch path, 1,024 HR rows 87 -> 239 us with a 128K-value threshold)
  tbn::host_parallel_for(total, (size_t)1 << 18, [&](size_t lo, size_t hi) {   // global range [lo, hi)
    size_t base = 0;
    for (const auto& j : jobs) {
      const size_t a = lo > base ? lo - base : 0, b = hi - base < j.n ? hi - base : j.n;
      if (hi > base && a < j.n && a < b) tbn::convert_span(j.dst + a, j.src + a, b - a);
      base += j.n;
      if (base >= hi) break;
    }
  });
}

template <typename T, typename OutT>
tbn_status forward_host_impl(const tbn_model* m, const T* x, int64_t rows, uint32_t flags,
                             const OutT* out) {
  if (!m) return fail(TBN_ERR_CONFIG, "null model");
  if (rows < 0) return fail(TBN_ERR_INVALID_INPUT, "rows must be >= 0");
  if (rows == 0) return TBN_OK;
  NvtxRange nv("tbn_forward_host");
  if (!x) return fail(TBN_ERR_INVALID_INPUT, "null input");
  DeviceGuard guard(m->device);
  CtxLease lease(m->device);
  HostCtx* hc = lease.hc;
  if (!hc) return fail(TBN_ERR_CUDA, "cannot create streams");
  const size_t F = m->cfg.feature_count, C = m->cfg.n_classes, S = m->cfg.n_steps;
  OutT o{};
  if (out) o = *out;
  const OutT user = o;
  if (m->regression) {          // identity head: compute the logits only, fill the rest below
    if (!o.logits) o.logits = o.probabilities;
    o.probabilities = nullptr;
    o.predicted_class = nullptr;
  }
  constexpr bool kF32 = sizeof(T) == 4;
  const bool pinned_all = kF32 && is_pinned(x) && is_pinned(o.logits) && is_pinned(o.probabilities) &&
                          is_pinned(o.masks) && is_pinned(o.importance) && is_pinned(o.predicted_class);
  // Up to kZeroCopyMax rows (kZeroCopyMaxStaged through the staging) the kernel
  // itself reads x from and writes the outputs and the error flag into
  // page-locked host memory over PCIe: one launch, no copy-engine transfers.
  // Caller buffers registered without a device mapping take the copy path.
  auto all_mapped = [&]() {
    const void* ps[] = {x, o.logits, o.probabilities, o.masks, o.importance, o.predicted_class};
    for (const void* q : ps)
      if (q && !mapped(q)) return false;
    return true;
  };
  const bool zc = pinned_all ? rows <= kZeroCopyMax && all_mapped() : rows <= kZeroCopyMaxStaged;
  const bool direct = pinned_all;              // outputs land in the caller's buffers (DMA or zero-copy)
  // Batch statistics (negative control) need the whole batch in one call.
  int64_t chunk = rows;
  if (!zc && !(flags & TBN_FLAG_BATCH_STATS) && rows > 2 * kMinChunk) {
    // page-locked caller buffers: 3 chunks; staged (float64) calls: 8 smaller
    // chunks, so the host conversions pipeline with the transfers (HR @ 65,536
    // float64 apply 2.21 -> 2.04 ms; 16 or 32 chunks of >= 2,048 rows measured
    // 3.3-3.8 ms; the fp32 pinned path is the same with 3 or 8)
    const int64_t nch = direct ? kNumStreams : 8;
    const int64_t minc = direct ? kMinChunk : 2048;
    chunk = (rows + nch - 1) / nch;
    chunk = ((chunk + 127) / 128) * 128;
    if (chunk < minc) chunk = minc;
  }
  const Layout L = layout_for(m, chunk, flags);
  DrainOnError drain_guard{hc};
  {
    NvtxRange nv_ensure("tbn_host: staging allocation");
    const int64_t nchunks = (rows + chunk - 1) / chunk;      // streams this call uses
    for (int i = 0; i < kNumStreams; ++i) {
      StreamCtx& sc = hc->s[i];
      if (sc.pending_r0 >= 0) TBN_CUDA(cudaStreamSynchronize(sc.stream));   // (defensive: never left set)
      sc.pending_r0 = -1;
      if (i < nchunks) TBN_CUDA(ensure(&sc, direct ? 256 : L.total, L.total));
    }
  }
  int32_t err_any = 0;
  const size_t err_off = direct ? 0 : L.err;   // pinned landing slot of the chunk's error flag
  // copy a finished chunk's staged outputs into the caller's arrays
  auto drain = [&](StreamCtx& sc) -> tbn_status {
    if (sc.pending_r0 < 0) return TBN_OK;
    NvtxRange nv("tbn_host: D2H wait + output conversion");
    {
      NvtxRange nv_sync("tbn_host: stream synchronize");
      TBN_CUDA(cudaStreamSynchronize(sc.stream));
    }
    char* P = (char*)sc.pin;
    const size_t r0 = sc.pending_r0, n = sc.pending_rows;
    err_any |= *(volatile int32_t*)(P + err_off);
    if (!direct) {
      using OutF = std::remove_pointer_t<decltype(o.logits)>;
      std::vector<ConvertJob<OutF, float>> jobs;
      if (o.logits) jobs.push_back({o.logits + r0 * C, (const float*)(P + L.logits), n * C});
      if (o.probabilities) jobs.push_back({o.probabilities + r0 * C, (const float*)(P + L.probs), n * C});
      if (o.masks)
        for (size_t s = 0; s < S; ++s)
          jobs.push_back({o.masks + (s * rows + r0) * F, (const float*)(P + L.masks) + s * n * F, n * F});
      if (o.importance) jobs.push_back({o.importance + r0 * F, (const float*)(P + L.imp), n * F});
      convert_all(jobs);
      if (o.predicted_class) std::memcpy(o.predicted_class + r0, P + L.pred, n * 4);
    }
    sc.pending_r0 = -1;
    return TBN_OK;
  };
  int ci = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk, ++ci) {
    StreamCtx& sc = hc->s[ci % kNumStreams];
    tbn_status st = drain(sc);
    if (st != TBN_OK) return st;
    const int64_t n = (rows - r0 < chunk) ? rows - r0 : chunk;
    NvtxRange nv_chunk("tbn_host: H2D + forward + D2H enqueue");
    char* P = (char*)sc.pin;
    char* D = (char*)sc.dev;
    cudaStream_t cs = sc.stream;
    if (zc) {
      // one chunk: the kernel reads/writes host memory through its device mapping
      const float* hx;
      tbn_outputs hout{};
      if (direct) {
        hx = (const float*)(const void*)x;
        hout.logits = (float*)(void*)o.logits;
        hout.probabilities = (float*)(void*)o.probabilities;
        hout.masks = (float*)(void*)o.masks;
        hout.importance = (float*)(void*)o.importance;
        hout.predicted_class = o.predicted_class;
      } else {
        convert_all(std::vector<ConvertJob<float, T>>{{(float*)(P + L.x), x, n * F}});
        hx = (const float*)(P + L.x);
        hout.logits = o.logits ? (float*)(P + L.logits) : nullptr;
        hout.probabilities = o.probabilities ? (float*)(P + L.probs) : nullptr;
        hout.masks = o.masks ? (float*)(P + L.masks) : nullptr;
        hout.importance = o.importance ? (float*)(P + L.imp) : nullptr;
        hout.predicted_class = o.predicted_class ? (int32_t*)(P + L.pred) : nullptr;
      }
      int32_t* herr = (int32_t*)(P + err_off);
      *(volatile int32_t*)herr = 0;               // the previous call on this stream has finished
      tbn_outputs dout{};
      const float* dx = (const float*)mapped(hx);
      int32_t* derr = (int32_t*)mapped(herr);
      dout.logits = (float*)mapped(hout.logits);
      dout.probabilities = (float*)mapped(hout.probabilities);
      dout.masks = (float*)mapped(hout.masks);
      dout.importance = (float*)mapped(hout.importance);
      dout.predicted_class = (int32_t*)mapped(hout.predicted_class);
      if (!dx || !derr || (hout.logits && !dout.logits) || (hout.probabilities && !dout.probabilities) ||
          (hout.masks && !dout.masks) || (hout.importance && !dout.importance) ||
          (hout.predicted_class && !dout.predicted_class))
        return fail(TBN_ERR_CUDA, "host buffer not mapped into the device address space");
      st = tbn_forward(m, dx, n, flags, &dout, derr, D + L.ws, L.total - L.ws, cs);
      if (st != TBN_OK) return st;
      sc.pending_r0 = r0;
      sc.pending_rows = n;
      continue;
    }
    if (direct) {
      TBN_CUDA(cudaMemsetAsync(D + L.err, 0, 4, cs));
      TBN_CUDA(cudaMemcpyAsync(D + L.x, (const float*)x + r0 * F, n * F * 4, cudaMemcpyHostToDevice, cs));
    } else {
      convert_all(std::vector<ConvertJob<float, T>>{{(float*)(P + L.x), x + r0 * F, n * F}});
      *(int32_t*)(P + L.err) = 0;                 // [x | err] in one copy
      TBN_CUDA(cudaMemcpyAsync(D + L.x, P + L.x, L.err + 4 - L.x, cudaMemcpyHostToDevice, cs));
    }
    tbn_outputs dout{};
    dout.logits = o.logits ? (float*)(D + L.logits) : nullptr;
    dout.probabilities = o.probabilities ? (float*)(D + L.probs) : nullptr;
    dout.masks = o.masks ? (float*)(D + L.masks) : nullptr;
    dout.importance = o.importance ? (float*)(D + L.imp) : nullptr;
    dout.predicted_class = o.predicted_class ? (int32_t*)(D + L.pred) : nullptr;
    st = tbn_forward(m, (const float*)(D + L.x), n, flags, &dout, (int32_t*)(D + L.err),
                     D + L.ws, L.total - L.ws, cs);
    if (st != TBN_OK) return st;
    if (direct) {
      float* fo;
      if ((fo = (float*)(void*)o.logits)) TBN_CUDA(cudaMemcpyAsync(fo + r0 * C, dout.logits, n * C * 4, cudaMemcpyDeviceToHost, cs));
      if ((fo = (float*)(void*)o.probabilities)) TBN_CUDA(cudaMemcpyAsync(fo + r0 * C, dout.probabilities, n * C * 4, cudaMemcpyDeviceToHost, cs));
      if ((fo = (float*)(void*)o.masks))
        TBN_CUDA(cudaMemcpy2DAsync(fo + r0 * F, rows * F * 4, dout.masks, n * F * 4, n * F * 4, S,
                                   cudaMemcpyDeviceToHost, cs));
      if ((fo = (float*)(void*)o.importance)) TBN_CUDA(cudaMemcpyAsync(fo + r0 * F, dout.importance, n * F * 4, cudaMemcpyDeviceToHost, cs));
      if (o.predicted_class) TBN_CUDA(cudaMemcpyAsync(o.predicted_class + r0, dout.predicted_class, n * 4, cudaMemcpyDeviceToHost, cs));
      TBN_CUDA(cudaMemcpyAsync(P + err_off, D + L.err, 4, cudaMemcpyDeviceToHost, cs));
    } else {
      if (dout.logits) TBN_CUDA(cudaMemcpyAsync(P + L.logits, dout.logits, n * C * 4, cudaMemcpyDeviceToHost, cs));
      if (dout.probabilities) TBN_CUDA(cudaMemcpyAsync(P + L.probs, dout.probabilities, n * C * 4, cudaMemcpyDeviceToHost, cs));
      if (dout.masks) TBN_CUDA(cudaMemcpyAsync(P + L.masks, dout.masks, S * n * F * 4, cudaMemcpyDeviceToHost, cs));
      if (dout.importance) TBN_CUDA(cudaMemcpyAsync(P + L.imp, dout.importance, n * F * 4, cudaMemcpyDeviceToHost, cs));
      if (dout.predicted_class) TBN_CUDA(cudaMemcpyAsync(P + L.pred, dout.predicted_class, n * 4, cudaMemcpyDeviceToHost, cs));
      TBN_CUDA(cudaMemcpyAsync(P + L.err, D + L.err, 4, cudaMemcpyDeviceToHost, cs));
    }
    sc.pending_r0 = r0;
    sc.pending_rows = n;
  }
  for (auto& sc : hc->s) {
    tbn_status st = drain(sc);
    if (st != TBN_OK) return st;
  }
  drain_guard.armed = false;
  if (err_any) return fail(TBN_ERR_INVALID_INPUT, "features must be finite");
  if (m->regression) {
    if (user.probabilities && user.probabilities != o.logits)
      std::memcpy(user.probabilities, o.logits, (size_t)rows * sizeof(*o.logits));
    if (user.predicted_class) std::memset(user.predicted_class, 0, (size_t)rows * 4);
  }
  return TBN_OK;
}

}  // namespace

extern "C" {

tbn_status tbn_forward_host(const tbn_model* m, const float* x, int64_t rows, uint32_t flags,
                            const tbn_outputs* out) {
  return forward_host_impl(m, x, rows, flags, out);
}

tbn_status tbn_forward_host_f64(const tbn_model* m, const double* x, int64_t rows, uint32_t flags,
                                const tbn_outputs_f64* out) {
  return forward_host_impl(m, x, rows, flags, out);
}

tbn_status tbn_sparsemax(const float* z, int64_t rows, int32_t n, float* out, void* stream) {
  if (rows < 0 || n < 1) return fail(TBN_ERR_INVALID_INPUT, "sparsemax input must have length >= 1");
  if (n > 512) return fail(TBN_ERR_UNSUPPORTED, "sparsemax width > 512");
  if (rows == 0) return TBN_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = tbn::launch_sparsemax(z, rows, n, out, nullptr, sms, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sparsemax launch");
  return TBN_OK;
}

tbn_status tbn_partition_mean(const float* v, int64_t per, int32_t partitions, int32_t width,
                              double* out, void* stream) {
  if (per < 1 || partitions < 1 || width < 1)
    return fail(TBN_ERR_INVALID_INPUT, "partition_mean needs rows_per_partition, partitions, width >= 1");
  if (!v || !out) return fail(TBN_ERR_INVALID_INPUT, "null buffer");
  cudaError_t e = tbn::launch_partition_mean(v, per, partitions, width, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "partition_mean launch");
  return TBN_OK;
}

tbn_status tbn_sparsemax_host_f64(const double* z, int64_t rows, int32_t n, double* out) {
  if (rows < 1 || n < 1) return fail(TBN_ERR_INVALID_INPUT, "sparsemax input must have length >= 1");
  if (tbn_device_count() <= 0) return fail(TBN_ERR_CUDA, "no CUDA device available");
  int dev = 0;
  cudaGetDevice(&dev);
  CtxLease lease(dev);
  HostCtx* hc = lease.hc;
  if (!hc) return fail(TBN_ERR_CUDA, "cannot create stream");
  StreamCtx* c = &hc->s[0];
  // float64 end to end (the reference helper's precision, any width)
  const size_t bytes = (size_t)rows * n * 8;
  const size_t total = align_up(bytes, 256) * 2 + 256;
  TBN_CUDA(ensure(c, total, total));
  std::memcpy(c->pin, z, bytes);
  char* D = (char*)c->dev;
  double* dz = (double*)D;
  double* dout = (double*)(D + align_up(bytes, 256));
  int32_t* derr = (int32_t*)(D + 2 * align_up(bytes, 256));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  TBN_CUDA(cudaMemsetAsync(derr, 0, 4, c->stream));
  TBN_CUDA(cudaMemcpyAsync(dz, c->pin, bytes, cudaMemcpyHostToDevice, c->stream));
  TBN_CUDA(tbn::launch_sparsemax_f64(dz, rows, n, dout, derr, sms, c->stream));
  double* po = (double*)((char*)c->pin + align_up(bytes, 256));
  int32_t* perr = (int32_t*)((char*)c->pin + 2 * align_up(bytes, 256));
  TBN_CUDA(cudaMemcpyAsync(po, dout, bytes, cudaMemcpyDeviceToHost, c->stream));
  TBN_CUDA(cudaMemcpyAsync(perr, derr, 4, cudaMemcpyDeviceToHost, c->stream));
  TBN_CUDA(cudaStreamSynchronize(c->stream));
  if (*perr) return fail(TBN_ERR_INVALID_INPUT, "sparsemax input must be finite");
  std::memcpy(out, po, bytes);
  return TBN_OK;
}

}  // extern "C"
