// kernel_k2_jit.cu — K2 for any model shape: the same kernel template
// (k2_kernel.cuh) compiled at model creation with NVRTC for the model's
// (F, n_d, n_a, n_steps, C, precision) when no prebuilt instance exists
// (the paper's own model F=35/n_d=n_a=8/S=3, a one-hot HR model F=52, ...).
//
// * NVRTC is loaded lazily (dlopen), so the library still loads without it;
//   TBN_NO_JIT=1 disables the path.  The kernel headers are read from the
//   csrc/ directory next to this library (they travel with it).
// * The program holds the kernel instantiation and a one-thread layout query
//   kernel that reports the shape's Cfg constants, so the host packer
//   (k2_pack_layout) uses exactly the offsets the kernel was compiled with.
// * cubins are cached per (shape, precision, header contents) in memory and
//   on disk ($TBN_JIT_CACHE, else ~/.cache/tabnet_b200).
// * A shape the kernel's static limits reject (TMEM columns, shared memory,
//   MMA N <= 256) fails the compile: the model reports UNSUPPORTED and
//   precision="auto" falls back to the CUDA-core kernel.
#include <dlfcn.h>
#include <sys/stat.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "k2_kernel.cuh"
#include "tbn_tc.h"

#ifndef TBN_CUDA_INC
#define TBN_CUDA_INC "/usr/local/cuda/include"
#endif

namespace tbn {
namespace {

// ---- NVRTC, resolved at run time ------------------------------------------
struct Nvrtc {
  typedef int (*Create)(void**, const char*, const char*, int, const char* const*, const char* const*);
  typedef int (*Compile)(void*, int, const char* const*);
  typedef int (*Size)(void*, size_t*);
  typedef int (*Get)(void*, char*);
  typedef int (*AddName)(void*, const char*);
  typedef int (*Lowered)(void*, const char*, const char**);
  typedef int (*Destroy)(void**);
  Create create = nullptr;
  Compile compile = nullptr;
  Size log_size = nullptr, cubin_size = nullptr;
  Get log = nullptr, cubin = nullptr;
  AddName add_name = nullptr;
  Lowered lowered = nullptr;
  Destroy destroy = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    if (const char* off = std::getenv("TBN_NO_JIT"))
      if (off[0] && off[0] != '0') return;
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return;
    n.create = (Nvrtc::Create)dlsym(h, "nvrtcCreateProgram");
    n.compile = (Nvrtc::Compile)dlsym(h, "nvrtcCompileProgram");
    n.log_size = (Nvrtc::Size)dlsym(h, "nvrtcGetProgramLogSize");
    n.log = (Nvrtc::Get)dlsym(h, "nvrtcGetProgramLog");
    n.cubin_size = (Nvrtc::Size)dlsym(h, "nvrtcGetCUBINSize");
    n.cubin = (Nvrtc::Get)dlsym(h, "nvrtcGetCUBIN");
    n.add_name = (Nvrtc::AddName)dlsym(h, "nvrtcAddNameExpression");
    n.lowered = (Nvrtc::Lowered)dlsym(h, "nvrtcGetLoweredName");
    n.destroy = (Nvrtc::Destroy)dlsym(h, "nvrtcDestroyProgram");
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.add_name &&
           n.lowered && n.destroy;
  });
  return n;
}

// directory of this shared library (its csrc/ holds the kernel headers)
std::string lib_dir() {
  Dl_info info{};
  if (dladdr((void*)&lib_dir, &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    const size_t s = p.rfind('/');
    return s == std::string::npos ? std::string(".") : p.substr(0, s);
  }
  return ".";
}

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

const char* kHeaders[] = {"k2_kernel.cuh", "tc_kernel.cuh", "tc_ptx.cuh", "tbn_rtc.h", "tbn_args.h"};
constexpr int kLayoutInts = 33;

// The throughput instance (up to 4 row groups), the latency instance (at
// most 2) and, for even n_d and n_a, the split latency instance (one 8-warp
// group) of one shape, as for the prebuilt shapes (kernel_k2.cu): same
// weight image, same arithmetic.
struct JitK2 {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr, kern_lat = nullptr, kern_split = nullptr;
  K2Layout L;
  int smem_lat = 0, threads_lat = 0, smem_split = 0, threads_split = 0;
  std::mutex attr_mu;
  bool attr_set[kMaxDevices] = {};
};

std::mutex g_mu;
std::map<std::string, std::unique_ptr<JitK2>> g_cache;

std::string cache_dir() {
  if (const char* d = std::getenv("TBN_JIT_CACHE")) return d;
  if (const char* x = std::getenv("XDG_CACHE_HOME")) return std::string(x) + "/tabnet_b200";
  if (const char* home = std::getenv("HOME")) return std::string(home) + "/.cache/tabnet_b200";
  return "/tmp/tabnet_b200";
}

void mkdirs(const std::string& d) {
  std::string cur;
  for (size_t i = 0; i <= d.size(); ++i) {
    if (i == d.size() || d[i] == '/') {
      if (!cur.empty()) mkdir(cur.c_str(), 0755);
    }
    if (i < d.size()) cur.push_back(d[i]);
  }
}

// NVRTC-compile the K2 instance + layout query for one shape; returns the cubin
bool compile(const std::string& src, const std::vector<std::string>& knames, std::vector<char>* cubin,
             std::vector<std::string>* lowered, std::string* log_out) {
  const Nvrtc& nv = nvrtc();
  void* prog = nullptr;
  if (nv.create(&prog, src.c_str(), "tbn_k2_jit.cu", 0, nullptr, nullptr) != 0) {
    *log_out = "nvrtcCreateProgram failed";
    return false;
  }
  for (const std::string& k : knames) nv.add_name(prog, k.c_str());
  const std::string inc_csrc = "-I" + lib_dir() + "/csrc";
  const char* cuda_inc_env = std::getenv("TBN_CUDA_INC");
  const std::string inc_cuda = std::string("-I") + (cuda_inc_env ? cuda_inc_env : TBN_CUDA_INC);
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo", "-DTBN_NVRTC",
                        inc_csrc.c_str(), inc_cuda.c_str(), "-diag-suppress=179,39,549"};
  const int rc = nv.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  std::string log(ls, '\0');
  if (ls) nv.log(prog, &log[0]);
  *log_out = log;
  bool ok = rc == 0;
  if (ok) {
    size_t n = 0;
    nv.cubin_size(prog, &n);
    cubin->resize(n);
    nv.cubin(prog, cubin->data());
    lowered->clear();
    for (const std::string& k : knames) {
      const char* low = nullptr;
      ok = ok && nv.lowered(prog, k.c_str(), &low) == 0 && low;
      if (ok) lowered->push_back(low);
    }
  }
  nv.destroy(&prog);
  return ok;
}

JitK2* get_or_build(const HostParams& hp, int prec, std::string* err) {
  const std::string dir = lib_dir() + "/csrc/";
  std::string hdrs;
  for (const char* h : kHeaders) hdrs += read_file(dir + h);
  if (hdrs.empty()) {
    *err = "unsupported: kernel headers not found in " + dir;
    return nullptr;
  }
  char shape[128];
  std::snprintf(shape, sizeof(shape), "%d, %d, %d, %d, %d, %d", hp.F, hp.ND, hp.NA, hp.S, hp.C, prec);
  const std::string cfg = std::string("tbn::k2::Cfg<") + shape + ">";
  const std::string cfl = std::string("tbn::k2::Cfg<") + shape + ", 2>";
  const std::string cfs = std::string("tbn::k2::Cfg<") + shape + ", 1, true>";
  // the split instance where its halves are even; dropped again if it does not
  // compile for the shape (e.g. no room for its staging next to a weight ring)
  bool split = hp.ND % 2 == 0 && hp.NA % 2 == 0;
  std::vector<std::string> knames;
  std::string source, key;
  auto make_source = [&]() {
    knames = {"tbn::k2::tabnet_rowthread<" + cfg + ">", "tbn::k2::tabnet_rowthread<" + cfl + ">"};
    if (split) knames.push_back("tbn::k2::tabnet_rowthread<" + cfs + ">");
    std::ostringstream src;
    src << "#include \"k2_kernel.cuh\"\n"
        << "typedef " << cfg << " JCF;\n"
        << "typedef " << cfl << " JCL;\n"
        << "static_assert(JCF::IMG_BYTES == JCL::IMG_BYTES && JCF::O_ATT == JCL::O_ATT && JCF::O_FC2 == JCL::O_FC2 &&\n"
        << "              JCF::C_HB == JCL::C_HB, \"the latency instance must read the same weight image\");\n"
        << "template __global__ void tbn::k2::tabnet_rowthread<JCF>(tbn::k2::Params, tbn::ForwardArgs);\n"
        << "template __global__ void tbn::k2::tabnet_rowthread<JCL>(tbn::k2::Params, tbn::ForwardArgs);\n";
    if (split)
      src << "typedef " << cfs << " JCS;\n"
          << "static_assert(JCF::IMG_BYTES == JCS::IMG_BYTES && JCF::O_ATT == JCS::O_ATT && JCF::O_FC2 == JCS::O_FC2 &&\n"
          << "              JCF::C_HB == JCS::C_HB, \"the split instance must read the same weight image\");\n"
          << "template __global__ void tbn::k2::tabnet_rowthread<JCS>(tbn::k2::Params, tbn::ForwardArgs);\n";
    src << "extern \"C\" __global__ void tbn_k2_layout(int* o) {\n"
        << "  const int v[] = {JCF::F, JCF::ND, JCF::NA, JCF::S, JCF::C, JCF::X3, JCF::BF, JCF::H, JCF::N2, JCF::NP,\n"
        << "    JCF::K1, JCF::KHID, JCF::KATT, JCF::FN, JCF::C_SCALE, JCF::C_SHIFT, JCF::C_HW, JCF::C_HB,\n"
        << "    JCF::O_SH1, JCF::O_SH2, JCF::O_FC1, JCF::O_FC2, JCF::O_ATT, tbn::tc::rup(JCF::B_HID, 128),\n"
        << "    tbn::tc::rup(JCF::B_ATT, 128), JCF::IMG_BYTES, JCF::SMEM_BYTES, JCF::THREADS,\n"
        << "    JCL::SMEM_BYTES, JCL::THREADS, JCL::NG, "
        << (split ? "JCS::SMEM_BYTES, JCS::THREADS" : "0, 0") << "};\n"
        << "  for (int i = 0; i < " << kLayoutInts << "; ++i) o[i] = v[i];\n}\n";
    source = src.str();
    key = source + "|" + hdrs;
  };
  make_source();

  std::lock_guard<std::mutex> lk(g_mu);
  {
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second.get();
  }

  const std::string cdir = cache_dir();
  std::string cpath, npath;
  auto set_paths = [&]() {
    char hex[32];
    std::snprintf(hex, sizeof(hex), "%016llx", (unsigned long long)fnv1a(key));
    cpath = cdir + "/k2_" + hex + ".cubin";
    npath = cdir + "/k2_" + hex + ".name";
  };
  set_paths();
  std::vector<char> cubin;
  std::vector<std::string> lowered;
  if (split && read_file(cpath).empty()) {
    // a shape whose split instance failed to compile before is cached without it
    split = false;
    make_source();
    set_paths();
    if (read_file(cpath).empty()) {
      split = true;
      make_source();
      set_paths();
    }
  }
  {
    const std::string c = read_file(cpath), nm = read_file(npath);
    std::istringstream names(nm);
    for (std::string line; std::getline(names, line);)
      if (!line.empty()) lowered.push_back(line);
    if (!c.empty() && lowered.size() == knames.size()) cubin.assign(c.begin(), c.end());
    else lowered.clear();
  }
  if (cubin.empty()) {
    if (!nvrtc().ok) {
      *err = "unsupported: no prebuilt K2 instance for this shape and NVRTC is unavailable";
      return nullptr;
    }
    std::string log;
    bool ok = compile(source, knames, &cubin, &lowered, &log);
    if (!ok && split) {                     // retry without the split instance
      split = false;
      make_source();
      set_paths();
      ok = compile(source, knames, &cubin, &lowered, &log);
    }
    if (!ok) {
      *err = "unsupported: K2 does not compile for this shape: " + log.substr(0, 600);
      return nullptr;
    }
    mkdirs(cdir);
    std::ofstream(cpath, std::ios::binary).write(cubin.data(), (std::streamsize)cubin.size());
    {
      std::ofstream nf(npath, std::ios::binary);
      for (const std::string& l : lowered) nf << l << "\n";
    }
  }
  std::unique_ptr<JitK2> j(new JitK2());
  cudaError_t e = cudaLibraryLoadData(&j->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&j->kern, j->lib, lowered[0].c_str());
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&j->kern_lat, j->lib, lowered[1].c_str());
  if (e == cudaSuccess && split) e = cudaLibraryGetKernel(&j->kern_split, j->lib, lowered[2].c_str());
  cudaKernel_t q = nullptr;
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&q, j->lib, "tbn_k2_layout");
  int* d = nullptr;
  int h[kLayoutInts] = {};
  if (e == cudaSuccess) e = cudaMalloc(&d, sizeof(h));
  if (e == cudaSuccess) {
    void* args[] = {&d};
    e = cudaLaunchKernel((const void*)q, dim3(1), dim3(1), args, 0, nullptr);
  }
  if (e == cudaSuccess) e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (d) cudaFree(d);
  if (e != cudaSuccess) {
    *err = std::string("JIT K2 load: ") + cudaGetErrorString(e);
    if (j->lib) cudaLibraryUnload(j->lib);
    return nullptr;
  }
  K2Layout& L = j->L;
  int i = 0;
  L.F = h[i++]; L.ND = h[i++]; L.NA = h[i++]; L.S = h[i++]; L.C = h[i++];
  L.X3 = h[i++] != 0; L.BF = h[i++] != 0; L.H = h[i++]; L.N2 = h[i++]; L.NP = h[i++];
  L.K1 = h[i++]; L.KHID = h[i++]; L.KATT = h[i++]; L.FN = h[i++];
  L.C_SCALE = h[i++]; L.C_SHIFT = h[i++]; L.C_HW = h[i++]; L.C_HB = h[i++];
  L.O_SH1 = h[i++]; L.O_SH2 = h[i++]; L.O_FC1 = h[i++]; L.O_FC2 = h[i++]; L.O_ATT = h[i++];
  L.HBR = h[i++]; L.ABR = h[i++]; L.IMG_BYTES = h[i++]; L.SMEM_BYTES = h[i++]; L.THREADS = h[i++];
  j->smem_lat = h[i++];
  j->threads_lat = h[i++];
  i++;                                      // JCL::NG (= threads_lat / 128)
  j->smem_split = h[i++];
  j->threads_split = h[i++];
  JitK2* raw = j.get();
  g_cache[key] = std::move(j);
  return raw;
}

int tc_prec(int precision) {
  return precision == 0 ? tc::kPrecTF32x3 : precision == 1 ? tc::kPrecTF32 : precision == 2 ? tc::kPrecBF16 : -1;
}

}  // namespace

bool k2_jit_available() { return nvrtc().ok; }

bool k2_jit_pack(const HostParams& hp, int precision, TcModel* out, std::string* err) {
  const int prec = tc_prec(precision);
  if (prec < 0) {
    if (err) *err = "unsupported: precision";
    return false;
  }
  std::string e;
  JitK2* j = get_or_build(hp, prec, &e);
  if (!j) {
    if (err) *err = e;
    return false;
  }
  out->kernel = 2;
  out->precision = precision;
  out->shape_id = -1;
  out->jit = j;
  return k2_pack_layout(j->L, hp, out, err);
}

cudaError_t k2_jit_launch(const TcModel& m, const ForwardArgs& a, int num_sms, cudaStream_t stream) {
  JitK2* j = const_cast<JitK2*>(static_cast<const JitK2*>(m.jit));
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  {
    std::lock_guard<std::mutex> lk(j->attr_mu);
    if (!j->attr_set[dev]) {
      e = cudaFuncSetAttribute((const void*)j->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, j->L.SMEM_BYTES);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute((const void*)j->kern_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, j->smem_lat);
      if (e == cudaSuccess && j->kern_split)
        e = cudaFuncSetAttribute((const void*)j->kern_split, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 j->smem_split);
      if (e != cudaSuccess) return e;
      j->attr_set[dev] = true;
    }
  }
  // the same geometry and instance choice as the prebuilt instances
  // (kernel_k2.cu launch_k2_impl)
  auto grid_for = [&](int64_t ng) {
    const int64_t nq = a.packed ? (a.rows + 128 * ng - 1) / (128 * ng) : (a.rows + 127) / 128;
    return (int)(nq < num_sms ? nq : num_sms);
  };
  const int64_t ng = j->L.THREADS / 128, ng_lat = j->threads_lat / 128;
  const void* kern = (const void*)j->kern;
  int threads = j->L.THREADS, smem = j->L.SMEM_BYTES, grid = grid_for(ng);
  static const bool nosplit = std::getenv("TBN_K2_NO_SPLIT") != nullptr;   // development A/B only
  if ((ng_lat < ng || j->kern_split) && !a.packed) {
    const int gl = grid_for(ng_lat);
    const int64_t rpc = (((a.rows + gl - 1) / gl) + 3) & ~(int64_t)3;
    if (j->kern_split && rpc <= 128 && !nosplit) {
      kern = (const void*)j->kern_split;
      threads = j->threads_split;
      smem = j->smem_split;
      grid = gl;
    } else if (ng_lat < ng && (rpc + 127) / 128 <= ng_lat) {
      kern = (const void*)j->kern_lat;
      threads = j->threads_lat;
      smem = j->smem_lat;
      grid = gl;
    }
  }
  k2::Params p = *(const k2::Params*)m.params;
  ForwardArgs fa = a;
  void* args[] = {&p, &fa};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL, as the prebuilt K2
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, kern, args);
}

}  // namespace tbn
