// jit.cu -- NVRTC specialisation of the step kernels on a scheme's bit-pack layout.
//
// At qmpm_create the runtime generates `struct Spec` (the layout as compile-time
// constants) and compiles step_kernels.cuh for sm_100a with NVRTC; the cubin is
// loaded with the driver API (entry points resolved through the runtime, so the
// library has no link-time dependency on libcuda or libnvrtc).  Modules are cached
// per process by their generated source.
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>

#include "jit.h"

namespace qmpm {

#include "jit_sources.inc"  // kSrc* (build.py JIT_HEADERS)

namespace {

struct Driver {
  decltype(&cuModuleLoadData) moduleLoadData = nullptr;
  decltype(&cuModuleGetFunction) moduleGetFunction = nullptr;
  decltype(&cuFuncSetAttribute) funcSetAttribute = nullptr;
  decltype(&cuLaunchKernel) launchKernel = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occupancy = nullptr;
  decltype(&cuFuncGetAttribute) funcGetAttribute = nullptr;
  decltype(&cuModuleGetGlobal) moduleGetGlobal = nullptr;
  decltype(&cuMemcpyDtoH) memcpyDtoH = nullptr;
  bool ok = false;
};

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) logSize = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubinSize = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) errstr = nullptr;
  bool ok = false;
};

std::mutex g_mu;
Driver g_drv;
Nvrtc g_rtc;

template <class T>
bool entry(const char* name, T& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return false;
  fn = reinterpret_cast<T>(p);
  return true;
}

bool init_driver(std::string& err) {
  if (g_drv.ok) return true;
  bool ok = entry("cuModuleLoadData", g_drv.moduleLoadData) && entry("cuModuleGetFunction", g_drv.moduleGetFunction) &&
            entry("cuFuncSetAttribute", g_drv.funcSetAttribute) && entry("cuLaunchKernel", g_drv.launchKernel) &&
            entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", g_drv.occupancy) &&
            entry("cuFuncGetAttribute", g_drv.funcGetAttribute) &&
            entry("cuModuleGetGlobal", g_drv.moduleGetGlobal) && entry("cuMemcpyDtoH", g_drv.memcpyDtoH);
  if (!ok) {
    err = "could not resolve CUDA driver entry points";
    return false;
  }
  g_drv.ok = true;
  return true;
}

template <class T>
bool sym(void* h, const char* name, T& fn) {
  fn = reinterpret_cast<T>(dlsym(h, name));
  return fn != nullptr;
}

bool init_nvrtc(std::string& err) {
  if (g_rtc.ok) return true;
  const char* cands[] = {"/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"};
  void* h = nullptr;
  for (const char* c : cands)
    if ((h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) {
    err = "libnvrtc.so.12 not found (NVRTC is required to specialise the step kernels)";
    return false;
  }
  bool ok = sym(h, "nvrtcCreateProgram", g_rtc.create) && sym(h, "nvrtcCompileProgram", g_rtc.compile) &&
            sym(h, "nvrtcGetProgramLogSize", g_rtc.logSize) && sym(h, "nvrtcGetProgramLog", g_rtc.log) &&
            sym(h, "nvrtcGetCUBINSize", g_rtc.cubinSize) && sym(h, "nvrtcGetCUBIN", g_rtc.cubin) &&
            sym(h, "nvrtcDestroyProgram", g_rtc.destroy) && sym(h, "nvrtcGetErrorString", g_rtc.errstr);
  if (!ok) {
    err = "incomplete libnvrtc";
    return false;
  }
  g_rtc.ok = true;
  return true;
}

}  // namespace

// The next step's sort key needs base = floor(fl(fl(u Delta) inv_dx) - 1/2) of every x code
// u.  When Delta and inv_dx are powers of two, the FIXED x fields have no offset and take
// the packed fast encode (width <= 23, so |u| < 2^22), every step is exact and base =
// (u - 2^(k-1)) >> k with 2^-k = Delta inv_dx: the same integer, from the code.
int integer_key_shift(int dim, const LayoutDev& L, float inv_dx) {
  auto log2_exact = [](double v, int& e) {
    int ex = 0;
    if (!(v > 0.0) || std::frexp(v, &ex) != 0.5) return false;
    e = ex - 1;
    return true;
  };
  int k = -1;
  for (int a = 0; a < dim; ++a) {
    const FieldDev& f = L.s[a];
    int ed = 0, ei = 0;
    if (!L.dither || f.kind != kKindFixed || f.width > 23 || f.offset != 0.0f) return 0;
    if (!log2_exact((double)f.delta, ed) || !log2_exact((double)inv_dx, ei)) return 0;
    const int ka = -(ed + ei);
    if (ka < 1 || ka > 24 || (k >= 0 && ka != k)) return 0;
    k = ka;
  }
  return k < 0 ? 0 : k;
}

std::string spec_source(int dim, int material, const LayoutDev& L, int p2g_warps, int g2p_warps, int p2g_minb,
                        int g2p_minb, int xk, bool slab) {
  std::string s;
  char buf[1024];
  const int ns = (int)L.ns;
  snprintf(buf, sizeof(buf),
           "struct Spec {\n  static constexpr int D = %d, MAT = %d, NS = %d, W = %u, SW = %u;\n"
           "  static constexpr int P2G_WARPS = %d, G2P_WARPS = %d, P2G_MINB = %d, G2P_MINB = %d;\n"
           "  static constexpr unsigned XMASK = %uu;\n  static constexpr int XK = %d;\n"
           "  static constexpr bool SLAB = %s;\n"
           "  static constexpr bool DITHER = %s, COUNTERS = %s, RANGES = %s;\n",
           dim, material, ns, L.W, L.SW, p2g_warps, g2p_warps, p2g_minb, g2p_minb, L.xword_mask, xk,
           slab ? "true" : "false",
           L.dither ? "true" : "false",
           L.counters ? "true" : "false", L.ranges ? "true" : "false");
  s += buf;
  auto ints = [&](const char* name, auto get) {
    s += "  __host__ __device__ static constexpr int ";
    s += name;
    s += "(int i) {\n    constexpr int a[" + std::to_string(ns) + "] = {";
    for (int i = 0; i < ns; ++i) s += std::to_string(get(L.s[i])) + (i + 1 < ns ? ", " : "");
    s += "};\n    return a[i];\n  }\n";
  };
  auto floats = [&](const char* name, auto get) {
    s += "  __host__ __device__ static constexpr float ";
    s += name;
    s += "(int i) {\n    constexpr float a[" + std::to_string(ns) + "] = {";
    for (int i = 0; i < ns; ++i) {
      snprintf(buf, sizeof(buf), "%af", (double)get(L.s[i]));
      s += buf;
      s += (i + 1 < ns ? ", " : "");
    }
    s += "};\n    return a[i];\n  }\n";
  };
  ints("word", [](const FieldDev& f) { return (int)f.word; });
  ints("shift", [](const FieldDev& f) { return (int)f.shift; });
  ints("width", [](const FieldDev& f) { return (int)f.width; });
  ints("kind", [](const FieldDev& f) { return (int)f.kind; });
  ints("idx", [](const FieldDev& f) { return (int)f.idx; });
  ints("ebits", [](const FieldDev& f) { return (int)f.ebits; });
  ints("gword", [](const FieldDev& f) { return (int)f.gword; });
  ints("gshift", [](const FieldDev& f) { return (int)f.gshift; });
  ints("glead", [](const FieldDev& f) { return f.kind == kKindShared ? (int)f.glead : -1; });
  floats("delta", [](const FieldDev& f) { return f.delta; });
  floats("inv_delta", [](const FieldDev& f) { return f.inv_delta; });
  floats("offset", [](const FieldDev& f) { return f.offset; });
  s += "  static constexpr int NSPEC = NS;\n};\n#include \"step_kernels.cuh\"\n";
  return s;
}

namespace {
std::map<std::string, CUmodule> g_modules;

// Compile `src` (which #includes the embedded headers) for sm_100a with NVRTC and load
// it; modules are cached per process by (device, QMPM_JIT_OPTS, source).  g_mu held.
cudaError_t compile_module(const std::string& src, const char* prog_name, CUmodule& mod, std::string& log,
                           std::string& err) {
  int dev = 0;
  cudaGetDevice(&dev);
  const char* jopts = getenv("QMPM_JIT_OPTS");
  const std::string key = std::to_string(dev) + "\n" + (jopts ? jopts : "") + "\n" + src;
  auto it = g_modules.find(key);
  if (it != g_modules.end()) {
    mod = it->second;
    return cudaSuccess;
  }
  if (!init_driver(err) || !init_nvrtc(err)) return cudaErrorNotSupported;
  cudaFree(nullptr);  // make sure the primary context is current
  nvrtcProgram prog;
  const char* hdrs[] = {kSrcDevice, kSrcCommon, kSrcField, kSrcStep, kSrcRecord, kSrcCodec, kSrcSmoke};
  const char* names[] = {"qmpm_device.cuh",  "mpm_common.cuh",    "field_codec.cuh",  "step_kernels.cuh",
                         "codec_record.cuh", "codec_kernels.cuh", "smoke_kernels.cuh"};
  nvrtcResult r = g_rtc.create(&prog, src.c_str(), prog_name, 7, hdrs, names);
  if (r != NVRTC_SUCCESS) {
    err = std::string("nvrtcCreateProgram: ") + g_rtc.errstr(r);
    return cudaErrorInvalidSource;
  }
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true",
                                   "-DQMPM_JIT=1"};
  // QMPM_JIT_OPTS: extra space-separated NVRTC options (tuning runs only, e.g. -DQMPM_SEG_L=24)
  std::vector<std::string> extra;
  if (jopts) {
    std::string e(jopts), tok;
    for (char ch : e + " ") {
      if (ch == ' ') {
        if (!tok.empty()) extra.push_back(tok);
        tok.clear();
      } else {
        tok += ch;
      }
    }
  }
  for (auto& x : extra) opts.push_back(x.c_str());
  r = g_rtc.compile(prog, (int)opts.size(), opts.data());
  size_t ls = 0;
  g_rtc.logSize(prog, &ls);
  log.assign(ls, '\0');
  if (ls) g_rtc.log(prog, &log[0]);
  if (r != NVRTC_SUCCESS) {
    err = std::string("NVRTC compile failed: ") + g_rtc.errstr(r) + "\n" + log;
    g_rtc.destroy(&prog);
    return cudaErrorInvalidSource;
  }
  size_t n = 0;
  g_rtc.cubinSize(prog, &n);
  std::vector<char> cubin(n);
  g_rtc.cubin(prog, cubin.data());
  g_rtc.destroy(&prog);
  CUresult cr = g_drv.moduleLoadData(&mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    err = "cuModuleLoadData failed (" + std::to_string((int)cr) + ")";
    return cudaErrorInvalidKernelImage;
  }
  g_modules[key] = mod;
  return cudaSuccess;
}
}  // namespace

cudaError_t jit_get(const std::string& src, JitModule& out, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  JitModule m{};
  std::string log;
  CUmodule mod;
  cudaError_t e = compile_module(src, "qmpm_step_spec.cu", mod, log, err);
  if (e) return e;
  m.module = mod;
  if (g_drv.moduleGetFunction(&m.bin_count, mod, "qmpm_bin_count") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&m.p2g, mod, "qmpm_p2g") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&m.g2p, mod, "qmpm_g2p") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&m.append, mod, "qmpm_append") != CUDA_SUCCESS) {
    err = "JIT module lacks a kernel";
    return cudaErrorSymbolNotFound;
  }
  auto regs = [&](CUfunction f) {
    int v = 0;
    g_drv.funcGetAttribute(&v, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
    return v;
  };
  {
    CUdeviceptr gp;
    size_t gb = 0;
    unsigned sz[2] = {0, 0};
    if (g_drv.moduleGetGlobal(&gp, &gb, mod, "qmpm_smem_per_warp") != CUDA_SUCCESS || gb != sizeof(sz) ||
        g_drv.memcpyDtoH(sz, gp, sizeof(sz)) != CUDA_SUCCESS) {
      err = "JIT module lacks qmpm_smem_per_warp";
      return cudaErrorSymbolNotFound;
    }
    m.smem_warp_p2g = sz[0];
    m.smem_warp_g2p = sz[1];
  }
  m.regs_p2g = regs(m.p2g);
  m.regs_g2p = regs(m.g2p);
  m.log = log;
  out = m;
  return cudaSuccess;
}

std::string codec_spec_struct(const char* name, const CodecDev& C, bool dither, bool counters, int wv, int vv) {
  std::string s;
  char buf[512];
  const int nf = (int)C.nf;
  snprintf(buf, sizeof(buf),
           "struct %s {\n  static constexpr int NF = %d, W = %u, STRIDE = %u, WV = %d, VV = %d;\n"
           "  static constexpr bool DITHER = %s, COUNTERS = %s;\n",
           name, nf, C.W, C.stride, wv, vv, dither ? "true" : "false", counters ? "true" : "false");
  s += buf;
  auto ints = [&](const char* name, auto get) {
    s += "  __host__ __device__ static constexpr int ";
    s += name;
    s += "(int i) {\n    constexpr int a[" + std::to_string(nf) + "] = {";
    for (int i = 0; i < nf; ++i) s += std::to_string(get(C.f[i])) + (i + 1 < nf ? ", " : "");
    s += "};\n    return a[i];\n  }\n";
  };
  auto floats = [&](const char* name, auto get) {
    s += "  __host__ __device__ static constexpr float ";
    s += name;
    s += "(int i) {\n    constexpr float a[" + std::to_string(nf) + "] = {";
    for (int i = 0; i < nf; ++i) {
      snprintf(buf, sizeof(buf), "%af", (double)get(C.f[i]));
      s += buf;
      s += (i + 1 < nf ? ", " : "");
    }
    s += "};\n    return a[i];\n  }\n";
  };
  ints("word", [](const FieldDev& f) { return (int)f.word; });
  ints("shift", [](const FieldDev& f) { return (int)f.shift; });
  ints("width", [](const FieldDev& f) { return (int)f.width; });
  ints("kind", [](const FieldDev& f) { return (int)f.kind; });
  ints("idx", [](const FieldDev& f) { return (int)f.idx; });
  ints("col", [](const FieldDev& f) { return (int)f.col; });
  ints("ebits", [](const FieldDev& f) { return (int)f.ebits; });
  ints("gword", [](const FieldDev& f) { return (int)f.gword; });
  ints("gshift", [](const FieldDev& f) { return (int)f.gshift; });
  ints("glead", [](const FieldDev& f) { return f.kind == kKindShared ? (int)f.glead : -1; });
  floats("delta", [](const FieldDev& f) { return f.delta; });
  floats("inv_delta", [](const FieldDev& f) { return f.inv_delta; });
  floats("offset", [](const FieldDev& f) { return f.offset; });
  s += "  static constexpr int NSPEC = NF;\n};\n";
  return s;
}

std::string codec_spec_source(const CodecDev& C, bool dither, bool counters, int wv, int vv) {
  return codec_spec_struct("Spec", C, dither, counters, wv, vv) + "#include \"codec_kernels.cuh\"\n";
}

std::string smoke_spec_source(const CodecDev& U, const CodecDev& P, int wvu, int wvp) {
  return codec_spec_struct("SpecU", U, U.dither != 0, false, wvu, 1) +
         codec_spec_struct("SpecP", P, P.dither != 0, false, wvp, 1) + "#include \"smoke_kernels.cuh\"\n";
}

cudaError_t jit_smoke(const std::string& src, SmokeJit& out, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::string log;
  CUmodule mod;
  cudaError_t e = compile_module(src, "qsmoke_spec.cu", mod, log, err);
  if (e) return e;
  if (g_drv.moduleGetFunction(&out.advect_u, mod, "qsmoke_advect_u") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.advect_refl, mod, "qsmoke_advect_refl") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.div, mod, "qsmoke_div") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.jacobi, mod, "qsmoke_jacobi") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.jacobi2, mod, "qsmoke_jacobi2") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.project, mod, "qsmoke_project") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.advect_rho, mod, "qsmoke_advect_rho") != CUDA_SUCCESS) {
    err = "smoke JIT module lacks a kernel";
    return cudaErrorSymbolNotFound;
  }
  return cudaSuccess;
}

cudaError_t jit_codec(const std::string& src, CodecJit& out, std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::string log;
  CUmodule mod;
  cudaError_t e = compile_module(src, "qmpm_codec_spec.cu", mod, log, err);
  if (e) return e;
  if (g_drv.moduleGetFunction(&out.encode, mod, "qmpm_codec_encode") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.decode, mod, "qmpm_codec_decode") != CUDA_SUCCESS ||
      g_drv.moduleGetFunction(&out.matmul3, mod, "qmpm_codec_matmul3") != CUDA_SUCCESS) {
    err = "codec JIT module lacks a kernel";
    return cudaErrorSymbolNotFound;
  }
  return cudaSuccess;
}

cudaError_t jit_set_smem(CUfunction f, size_t bytes) {
  return g_drv.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)bytes) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorInvalidValue;
}

int jit_occupancy(CUfunction f, int threads, size_t smem) {
  int n = 0;
  if (g_drv.occupancy(&n, f, threads, smem) != CUDA_SUCCESS) return 1;
  return n > 0 ? n : 1;
}

cudaError_t jit_launch3(CUfunction f, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void** args) {
  CUresult r = g_drv.launchKernel(f, grid.x, grid.y, grid.z, block.x, block.y, block.z, (unsigned)smem, (CUstream)st,
                                  args, nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

cudaError_t jit_launch(CUfunction f, unsigned grid, unsigned block, size_t smem, cudaStream_t st, void** args) {
  CUresult r = g_drv.launchKernel(f, grid, 1, 1, block, 1, 1, (unsigned)smem, (CUstream)st, args, nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

}  // namespace qmpm
