// codegen.h -- circuit-specialised pass kernels, compiled at program load by NVRTC.
//
// The generic pass_kernel decodes every op at run time (switch over kind and
// register positions); on B200 that decode costs more issue slots than the
// arithmetic it dispatches (ncu: ALU pipe 72%, FMA pipe 10%).  Here each
// fused pass becomes its own kernel whose phase bodies are straight-line
// calls with compile-time register positions and literal matrix entries
// (hex-float, so c128 stays bit-identical to the operator table and c64 gets
// exactly the host's float rounding); cx / swap / x compile to register
// renaming.  Noise sites stay data-driven: one CTA-uniform test of the
// trajectory's outcome per site.
//
// NVRTC and the driver API are reached without link-time dependencies
// (dlopen + cudaGetDriverEntryPoint), so libptsbe.so still loads on hosts
// without a GPU driver (the CPU test suite checks its exports).
#pragma once
#include <cuda.h>
#include <dlfcn.h>

#include <cstdio>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "gen_prelude.inc"   // kGenPrelude: gen_prelude.cuh as a string (build.py)

namespace ptsbe {
namespace gen {

// ---------------------------------------------------------------- runtime loaders
typedef int (*nvrtcCreateProgram_t)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*nvrtcCompileProgram_t)(void*, int, const char* const*);
typedef int (*nvrtcGetSize_t)(void*, size_t*);
typedef int (*nvrtcGetBuf_t)(void*, char*);
typedef int (*nvrtcDestroyProgram_t)(void**);

struct Api {
  bool ok = false;
  std::string why;
  nvrtcCreateProgram_t create = nullptr;
  nvrtcCompileProgram_t compile = nullptr;
  nvrtcGetSize_t log_size = nullptr, cubin_size = nullptr;
  nvrtcGetBuf_t get_log = nullptr, get_cubin = nullptr;
  nvrtcDestroyProgram_t destroy = nullptr;
  CUresult (*module_load)(CUmodule*, const void*) = nullptr;
  CUresult (*get_function)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  CUresult (*func_set_attr)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
};

inline Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!lib) { a.why = "libnvrtc.so.12 not found"; return; }
    a.create = (nvrtcCreateProgram_t)dlsym(lib, "nvrtcCreateProgram");
    a.compile = (nvrtcCompileProgram_t)dlsym(lib, "nvrtcCompileProgram");
    a.log_size = (nvrtcGetSize_t)dlsym(lib, "nvrtcGetProgramLogSize");
    a.get_log = (nvrtcGetBuf_t)dlsym(lib, "nvrtcGetProgramLog");
    a.cubin_size = (nvrtcGetSize_t)dlsym(lib, "nvrtcGetCUBINSize");
    a.get_cubin = (nvrtcGetBuf_t)dlsym(lib, "nvrtcGetCUBIN");
    a.destroy = (nvrtcDestroyProgram_t)dlsym(lib, "nvrtcDestroyProgram");
    if (!a.create || !a.compile || !a.cubin_size || !a.get_cubin) { a.why = "nvrtc symbols missing"; return; }
    auto entry = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    bool good = entry("cuModuleLoadData", (void**)&a.module_load) &&
                entry("cuModuleGetFunction", (void**)&a.get_function) &&
                entry("cuLaunchKernel", (void**)&a.launch) &&
                entry("cuFuncSetAttribute", (void**)&a.func_set_attr) &&
                entry("cuOccupancyMaxActiveBlocksPerMultiprocessor", (void**)&a.occupancy);
    if (!good) { a.why = "driver entry points unavailable"; return; }
    a.ok = true;
  });
  return a;
}

// ---------------------------------------------------------------- source generation
struct OpMat {            // one concrete operator: kind + 4x4 complex (row-major, padded)
  int kind;
  const double* m;        // 32 doubles
};

inline std::string hexd(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}

inline uint32_t swz_host(bool c64, uint32_t i) {
  if (c64) {
    const uint32_t h = (i >> 3) ^ (i >> 7) ^ ((i >> 7) << 1) ^ (i >> 11);
    return i ^ (h & 14u);
  }
  const uint32_t h = (i >> 3) ^ (i >> 6) ^ ((i >> 6) << 1) ^ (i >> 9) ^ (i >> 12);
  return i ^ (h & 7u);
}

struct Emitter {
  std::ostringstream o;
  bool c64;
  std::string V, R;
  explicit Emitter(bool c64_) : c64(c64_), V(c64_ ? "float2" : "double2"), R(c64_ ? "float" : "double") {}

  std::string cx(const double* m, int r, int c) {   // complex entry literal
    return "ptg::mk((" + V + "*)0, " + hexd(m[2 * (4 * r + c)]) + ", " + hexd(m[2 * (4 * r + c) + 1]) + ")";
  }
  std::string rl(const double* m, int r, int c) { return "(" + R + ")" + hexd(m[2 * (4 * r + c)]); }

  void op(int kind, int k0, int k1, const double* m) {
    switch (kind) {
      case 1:  // MK_REAL1
        o << "ptg::g1r<" << k0 << ">(a, " << rl(m, 0, 0) << ", " << rl(m, 0, 1) << ", " << rl(m, 1, 0) << ", "
          << rl(m, 1, 1) << ");\n";
        break;
      case 2:  // MK_DIAG1
        o << "ptg::g1d<" << k0 << ">(a, " << cx(m, 0, 0) << ", " << cx(m, 1, 1) << ");\n";
        break;
      case 3:  // MK_PHASE1
        o << "ptg::g1p<" << k0 << ">(a, " << cx(m, 1, 1) << ");\n";
        break;
      case 4: {  // MK_ANTI1
        const bool x = m[2] == 1.0 && m[3] == 0.0 && m[8] == 1.0 && m[9] == 0.0;
        if (x) o << "ptg::g1x<" << k0 << ">(a);\n";
        else o << "ptg::g1a<" << k0 << ">(a, " << cx(m, 0, 1) << ", " << cx(m, 1, 0) << ");\n";
        break;
      }
      case 8: {  // MK_GEN2
        o << "{ const " << V << " m_[16] = {";
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) o << cx(m, r, c) << (r * 4 + c < 15 ? ", " : "");
        o << "}; ptg::g2<" << k0 << ", " << k1 << ">(a, m_); }\n";
        break;
      }
      case 9: o << "ptg::g2cx<" << k0 << ", " << k1 << ">(a);\n"; break;
      case 10: o << "ptg::g2sw<" << k0 << ", " << k1 << ">(a);\n"; break;
      case 11:
        o << "ptg::g2d<" << k0 << ", " << k1 << ">(a, " << cx(m, 0, 0) << ", " << cx(m, 1, 1) << ", " << cx(m, 2, 2)
          << ", " << cx(m, 3, 3) << ");\n";
        break;
      default:  // MK_GEN1
        o << "ptg::g1<" << k0 << ">(a, " << cx(m, 0, 0) << ", " << cx(m, 0, 1) << ", " << cx(m, 1, 0) << ", "
          << cx(m, 1, 1) << ");\n";
        break;
    }
  }
};

struct GenPass {
  int L, c;
  uint64_t qmask;
  std::vector<DevPhase> phases;
  std::vector<DevOp> ops;   // phase-major, k0/k1 filled
};

struct GenProgram {
  bool c64;
  int n;
  const double* mats;       // n_mats x 32 doubles
  const int32_t* kinds;     // n_mats
  const ptsbe_channel* chans;
  const int32_t* site_chan;
  std::vector<GenPass> passes;
};

inline std::string kernel_name(int pass) { return "ptsbe_pass_" + std::to_string(pass); }

// Lambda scattering the low bits of x onto the set bits of `mask` (PDEP as shift/mask runs).
inline std::string scatter_fn(uint64_t mask, const char* arg_type) {
  std::ostringstream o;
  o << "[](" << arg_type << " x_) -> uint64_t { return 0ull";
  int src = 0;
  for (int q = 0; q < 64;) {
    if (!((mask >> q) & 1)) { ++q; continue; }
    int len = 0;
    while (q + len < 64 && ((mask >> (q + len)) & 1)) ++len;
    const uint64_t m = len >= 64 ? ~0ull : ((1ull << len) - 1);
    o << " | ((((uint64_t)x_ >> " << src << ") & 0x" << std::hex << m << std::dec << "ull) << " << q << ")";
    src += len;
    q += len;
  }
  o << "; }";
  return o.str();
}

inline std::string generate(const GenProgram& P) {
  Emitter e(P.c64);
  std::ostringstream& o = e.o;
  o << kGenPrelude << "\n";
  for (size_t pi = 0; pi < P.passes.size(); ++pi) {
    const GenPass& gp = P.passes[pi];
    const int threads = std::max(32, 1 << (gp.L - 4));
    const uint64_t nmask = P.n >= 64 ? ~0ull : ((1ull << P.n) - 1);
    const uint64_t comp = ~gp.qmask & nmask;
    const uint64_t hmask = gp.qmask & ~((1ull << gp.c) - 1);
    o << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", " << (threads <= 256 ? 2 : 1) << ") "
      << kernel_name((int)pi) << "(const ptg::PassParams p) {\n"
      << "  typedef " << e.V << " V;\n"
      << "  ptg::run_pass<" << e.R << ", " << gp.L << ", " << gp.c << ", " << (P.n - gp.L) << ">(p,\n"
      << "    " << scatter_fn(comp, "uint64_t") << ",\n"
      << "    " << scatter_fn(hmask, "uint32_t") << ",\n"
      << "    [&](V* cur, int b, const uint8_t* sel, long long tile, uint64_t base, double scale, double* red) {\n"
      << "    const uint32_t g = threadIdx.x;\n"
      << "    const bool active = g < " << (1u << (gp.L - 4)) << "u;\n"
      << "    V a[16];\n";
    for (size_t ph = 0; ph < gp.phases.size(); ++ph) {
      const DevPhase& D = gp.phases[ph];
      const int pb[4] = {(int)(D.pbits & 31), (int)((D.pbits >> 5) & 31), (int)((D.pbits >> 10) & 31),
                         (int)((D.pbits >> 15) & 31)};
      uint32_t off[16], so[16];
      for (int j = 0; j < 16; ++j) {
        off[j] = 0;
        for (int k = 0; k < 4; ++k)
          if ((j >> k) & 1) off[j] |= 1u << pb[k];
        so[j] = swz_host(P.c64, off[j]);
      }
      o << "    { // phase " << ph << "\n"
        << "      const uint32_t gb = ptg::ins0(ptg::ins0(ptg::ins0(ptg::ins0(g, " << pb[0] << "), " << pb[1] << "), "
        << pb[2] << "), " << pb[3] << ");\n"
        << "      const uint32_t sg = ptg::swz((V*)0, gb);\n"
        << "      const uint32_t so[16] = {";
      for (int j = 0; j < 16; ++j) o << so[j] << "u" << (j < 15 ? ", " : "");
      o << "};\n";
      if (ph == 0) {
        o << "      const uint32_t off[16] = {";
        for (int j = 0; j < 16; ++j) o << off[j] << "u" << (j < 15 ? ", " : "");
        o << "};\n"
          << "      if (p.gen_zero) ptg::zero16(a, base, gb, off, active);\n"
          << "      else ptg::ld16<V, " << pb[0] << ">(a, cur, sg, so, active, scale);\n";
      } else {
        o << "      ptg::ld16<V, " << pb[0] << ">(a, cur, sg, so, active, 1.0);\n";
      }
      // CTA-uniform: does this trajectory take any non-default outcome in this phase?
      std::ostringstream err;
      for (int k = D.op_begin; k < D.op_begin + D.n_ops; ++k)
        if (gp.ops[k].kind == 1) err << (err.tellp() > 0 ? " | " : "") << "sel[" << gp.ops[k].ref << "]";
      const bool has_sites = err.tellp() > 0;
      if (has_sites) o << "      if ((" << err.str() << ") == 0) {\n";
      // fast path: every site at its default outcome -> straight-line gates only
      for (int k = D.op_begin; k < D.op_begin + D.n_ops; ++k) {
        const DevOp& op = gp.ops[k];
        const int k1 = op.arity == 2 ? op.k1 : 0;
        if (op.kind == 0) {
          o << "      ";
          e.op(P.kinds[op.ref], op.k0, k1, P.mats + (size_t)op.ref * 32);
          continue;
        }
        const ptsbe_channel& ch = P.chans[P.site_chan[op.ref]];
        if (!(ch.identity_mask & 1ull)) {   // outcome 0 is not the identity (e.g. damping K0)
          o << "      ";
          e.op(P.kinds[ch.mat_base], op.k0, k1, P.mats + (size_t)ch.mat_base * 32);
        }
        if (ch.general) {
          o << "      { double s_ = 0.0;\n"
            << "#pragma unroll\n"
            << "        for (int j = 0; j < 16; ++j) s_ += ptg::prob64(a[j]);\n"
            << "        s_ = ptg::block_sum(s_, red);\n"
            << "        if (threadIdx.x == 0) p.partials[((size_t)" << op.slot
            << " * p.B + b) * p.tiles + tile] = s_; }\n";
        }
      }
      if (has_sites) {
        // rare path: run the phase through the run-time interpreter on shared memory
        o << "      } else {\n"
          << "        ptg::st16<V, " << pb[0] << ">(a, cur, sg, so, active);\n"
          << "        const uint32_t sb_[4] = {so[1], so[2], so[4], so[8]};\n"
          << "        ptg::interp_phase<V>(cur, sg, sb_, p, " << ph << ", sel, b, tile, red, active);\n"
          << "        ptg::ld16<V, " << pb[0] << ">(a, cur, sg, so, active, 1.0);\n"
          << "      }\n";
      }
      o << "      ptg::st16<V, " << pb[0] << ">(a, cur, sg, so, active);\n"
        << "      __syncthreads();\n"
        << "    }\n";
    }
    o << "  });\n}\n";
  }
  return o.str();
}

// ---------------------------------------------------------------- compile + cache
struct Module {
  CUmodule mod = nullptr;
  std::vector<CUfunction> fns;
};

inline bool compile(const std::string& src, int n_passes, int dev, Module& out, std::string& err) {
  Api& A = api();
  if (!A.ok) { err = A.why; return false; }
  static std::mutex mu;
  static std::map<std::pair<int, std::string>, Module> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, src);
  auto it = cache.find(key);
  if (it != cache.end()) { out = it->second; return true; }
  void* prog = nullptr;
  if (A.create(&prog, src.c_str(), "ptsbe_gen.cu", 0, nullptr, nullptr) != 0) { err = "nvrtcCreateProgram failed"; return false; }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--device-as-default-execution-space"};
  const int rc = A.compile(prog, 4, opts);
  if (rc != 0) {
    size_t n = 0;
    A.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) A.get_log(prog, &log[0]);
    err = "NVRTC compile failed: " + log.substr(0, 2000);
    A.destroy(&prog);
    return false;
  }
  size_t n = 0;
  A.cubin_size(prog, &n);
  std::vector<char> cubin(n);
  A.get_cubin(prog, cubin.data());
  A.destroy(&prog);
  Module m;
  if (A.module_load(&m.mod, cubin.data()) != CUDA_SUCCESS) { err = "cuModuleLoadData failed"; return false; }
  for (int i = 0; i < n_passes; ++i) {
    CUfunction f = nullptr;
    if (A.get_function(&f, m.mod, kernel_name(i).c_str()) != CUDA_SUCCESS) { err = "cuModuleGetFunction failed"; return false; }
    A.func_set_attr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 227 * 1024);
    m.fns.push_back(f);
  }
  cache[key] = m;
  out = m;
  return true;
}

inline size_t smem_bytes(int L, int /*c*/, size_t amp_bytes) {
  return 2 * ((size_t)1 << L) * amp_bytes + 32 * 8;
}

}  // namespace gen
}  // namespace ptsbe
