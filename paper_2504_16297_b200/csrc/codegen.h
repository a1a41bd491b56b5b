// codegen.h -- circuit-specialised pass kernels, compiled at program load by NVRTC.
//
// The generic pass_kernel decodes every op at run time (switch over kind and
// register positions); on B200 that decode costs more issue slots than the
// arithmetic it dispatches (ncu: ALU pipe 72%, FMA pipe 10%).  Here each
// fused pass becomes its own kernel whose phase bodies are straight-line
// calls with compile-time register positions and literal matrix entries
// (hex-float, so c128 stays bit-identical to the operator table and c64 gets
// exactly the host's float rounding); cx / swap / x compile to register
// renaming; consecutive diagonal gates merge into one deferred register-group
// diagonal.  Noise sites stay data-driven: per phase, hit words say which sites
// the trajectory takes a non-default outcome at; a phase without hits runs its
// fast straight-line code, a phase with hits calls an out-of-line slow variant
// (per 8-site segment) whose sites test their bit and apply the outcome's
// operator from the table.  Per pass the generator also picks the register
// width (4 or 5 bits), the shared-memory swizzle (bank-conflict model), and, for
// the last pass of a unitary program, fuses the sampler's block sums.
//
// NVRTC and the driver API are reached without link-time dependencies
// (dlopen + cudaGetDriverEntryPoint), so libptsbe.so still loads on hosts
// without a GPU driver (the CPU test suite checks its exports).
#pragma once
#include <cuda.h>
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <atomic>
#include <thread>
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
    // The CUDA toolkit's NVRTC first (the one nvcc ships with): a process that
    // imported torch already has torch's bundled NVRTC under the same soname, and
    // that older ptxas materialises i*x with MOV + FADD instead of the FFMA2 .NP
    // operand modifier (config 4: +2.1 K instructions, hot bodies 20% larger).
    void* lib = nullptr;
    if (const char* home = std::getenv("CUDA_HOME")) {
      const std::string path = std::string(home) + "/lib64/libnvrtc.so.12";
      lib = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
    }
    if (!lib) lib = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
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

// Shared-memory swizzle of one pass: slot(i) = i ^ XOR_{b set in i} m[b], where
// only bits above the bank-select bits carry masks and the masks touch only the
// bank-select bits (c64: bits 1-3 of the 8-B amplitude index, bit 0 stays so
// amplitude pairs remain aligned 16-B vectors; c128: bits 0-2).  Linear over
// GF(2) and triangular, hence a bijection, and slot(a ^ b) = slot(a) ^ slot(b),
// so every phase address is a per-thread base XOR a compile-time constant.
struct Swizzle {
  bool c64 = true;
  uint32_t m[32] = {0};
  uint32_t operator()(uint32_t i) const {
    uint32_t r = i;
    for (int b = 0; b < 32; ++b)
      if ((i >> b) & 1u) r ^= m[b];
    return r;
  }
  static Swizzle fixed(bool c64) {   // the default map (swz_host)
    Swizzle z;
    z.c64 = c64;
    for (int b = 0; b < 20; ++b) z.m[b] = swz_host(c64, 1u << b) ^ (1u << b);
    return z;
  }
};

inline uint32_t ins0_host(uint32_t p, int bit) {
  const uint32_t lo = p & ((1u << bit) - 1u);
  return ((p ^ lo) << 1) | lo;
}

// Shared-memory wavefronts of one warp's phase loads (stores are symmetric) under
// swizzle z: lanes 0..31 hold consecutive register groups.  16-B accesses (c128,
// or c64 phases holding bit 0, which load amplitude pairs) are served per quarter
// warp by distinct 16-B chunks of a 128-B line; 8-B accesses per half warp by
// distinct 8-B slots.  Minimum = conflict free.
inline int phase_wavefronts(const Swizzle& z, const DevPhase& D, int GB) {
  int pb[5];
  for (int q = 0; q < GB; ++q) pb[q] = (int)((D.pbits >> (5 * q)) & 31);
  uint32_t lanes[32];
  for (int l = 0; l < 32; ++l) {
    uint32_t g = (uint32_t)l;
    for (int q = 0; q < GB; ++q) g = ins0_host(g, pb[q]);
    lanes[l] = g;
  }
  const bool wide = !z.c64 || pb[0] == 0;
  int tot = 0;
  for (int j = 0; j < (1 << GB); j += (z.c64 && wide) ? 2 : 1) {
    uint32_t off = 0;
    for (int q = 0; q < GB; ++q)
      if ((j >> q) & 1) off |= 1u << pb[q];
    if (wide) {
      for (int qw = 0; qw < 4; ++qw) {
        int cnt[8] = {0}, mx = 0;
        for (int l = qw * 8; l < qw * 8 + 8; ++l) {
          const uint32_t a = z(lanes[l] | off);
          const int c = z.c64 ? (int)((a >> 1) & 7u) : (int)(a & 7u);
          mx = std::max(mx, ++cnt[c]);
        }
        tot += mx;
      }
    } else {   // 8-B accesses: modelled per half warp (16 lanes on 16 distinct 8-B slots)
      for (int hw = 0; hw < 2; ++hw) {
        int cnt[16] = {0}, mx = 0;
        for (int l = hw * 16; l < hw * 16 + 16; ++l) mx = std::max(mx, ++cnt[z(lanes[l] | off) & 15u]);
        tot += mx;
      }
    }
  }
  return tot;
}

// Per pass: coordinate descent over the masks of the tile bits above the
// bank-select bits, from the default map, minimising the phases' wavefronts.
inline Swizzle choose_swizzle(bool c64, int L, const std::vector<DevPhase>& phases, int GB) {
  Swizzle best = Swizzle::fixed(c64);
  for (int b = L; b < 32; ++b) best.m[b] = 0;
  auto cost = [&](const Swizzle& z) {
    int t = 0;
    for (const DevPhase& D : phases) t += phase_wavefronts(z, D, GB);
    return t;
  };
  int bc = cost(best);
  const int lo = c64 ? 4 : 3;
  for (int sweep = 0; sweep < 3; ++sweep) {
    bool improved = false;
    for (int b = lo; b < L; ++b)
      for (uint32_t v = 0; v < 8; ++v) {
        Swizzle cand = best;
        cand.m[b] = c64 ? (v << 1) : v;
        const int c = cost(cand);
        if (c < bc) { bc = c; best = cand; improved = true; }
      }
    if (!improved) break;
  }
  return best;
}

// Tile buffers per CTA: two (the next tile streams in while this one computes) for 32-KB
// tiles; ONE for 64-KB tiles (c128 L = 12, c64 L = 13), where a second buffer would leave a
// single CTA per SM -- three single-buffered CTAs hide the load latency for each other
// instead (PTSBE_STAGES = 1 / 2 overrides).
inline int stages_for(int L, size_t amp_bytes) {
  if (const char* e = std::getenv("PTSBE_STAGES")) return std::atoi(e) == 1 ? 1 : 2;
  return ((size_t)1 << L) * amp_bytes > (48u << 10) ? 1 : 2;
}
inline size_t smem_bytes_for(int L, size_t amp_bytes, int teams = 1, int stages = 0);   // below (smem_bytes)

// Compute teams per CTA (gen_prelude.cuh run_pass TEAMS): a single-buffered TMA pass runs
// as ONE CTA per SM of two teams sharing three tile buffers -- each team finds its next
// tile already loading while it computes -- instead of two single-buffered CTAs that each
// wait out their own loads.  The teams are coupled (a team's next tile is loaded by the
// other team once it frees a buffer), which costs the light, memory-bound passes what it
// gains on the compute-heavy ones.  Measured on config 4 (complex128, 12-qubit tiles,
// per-pass GB/s, 2 teams vs 2 CTAs): passes with 41-86 gates +3..16 %, passes with 11-30
// gates -5..-8 % -> two teams from 40 gates (PTSBE_TEAMS_MIN_GATES); PTSBE_TEAMS = 1 / 2
// forces one / two teams everywhere (A/B knob).
inline int teams_for(int L, size_t amp_bytes, bool tma, int n_gates) {
  if (!tma || stages_for(L, amp_bytes) != 1) return 1;
  static const int force = std::getenv("PTSBE_TEAMS") ? std::atoi(std::getenv("PTSBE_TEAMS")) : 0;
  static const int min_gates = std::getenv("PTSBE_TEAMS_MIN_GATES") ? std::atoi(std::getenv("PTSBE_TEAMS_MIN_GATES")) : 40;
  if (force) return force >= 2 ? 2 : 1;
  return n_gates >= min_gates ? 2 : 1;
}
// Tile buffers of a one-team pass.  Light complex128 passes (below the teams threshold:
// memory-bound, little FP64 work per tile) on single-buffered 64-KB tiles run as ONE CTA
// per SM with three buffers instead: two tiles stream in while one computes
// (PTSBE_LIGHT_STAGES = 1 keeps two single-buffered CTAs per SM).
inline int pass_stages(int L, size_t amp_bytes, bool tma, int teams) {
  const int st = stages_for(L, amp_bytes);
  if (teams > 1 || st != 1 || !tma) return st;
  static const int light = std::getenv("PTSBE_LIGHT_STAGES") ? std::atoi(std::getenv("PTSBE_LIGHT_STAGES")) : 1;
  return light >= 3 ? 3 : 1;
}
constexpr const char* kTeamsTag = "// @@ptsbe-teams@@ ";   // "<teams> <stages>" of a pass kernel

// TMA tile staging for a pass (gen_prelude.cuh run_pass TMA): 128-B rows need the pass's
// contiguous low run to cover a row (c64: 16 amplitudes, c128: 8) and the row table holds
// <= 64 gather groups (256 rows).  Default: complex128 passes (config 4: 456 K vs 445 K
// shots/s with cp.async, pass roofline 0.757 vs 0.739); complex64 passes keep cp.async
// (1.371 M vs 1.385 M: the 5-bit 128-thread passes lose a few % to the store drain).
// PTSBE_TMA=1 / 0 forces either way.
inline bool tma_ok(bool c64, int c, int L) {
  const char* e = std::getenv("PTSBE_TMA");
  const bool want = std::getenv("PTSBE_NO_TMA") ? false : e ? std::atoi(e) != 0 : !c64;
  return want && c >= (c64 ? 4 : 3) && L - (c64 ? 4 : 3) <= 9;   // <= 128 gather groups (row table)
}

// TMA tile staging lands each 128-B tile row u at shared-memory row slot(u) with the
// hardware's 128-B swizzle (16-B chunk ^= slot & 7).  With slot = any GF(2)-linear
// bijection whose low three bits are B(u), the chunk of row u is XORed with B(u): exactly
// the free family above (chunk ^= a linear function of the row bits) whenever that
// function has rank 3.  make_tma_layout takes the model-chosen free swizzle, repairs its
// rank if needed (coordinate descent under the rank constraint), and returns the
// amplitude-index map (row bits move too) plus slot^-1 for the gathers.
struct TmaLayout {
  Swizzle sw;              // amplitude index -> shared-memory slot (rows and chunks)
  uint32_t inv[32] = {0};  // slot row -> tile row u (linear: XOR of inv[j] over set bits j)
  int R = 0;               // row bits
};

inline int gf2_rank3(const uint32_t* col, int R) {   // rank of 3-bit columns
  uint32_t basis[3] = {0, 0, 0};
  int r = 0;
  for (int k = 0; k < R; ++k) {
    uint32_t v = col[k] & 7u;
    for (int b = 2; b >= 0 && v; --b)
      if ((v >> b) & 1u) {
        if (basis[b]) v ^= basis[b];
        else { basis[b] = v; ++r; v = 0; }
      }
  }
  return r;
}

inline bool make_tma_layout(bool c64, int L, const std::vector<DevPhase>& phases, int GB, const Swizzle& free_sw,
                            TmaLayout* out) {
  const int cb = c64 ? 1 : 0, lo = c64 ? 4 : 3;
  const int R = L - lo;
  if (R < 3 || R > 20) return false;
  uint32_t col[32] = {0};
  for (int k = 0; k < R; ++k) col[k] = (free_sw.m[lo + k] >> cb) & 7u;
  auto build = [&](const uint32_t* c) {
    Swizzle z;
    z.c64 = c64;
    for (int k = 0; k < R; ++k) z.m[lo + k] = c[k] << cb;
    return z;
  };
  auto cost = [&](const uint32_t* c) {
    if (gf2_rank3(c, R) < 3) return 1 << 30;
    const Swizzle z = build(c);
    int t = 0;
    for (const DevPhase& D : phases) t += phase_wavefronts(z, D, GB);
    return t;
  };
  int bc = cost(col);
  if (bc >= (1 << 30)) {   // rank < 3: start from the row-low-bits map and descend
    uint32_t c2[32] = {0};
    for (int k = 0; k < R; ++k) c2[k] = k < 3 ? (1u << k) : col[k];
    std::memcpy(col, c2, sizeof c2);
    bc = cost(col);
    for (int sweep = 0; sweep < 4; ++sweep) {
      bool improved = false;
      for (int k = 0; k < R; ++k)
        for (uint32_t v = 0; v < 8; ++v) {
          uint32_t cand[32];
          std::memcpy(cand, col, sizeof cand);
          cand[k] = v;
          const int c = cost(cand);
          if (c < bc) { bc = c; std::memcpy(col, cand, sizeof cand); improved = true; }
        }
      if (!improved) break;
    }
  }
  // pivots: three row bits with independent columns -> slot bits 0-2 carry B(u)
  int piv[3] = {-1, -1, -1};
  {
    uint32_t basis[3] = {0, 0, 0};
    for (int k = 0, got = 0; k < R && got < 3; ++k) {
      uint32_t v = col[k];
      for (int b = 2; b >= 0 && v; --b)
        if ((v >> b) & 1u) {
          if (basis[b]) v ^= basis[b];
          else { basis[b] = v; piv[got++] = k; v = 0; }
        }
    }
    if (piv[2] < 0) return false;
  }
  uint32_t slot_of[32] = {0};   // slot(e_k)
  for (int k = 0, nxt = 3; k < R; ++k) {
    const bool is_piv = k == piv[0] || k == piv[1] || k == piv[2];
    slot_of[k] = col[k] | (is_piv ? 0u : (1u << nxt));
    if (!is_piv) ++nxt;
  }
  // invert the R x R slot matrix over GF(2) (columns slot_of[k])
  uint32_t a[32], inv[32];
  for (int j = 0; j < R; ++j) { a[j] = 0; inv[j] = 0; }
  for (int k = 0; k < R; ++k)   // row j of the matrix: bit k set iff slot_of[k] has bit j
    for (int j = 0; j < R; ++j)
      if ((slot_of[k] >> j) & 1u) a[j] |= 1u << k;
  uint32_t e[32];
  for (int j = 0; j < R; ++j) e[j] = 1u << j;     // augmented identity rows
  for (int c = 0; c < R; ++c) {
    int pr = -1;
    for (int j = c; j < R; ++j)
      if ((a[j] >> c) & 1u) { pr = j; break; }
    if (pr < 0) return false;
    std::swap(a[c], a[pr]);
    std::swap(e[c], e[pr]);
    for (int j = 0; j < R; ++j)
      if (j != c && ((a[j] >> c) & 1u)) { a[j] ^= a[c]; e[j] ^= e[c]; }
  }
  // a is identity now; row k of the inverse (u bit k) = e[k]: u_k = parity(e[k] & s)
  for (int j = 0; j < R; ++j)      // inv[j] = slot^-1(e_j): bit k set iff e[k] has bit j
    for (int k = 0; k < R; ++k)
      if ((e[k] >> j) & 1u) inv[j] |= 1u << k;
  out->R = R;
  out->sw = Swizzle();
  out->sw.c64 = c64;
  for (int k = 0; k < R; ++k) out->sw.m[lo + k] = ((slot_of[k] ^ (1u << k)) << lo) | (col[k] << cb);
  std::memcpy(out->inv, inv, sizeof inv);
  return true;
}

// Device functor for the slot -> tile-row map of a TMA layout.
inline std::string slot_inv_struct(const std::string& name, const TmaLayout& t) {
  std::ostringstream o;
  o << "struct " << name << " { __device__ __forceinline__ uint32_t operator()(uint32_t s) const { return 0u";
  for (int j = 0; j < t.R; ++j) o << " ^ ((0u - ((s >> " << j << ") & 1u)) & " << t.inv[j] << "u)";
  o << "; } };\n";
  return o.str();
}

// TMA row table of a pass as a __constant__ array (the warp-uniform issue path reads it with
// uniform constant loads straight into uniform registers): gather group g, row q -> tile-relative
// 128-B row coordinate of shared-memory slot 4g + q (gen_prelude.cuh fill_rowtab computes the
// same table into shared memory for the per-lane path).
inline std::string rowtab_struct(const std::string& name, bool tma, bool c64, int C, int L, uint64_t hmask,
                                 const TmaLayout& t) {
  std::ostringstream o;
  if (!tma) {
    o << "struct " << name << " { __device__ __forceinline__ uint4 operator()(int) const { return make_uint4(0u, 0u, 0u, 0u); } };\n";
    return o.str();
  }
  const int LOGU = c64 ? 4 : 3;
  const int NGRP = (1 << (L - LOGU)) / 4;
  auto pdep = [&](uint64_t x) {
    uint64_t r = 0;
    for (int q = 0; q < 64; ++q)
      if ((hmask >> q) & 1) { r |= (x & 1) << q; x >>= 1; }
    return r;
  };
  o << "__constant__ uint4 k" << name << "[" << NGRP << "] = {";
  for (int g = 0; g < NGRP; ++g) {
    o << (g ? ", " : "") << "{";
    for (int q = 0; q < 4; ++q) {
      const uint32_t sidx = (uint32_t)(4 * g + q);
      uint32_t u = 0;
      for (int j = 0; j < t.R; ++j)
        if ((sidx >> j) & 1u) u ^= t.inv[j];
      const uint64_t lo = u & ((1u << (C - LOGU)) - 1u);
      const uint64_t v = ((lo << LOGU) | pdep(u >> (C - LOGU))) >> LOGU;
      o << (q ? ", " : "") << (uint32_t)v << "u";
    }
    o << "}";
  }
  o << "};\nstruct " << name << " { __device__ __forceinline__ uint4 operator()(int g) const { return k" << name
    << "[g]; } };\n";
  return o.str();
}

// Device functor for a swizzle (compile-time masks).
inline std::string swizzle_struct(const std::string& name, const Swizzle& z, int L) {
  std::ostringstream o;
  o << "struct " << name << " { __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return i";
  for (int b = 0; b < L; ++b)
    if (z.m[b]) o << " ^ ((0u - ((i >> " << b << ") & 1u)) & " << z.m[b] << "u)";
  o << "; } };\n";
  return o.str();
}

// Complex scalar helpers for the host-side factor bookkeeping.
struct Cx { double re, im; };
inline Cx cxmul(Cx a, Cx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline Cx cxdiv(Cx a, Cx b) {
  const double d = b.re * b.re + b.im * b.im;
  return {(a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d};
}
inline double cxabs(Cx a) { return std::sqrt(a.re * a.re + a.im * a.im); }

struct Emitter {
  std::ostringstream o;
  bool c64;
  std::string V, R;
  explicit Emitter(bool c64_) : c64(c64_), V(c64_ ? "float2" : "double2"), R(c64_ ? "float" : "double") {}

  std::string lit(double re, double im) { return "ptg::mk((" + V + "*)0, " + hexd(re) + ", " + hexd(im) + ")"; }
  std::string cx(const double* m, int r, int c) { return lit(m[2 * (4 * r + c)], m[2 * (4 * r + c) + 1]); }
  std::string rl(double v) { return "(" + R + ")" + hexd(v); }
  static Cx at(const double* m, int r, int c) { return {m[2 * (4 * r + c)], m[2 * (4 * r + c) + 1]}; }

  // Phase-only multiply of the amplitudes whose bit K is 1 (literal ±1, ±i specialised).
  void phase(int k, Cx d) {
    if (d.re == 1.0 && d.im == 0.0) { o << "\n"; return; }
    if (d.im == 0.0 && d.re == -1.0) { o << "ptg::g1neg<" << k << ">(a);\n"; return; }
    if (d.re == 0.0 && d.im == 1.0) { o << "ptg::g1pi<" << k << ">(a, false);\n"; return; }
    if (d.re == 0.0 && d.im == -1.0) { o << "ptg::g1pi<" << k << ">(a, true);\n"; return; }
    o << "ptg::g1p<" << k << ">(a, " << lit(d.re, d.im) << ");\n";
  }

  // a[j] *= d for one register (literal d; 1 is skipped, +-1 / +-i specialised).
  void dmul(int j, Cx d) {
    if (d.re == 1.0 && d.im == 0.0) return;
    o << "      ";
    // -1, +i, -i: sign flips and a re/im swap (operand modifiers / renaming, no multiply)
    if (d.im == 0.0 && d.re == -1.0) o << "a[" << j << "] = ptg::neg(a[" << j << "]);\n";
    else if (d.re == 0.0 && d.im == 1.0) o << "a[" << j << "] = ptg::ix(a[" << j << "]);\n";
    else if (d.re == 0.0 && d.im == -1.0) o << "a[" << j << "] = ptg::neg(ptg::ix(a[" << j << "]));\n";
    else o << "a[" << j << "] = ptg::cmul(" << lit(d.re, d.im) << ", a[" << j << "]);\n";
  }
  // A merged diagonal entry (a product of several gates' entries) within a few ulps of
  // +-1 or +-i is taken as exactly that value: the product's rounding residue (e.g. T * T =
  // 2^-52 + i) is below the fp64 parity tolerance, and the exact value costs no multiply.
  static Cx snap(Cx d) {
    const double eps = 0x1p-49;
    auto near = [&](double x, double v) { return std::fabs(x - v) <= eps; };
    if (std::fabs(d.im) <= eps && (near(d.re, 1.0) || near(d.re, -1.0))) return {d.re > 0 ? 1.0 : -1.0, 0.0};
    if (std::fabs(d.re) <= eps && (near(d.im, 1.0) || near(d.im, -1.0))) return {0.0, d.im > 0 ? 1.0 : -1.0};
    return d;
  }

  // Emit one gate.  With `scaled`, a factor f is pulled out of the matrix
  // (M = f * M', M' applied) and returned; otherwise f = 1.
  Cx op(int kind, int k0, int k1, const double* m, bool scaled) {
    switch (kind) {
      case 1: {  // MK_REAL1
        double a = m[0], b = m[2], c = m[8], d = m[10];
        double f = 1.0;
        if (scaled) { f = std::fabs(a) >= std::fabs(b) ? a : b; a /= f; b /= f; c /= f; d /= f; }
        if (a == 1.0 && b == 1.0 && c == 1.0 && d == -1.0)        // scaled Hadamard
          o << "ptg::g1h<" << k0 << ">(a);\n";
        else if (a == 1.0 && d == 1.0)                             // scaled rotation
          o << "ptg::g1rot<" << k0 << ">(a, " << rl(b) << ", " << rl(c) << ");\n";
        else
          o << "ptg::g1r<" << k0 << ">(a, " << rl(a) << ", " << rl(b) << ", " << rl(c) << ", " << rl(d) << ");\n";
        return {f, 0.0};
      }
      case 2: {  // MK_DIAG1
        const Cx d0 = at(m, 0, 0), d1 = at(m, 1, 1);
        if (scaled && cxabs(d0) > 0.0) {
          phase(k0, cxdiv(d1, d0));
          return d0;
        }
        o << "ptg::g1d<" << k0 << ">(a, " << cx(m, 0, 0) << ", " << cx(m, 1, 1) << ");\n";
        return {1.0, 0.0};
      }
      case 3:  // MK_PHASE1
        phase(k0, at(m, 1, 1));
        return {1.0, 0.0};
      case 4: {  // MK_ANTI1
        const bool x = m[2] == 1.0 && m[3] == 0.0 && m[8] == 1.0 && m[9] == 0.0;
        if (x) o << "ptg::g1x<" << k0 << ">(a);\n";
        else o << "ptg::g1a<" << k0 << ">(a, " << cx(m, 0, 1) << ", " << cx(m, 1, 0) << ");\n";
        return {1.0, 0.0};
      }
      case 8: {  // MK_GEN2
        o << "{ const " << V << " m_[16] = {";
        for (int r = 0; r < 4; ++r)
          for (int c = 0; c < 4; ++c) o << cx(m, r, c) << (r * 4 + c < 15 ? ", " : "");
        o << "}; ptg::g2<" << k0 << ", " << k1 << ">(a, m_); }\n";
        return {1.0, 0.0};
      }
      case 9: o << "ptg::g2cx<" << k0 << ", " << k1 << ">(a);\n"; return {1.0, 0.0};
      case 10: o << "ptg::g2sw<" << k0 << ", " << k1 << ">(a);\n"; return {1.0, 0.0};
      case 11: {  // MK_DIAG2: multiply only the entries that are not exactly 1
        o << "\n";
        for (int s = 0; s < 4; ++s) {
          const Cx d = at(m, s, s);
          if (d.re == 1.0 && d.im == 0.0) continue;
          o << "      ptg::g2dsel<" << k0 << ", " << k1 << ", " << s << ">(a, " << lit(d.re, d.im) << ");\n";
        }
        return {1.0, 0.0};
      }
      default:  // MK_GEN1
        o << "ptg::g1<" << k0 << ">(a, " << cx(m, 0, 0) << ", " << cx(m, 0, 1) << ", " << cx(m, 1, 0) << ", "
          << cx(m, 1, 1) << ");\n";
        return {1.0, 0.0};
    }
  }
};

struct GenPass {
  int L, c;
  int gb = 4;                     // register bits per phase (4 or 5)
  uint64_t qmask;
  std::vector<DevPhase> phases;   // pbits: GB positions, 5 bits each
  std::vector<DevOp> ops;         // phase-major, k0/k1 filled
};

struct GenProgram {
  bool c64;
  int n;
  const double* mats;       // n_mats x 32 doubles
  const int32_t* kinds;     // n_mats
  const ptsbe_channel* chans;
  const int32_t* site_chan;
  std::vector<GenPass> passes;
  bool tma = true;          // the engine has a tensor map over its states (TMA tile staging allowed)
};

inline std::string kernel_name(int pass) { return "ptsbe_pass_" + std::to_string(pass); }

// Register groups a pass kernel's thread walks per phase (a run-time loop over
// the same straight-line phase body): G groups per thread fetch each instruction
// once per G executions.  Once the slow variants moved out of line the hot body
// of every config-4 pass fits the 32 KB L1.5 instruction cache and G = 1 (256
// threads, 2 CTAs/SM) measured fastest (965 K vs 954 K shots/s at G = 2), so G
// is a tuning knob (PTSBE_GROUP_LOOP).  Passes with renormalising sites keep
// G = 1 (their per-tile norm reduction is per phase).
inline int group_loop(int L, int gb, bool general) {
  if (general) return 1;
  static const int want = [] {
    const char* e = std::getenv("PTSBE_GROUP_LOOP");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  int g = 1;
  while (g < want && ((1 << (L - gb)) / (2 * g)) >= 64) g *= 2;
  return g;
}
inline int threads_for(int L, int gb, bool general) {
  return std::max(32, (1 << (L - gb)) / group_loop(L, gb, general));
}

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

// Hit words of a pass: site number i of phase ph (in op order) owns bit i % 64 of
// word hit_word(ph) + i / 64.
inline std::vector<int> hit_word_offsets(const GenPass& gp) {
  std::vector<int> off(gp.phases.size() + 1, 0);
  for (size_t ph = 0; ph < gp.phases.size(); ++ph) {
    const DevPhase& D = gp.phases[ph];
    int ns = 0;
    for (int q = D.op_begin; q < D.op_begin + D.n_ops; ++q) ns += gp.ops[q].kind == 1;
    off[ph + 1] = off[ph] + (ns + 63) / 64;
  }
  return off;
}
constexpr int kMaxHitWords = 480;   // shared-memory room reserved per CTA (smem_bytes)

// Per-trajectory outcome summary, evaluated by one thread per CTA when the
// trajectory changes: hit words (bit set iff that site takes a non-default
// outcome) into shared memory, and the returned phase mask (bit ph set iff phase
// ph has a hit; phases past 63 share bit 63).  The slow variant of a phase then
// tests compile-time bits of a word it reads once, instead of re-reading every
// site's outcome byte for every register group.
inline std::string err_mask_fn(const GenPass& gp) {
  const std::vector<int> woff = hit_word_offsets(gp);
  std::ostringstream o;
  o << "[](const uint8_t* sel, uint64_t* hw) -> uint64_t { uint64_t m_ = 0, w_;";
  for (size_t ph = 0; ph < gp.phases.size(); ++ph) {
    const DevPhase& D = gp.phases[ph];
    int i = 0;
    for (int q = D.op_begin; q < D.op_begin + D.n_ops; ++q) {
      if (gp.ops[q].kind != 1) continue;
      if (i % 64 == 0) o << " w_ = 0;";
      o << " w_ |= (uint64_t)(sel[" << gp.ops[q].ref << "] != 0) << " << (i % 64) << ";";
      ++i;
      if (i % 64 == 0) o << " hw[" << woff[ph] + i / 64 - 1 << "] = w_; m_ |= (uint64_t)(w_ != 0) << " << std::min<size_t>(ph, 63) << ";";
    }
    if (i % 64) o << " hw[" << woff[ph] + i / 64 << "] = w_; m_ |= (uint64_t)(w_ != 0) << " << std::min<size_t>(ph, 63) << ";";
  }
  o << " return m_; }";
  return o.str();
}


// Factor bookkeeping (fast path): each scaled gate applies M/f; per phase the
// product F_ph is shared by both copies of the phase (same gate code), per pass the
// magnitude |F| is multiplied back before the tile is stored, and the phase
// arg(F) of every pass is folded into the initial |0...0> amplitude G, so the
// stored state equals the true state after every pass.  Passes holding
// renormalising (general) sites are never scaled: their per-site norms must
// be measured in the true frame.
constexpr const char* kSplit = "\n// @@ptsbe-pass@@\n";

inline std::string generate(const GenProgram& P) {
  std::ostringstream o;
  Cx G{1.0, 0.0};
  std::vector<std::string> kernels;
  for (size_t pi = 0; pi < P.passes.size(); ++pi)
    if (hit_word_offsets(P.passes[pi]).back() > kMaxHitWords) return std::string();   // caller falls back
  for (size_t pi = 0; pi < P.passes.size(); ++pi) {
    const GenPass& gp = P.passes[pi];
    const int GB = gp.gb, N = 1 << GB;
    bool has_general = false;
    for (const DevOp& op : gp.ops)
      if (op.kind == 1 && P.chans[P.site_chan[op.ref]].general) has_general = true;
    const bool scaled = !has_general;
    const int threads = threads_for(gp.L, GB, has_general);
    const int groups = 1 << (gp.L - GB);
    const int gloop = groups / threads;   // >= 1 when threads <= groups
    const bool all_active = threads <= groups;
    // 3 CTAs/SM (<= 80 registers, small spills) hide more latency on the compute-heavy
    // 256-thread passes (config 4: -3 % on its two heaviest 4-bit passes); light
    // passes keep 2 (their spills would cost more than the extra warps give)
    int n_gates = 0;
    for (const DevOp& op : gp.ops) n_gates += op.kind == 0;
    static const int mb128 = std::getenv("PTSBE_GB5_MB") ? std::atoi(std::getenv("PTSBE_GB5_MB")) : 3;
    // complex128 256-thread passes: 2 CTAs/SM at <= 128 registers (16 amplitudes = 64 registers
    // per thread; a 3-CTA budget of 85 spills 50-200 B per thread: config 4 558 K vs 566 K)
    int min_blocks = threads <= 128 ? mb128 : (threads <= 256 ? (!P.c64 ? 2 : (n_gates >= 40 ? 3 : 2)) : 1);
    {   // never budget registers for more CTAs than the tile buffers let share an SM
      const int by_smem = std::max(1, (int)((227u << 10) / smem_bytes_for(gp.L, P.c64 ? 8 : 16)));
      min_blocks = std::min(min_blocks, by_smem);
      if (const char* e = std::getenv("PTSBE_MIN_BLOCKS")) min_blocks = std::max(1, std::atoi(e));   // A/B knob
    }
    const uint64_t nmask = P.n >= 64 ? ~0ull : ((1ull << P.n) - 1);
    const uint64_t comp = ~gp.qmask & nmask;
    const uint64_t hmask = gp.qmask & ~((1ull << gp.c) - 1);
    const Swizzle free_sw = std::getenv("PTSBE_FIXED_SWIZZLE") ? Swizzle::fixed(P.c64)   // A/B knob
                                                               : choose_swizzle(P.c64, gp.L, gp.phases, GB);
    TmaLayout tl;
    const bool tma = P.tma && tma_ok(P.c64, gp.c, gp.L) &&
                     (1 << (gp.L - (P.c64 ? 4 : 3))) / 4 <= threads &&   // one gather group per issuing lane
                     make_tma_layout(P.c64, gp.L, gp.phases, GB, free_sw, &tl);
    const Swizzle sw = tma ? tl.sw : free_sw;
    uint32_t lowm = 0;   // every bit a swizzle mask can flip (gen_prelude.cuh slot_ptr)
    for (int b = 0; b < 32; ++b) lowm |= sw.m[b];
    if (std::getenv("PTSBE_SWIZZLE_REPORT")) {   // analysis: model wavefronts, free vs TMA layout
      auto cost = [&](const Swizzle& z) { int t = 0; for (const DevPhase& D : gp.phases) t += phase_wavefronts(z, D, GB); return t; };
      std::fprintf(stderr, "pass %zu gb %d phases %zu wavefronts: free %d tma %d\n", pi, GB, gp.phases.size(),
                   cost(free_sw), tma ? cost(tl.sw) : -1);
    }
    const std::string swname = "Swz" + std::to_string(pi);
    const int teams = teams_for(gp.L, P.c64 ? 8 : 16, tma, n_gates);
    const int stages = pass_stages(gp.L, P.c64 ? 8 : 16, tma, teams);
    if (teams > 1 || stages > 2) min_blocks = 1;
    else if (!P.c64 && stages == 1 && threads == 256) {
      // light single-buffered c128 passes: CTAs per SM (2: <= 128 registers, 3: <= 85)
      static const int lb = std::getenv("PTSBE_LIGHT_BLOCKS") ? std::atoi(std::getenv("PTSBE_LIGHT_BLOCKS")) : 2;
      min_blocks = std::max(1, std::min(lb, 3));
    }
    const std::string tix = "ptg::gtid<" + std::to_string(threads) + ">()";   // team-local thread index
    Emitter ke(P.c64);
    std::ostringstream slow_fns;   // out-of-line slow variants of this pass's phases
    const std::vector<int> woff = hit_word_offsets(gp);
    std::ostringstream& k = ke.o;
    Cx F{1.0, 0.0};
    k << kTeamsTag << teams << " " << stages << "\n"
      << "extern \"C\" __global__ void __launch_bounds__(" << threads * teams << ", " << min_blocks << ") "
      << kernel_name((int)pi) << "(const ptg::PassParams p, const __grid_constant__ ptg::TMapDesc tm) {\n"
      << "  typedef " << ke.V << " V;\n"
      << "  ptg::run_pass<" << ke.R << ", " << gp.L << ", " << gp.c << ", " << (P.n - gp.L) << ", " << threads
      << ", " << (pi + 1 == P.passes.size() ? "true" : "false") << ", " << (tma ? "true" : "false") << ", " << (tma && !std::getenv("PTSBE_NO_TMA_STORE") ? "true" : "false")
      << ", " << (std::getenv("PTSBE_TMA_LANES") ? std::atoi(std::getenv("PTSBE_TMA_LANES")) : 32)
      << ", " << stages << ", " << (std::getenv("PTSBE_TMA_PREFETCH") ? "true" : "false")
      << ", " << teams << ">(p, &tm, "
      << swname << "(), " << swname << "Inv(),\n"
      << "    " << scatter_fn(comp, "uint64_t") << ",\n"
      << "    " << scatter_fn(hmask, "uint32_t") << ",\n"
      << "    " << err_mask_fn(gp) << ",\n"
      << "    [&](V* cur, uint32_t kofs, int b, const uint8_t* sel, long long tile, uint64_t base, double scale, double* red,\n"
      << "        uint64_t emask, const uint64_t* hits) {\n"
      << "    const bool active = "
      << (all_active ? std::string("true") : tix + " < " + std::to_string(groups) + "u") << ";\n"
      << "    V a[" << N << "];\n";
    for (size_t ph = 0; ph < gp.phases.size(); ++ph) {
      const DevPhase& D = gp.phases[ph];
      int pb[5];
      for (int q = 0; q < GB; ++q) pb[q] = (int)((D.pbits >> (5 * q)) & 31);
      std::vector<uint32_t> off(N), so(N);
      for (int j = 0; j < N; ++j) {
        off[j] = 0;
        for (int q = 0; q < GB; ++q)
          if ((j >> q) & 1) off[j] |= 1u << pb[q];
        so[j] = sw(off[j]);
      }
      bool has_sites = false;
      for (int q = D.op_begin; q < D.op_begin + D.n_ops; ++q) has_sites = has_sites || gp.ops[q].kind == 1;
      const bool last = ph + 1 == gp.phases.size();
      // slow == true: the trajectory takes a non-default outcome at some site of
      // this phase; sites then read their outcome and apply its operator from the
      // table (same gate code, so the frame factor is unchanged).  Each variant is
      // a complete load -> ops -> store block: no amplitude register is live across
      // the CTA-uniform branch, so the join costs no register-shuffling moves.
      int chk_lo = 0, chk_hi = 1 << 30;   // slow variant: site indices that are tested for hits
      auto emit_ops = [&](bool slow) {
        Cx f{1.0, 0.0};
        int site_i = 0;
        if (slow) {
          k << "      uint64_t hw_[" << std::max(1, woff[ph + 1] - woff[ph]) << "];\n";
          for (int w = 0; w < woff[ph + 1] - woff[ph]; ++w) k << "      hw_[" << w << "] = hits[" << woff[ph] + w << "];\n";
        }
        // Diagonal gates of the phase are multiplied into one pending
        // diagonal over the register group, deferred while it commutes with the ops
        // that follow (ops on other bits; CX whose target it does not touch; sites
        // are the identity here) and applied once -- a layer of k diagonal gates
        // costs one complex multiply per amplitude instead of k/2.  Slow variants
        // flush it before every tested site on its bits (a hit's Pauli does not
        // commute with it); all variants pull out the same pivot factors.
        std::vector<Cx> pend(N, Cx{1.0, 0.0});
        uint32_t pmask = 0;
        const bool merge_diag = !std::getenv("PTSBE_NO_DIAG_MERGE");
        auto flush = [&]() {
          if (!pmask) return;
          for (int j = 0; j < N; ++j) ke.dmul(j, Emitter::snap(pend[j]));
          std::fill(pend.begin(), pend.end(), Cx{1.0, 0.0});
          pmask = 0;
        };
        for (int q = D.op_begin; q < D.op_begin + D.n_ops; ++q) {
          const DevOp& op = gp.ops[q];
          const int k1 = op.arity == 2 ? op.k1 : 0;
          const uint32_t bits = (1u << op.k0) | (op.arity == 2 ? (1u << op.k1) : 0u);
          if (op.kind == 0) {
            const int kind = P.kinds[op.ref];
            const double* m = P.mats + (size_t)op.ref * 32;
            if (merge_diag && (kind == 2 || kind == 3 || kind == 11)) {
              Cx e[4];
              if (kind == 2) {          // diag(d0, d1), pivot-scaled like Emitter::op
                const Cx d0 = Emitter::at(m, 0, 0), d1 = Emitter::at(m, 1, 1);
                if (scaled && cxabs(d0) > 0.0) { e[0] = {1.0, 0.0}; e[1] = cxdiv(d1, d0); f = cxmul(f, d0); }
                else { e[0] = d0; e[1] = d1; }
              } else if (kind == 3) {   // diag(1, m11)
                e[0] = {1.0, 0.0}; e[1] = Emitter::at(m, 1, 1);
              } else {                  // 2-qubit diagonal, local index (bit k0) << 1 | bit k1
                for (int t = 0; t < 4; ++t) e[t] = Emitter::at(m, t, t);
              }
              for (int j = 0; j < N; ++j) {
                const int loc = op.arity == 2 ? (((j >> op.k0) & 1) << 1) | ((j >> op.k1) & 1) : ((j >> op.k0) & 1);
                pend[j] = cxmul(pend[j], e[loc]);
              }
              pmask |= bits;
              continue;
            }
            const bool commutes = kind == 9 ? !((pmask >> op.k1) & 1u) : !(pmask & bits);
            if (!commutes) flush();
            k << "      ";
            f = cxmul(f, ke.op(kind, op.k0, k1, m, scaled));
            continue;
          }
          const ptsbe_channel& ch = P.chans[P.site_chan[op.ref]];
          const int si = site_i++;
          // a tested site (slow variant) may apply any outcome, a non-identity default
          // acts here, a renormalising site reads every amplitude: the pending diagonal
          // goes first
          const bool checked = slow && si >= chk_lo && si < chk_hi;
          if (ch.general || ((checked || !(ch.identity_mask & 1ull)) && (pmask & bits))) flush();
          if (slow && si >= chk_lo && si < chk_hi) {
            // hit: this trajectory's outcome at the site is not 0 -> apply it from the table
            // 32-bit halves + immediate mask: one predicate-setting LOP3 per site on the no-hit path
            k << "      if (__builtin_expect(((uint32_t)(hw_[" << si / 64 << "] >> " << (si % 64 >= 32 ? 32 : 0)
              << ") & 0x" << std::hex << (1u << (si % 32)) << std::dec << "u) != 0, 0)) { const int o_ = sel[" << op.ref
              << "];\n"
              << "        if (!((0x" << std::hex << ch.identity_mask << std::dec << "ull >> o_) & 1ull)) {\n"
              << "          const V* m_ = reinterpret_cast<const V*>(p.mats) + (size_t)(" << ch.mat_base
              << " + o_) * 16;\n";
            if (ch.identity_mask & 1ull) {   // through the tile slots (no register shuffle on the no-hit path)
              k << "          if (active) { ptg::stg<V, " << N << ", " << pb[0] << ", " << lowm << "u>(a, cur, sg, so, true);\n"
                << "            ptg::err_apply<V, " << GB << ", " << swname << ">(cur, gb, " << D.pbits << "u, "
            << op.arity << ", "
                << op.k0 << ", " << k1 << ", m_);\n"
                << "            ptg::ldg<V, " << N << ", " << pb[0] << ", " << lowm << "u>(a, cur, sg, so, true, 1.0); }\n";
            } else {
              if (op.arity == 1) k << "          ptg::g1<" << op.k0 << ">(a, m_[0], m_[1], m_[4], m_[5]);\n";
              else k << "          ptg::g2<" << op.k0 << ", " << k1 << ">(a, m_);\n";
            }
            k << "      } }";
            if (!(ch.identity_mask & 1ull)) {   // no hit: outcome 0, which is not the identity
              k << " else {\n        ";
              ke.op(P.kinds[ch.mat_base], op.k0, k1, P.mats + (size_t)ch.mat_base * 32, false);
              k << "      }";
            }
            k << "\n";
          } else if (!(ch.identity_mask & 1ull)) {   // outcome 0 is not the identity (e.g. damping K0): no hit here
            k << "      ";
            ke.op(P.kinds[ch.mat_base], op.k0, k1, P.mats + (size_t)ch.mat_base * 32, false);
          }
          if (ch.general) {
            k << "      { double s_ = 0.0;\n"
              << "#pragma unroll\n"
              << "        for (int j = 0; j < " << N << "; ++j) s_ += ptg::prob64(a[j]);\n"
              << "        s_ = ptg::block_sum<" << threads << ">(s_, red);\n"
              << "        if (" << tix << " == 0) p.partials[((size_t)" << op.slot
              << " * p.B + b) * p.tiles + tile] = s_; }\n";
          }
        }
        flush();
        return f;
      };
      auto emit_block = [&](bool slow) {
        if (gloop > 1)
          k << "    #pragma unroll 1\n    for (uint32_t g = " << tix << "; g < " << groups << "u; g += " << threads
            << "u) {\n";
        else
          k << "    { const uint32_t g = " << tix << ";\n";
        k << "      const uint32_t gb = ";
        for (int q = 0; q < GB; ++q) k << "ptg::ins0(";
        k << "g";
        for (int q = 0; q < GB; ++q) k << ", " << pb[q] << ")";
        k << ";\n      const uint32_t sg = " << swname << "()(gb) | kofs;\n      const uint32_t so[" << N << "] = {";
        for (int j = 0; j < N; ++j) k << so[j] << "u" << (j + 1 < N ? ", " : "");
        k << "};\n";
        if (ph == 0) {
          k << "      const uint32_t off[" << N << "] = {";
          for (int j = 0; j < N; ++j) k << off[j] << "u" << (j + 1 < N ? ", " : "");
          k << "};\n"
            << "      if (p.gen_zero) ptg::zerog(a, base, gb, off, active && p.gen_zero == 1, GZERO_RE, GZERO_IM);\n"
            << "      else ptg::ldg<V, " << N << ", " << pb[0] << ", " << lowm << "u>(a, cur, sg, so, active, scale);\n";
          if (pi == 0)   // a loaded (not synthesized) input also needs the global phase G
            k << "      if (!p.gen_zero) ptg::cscale(a, ptg::mk((V*)0, GZERO_RE, GZERO_IM));\n";
        } else {
          k << "      ptg::ldg<V, " << N << ", " << pb[0] << ", " << lowm << "u>(a, cur, sg, so, active, 1.0);\n";
        }
        const Cx f = emit_ops(slow);
        if (last) {
          const double mag = cxabs(cxmul(F, f));
          if (mag != 1.0) k << "      ptg::rscale(a, " << hexd(mag) << ");\n";
        }
        k << "      ptg::stg<V, " << N << ", " << pb[0] << ", " << lowm << "u>(a, cur, sg, so, active);\n"
          << "    }\n";
        return f;
      };
      k << "    { // phase " << ph << "\n";
      const bool branchy = has_sites;
      if (branchy) k << "    if (!((emask >> " << std::min<size_t>(ph, 63) << ") & 1ull)) {\n";
      const Cx Fph = emit_block(false);
      static const bool no_slow = std::getenv("PTSBE_GEN_ANALYSE_FAST_ONLY") != nullptr;   // offline analysis only
      if (!branchy) {
      } else if (no_slow) {
        k << "    }\n";
      } else {
        // The slow variants live out of line (non-inlined functions), so the hot
        // straight-line code stays dense in the instruction cache.  A phase with up to
        // 64 sites also gets one variant per segment of 8 consecutive sites (PTSBE_SEG) that
        // tests only that segment: a trajectory whose hits in the phase fall in one
        // segment (the common case) runs a function several times smaller than the full one,
        // which matters because slow code is instruction-fetch bound.
        const std::string base_name = "ptsbe_slow_" + std::to_string(pi) + "_" + std::to_string(ph);
        const char* args = "(p.mats, p.partials, p.B, p.tiles, p.gen_zero, cur + kofs, b, sel, tile, base, scale, red, active, "
                           "hits)";
        auto emit_variant = [&](const std::string& fname, int lo, int hi) {
          const std::string before = k.str();
          chk_lo = lo;
          chk_hi = hi;
          emit_block(true);
          chk_lo = 0;
          chk_hi = 1 << 30;
          const std::string all = k.str();
          slow_fns << "__device__ __noinline__ void " << fname << "(const void* mats_, double* partials_, int B_, "
                   << "long long tiles_, int gen_zero_, " << ke.V << "* cur, int b, const uint8_t* sel, long long tile, "
                   << "uint64_t base, double scale, double* red, bool active, const uint64_t* hits) {\n"
                   << "  typedef " << ke.V << " V;\n"
                   << "  const uint32_t kofs = 0u;   // cur is this tile's buffer\n"
                   << "  struct { const void* mats; double* partials; int B; long long tiles; int gen_zero; } p = "
                   << "{mats_, partials_, B_, tiles_, gen_zero_};\n"
                   << "  V a[" << N << "];\n"
                   << all.substr(before.size()) << "}\n";
          k.str(before);
          k.seekp(0, std::ios_base::end);
        };
        int nsites = 0;
        for (int q = D.op_begin; q < D.op_begin + D.n_ops; ++q) nsites += gp.ops[q].kind == 1;
        static const int SEG = std::getenv("PTSBE_SEG") ? std::max(1, std::atoi(std::getenv("PTSBE_SEG"))) : 8;
        const int nseg = (nsites + SEG - 1) / SEG;
        static const bool no_seg = std::getenv("PTSBE_NO_SEGMENT_VARIANTS") != nullptr;   // A/B knob
        k << "    } else {\n";
        if (nsites <= 64 && nseg >= 2 && !no_seg) {
          k << "      const uint64_t hw0_ = hits[" << woff[ph] << "];\n      ";
          for (int sgi = 0; sgi < nseg; ++sgi) {
            const uint64_t own = (sgi * SEG + SEG >= 64 ? ~0ull : ((1ull << (sgi * SEG + SEG)) - 1)) &
                                 ~((1ull << (sgi * SEG)) - 1);
            k << "if (!(hw0_ & 0x" << std::hex << ~own << std::dec << "ull)) " << base_name << "_s" << sgi << args
              << ";\n      else ";
            emit_variant(base_name + "_s" + std::to_string(sgi), sgi * SEG, sgi * SEG + SEG);
          }
        }
        k << base_name << args << ";\n    }\n";
        emit_variant(base_name, 0, 1 << 30);
      }
      F = cxmul(F, Fph);
      k << "      ptg::gsync<" << threads << ">();\n";
      k << "    }\n";
    }
    k << "  }, RowTab" << pi << "());\n}\n";
    const double mag = cxabs(F);
    G = cxmul(G, Cx{F.re / mag, F.im / mag});
    kernels.push_back(swizzle_struct(swname, sw, gp.L) + slot_inv_struct(swname + "Inv", tl) +
                      rowtab_struct("RowTab" + std::to_string(pi), tma, P.c64, gp.c, gp.L, hmask, tl) +
                      slow_fns.str() + k.str());
  }
  if (std::getenv("PTSBE_TEAM_TAIL_SYNC")) o << "#define PTG_TEAM_TAIL_SYNC 1\n";
  o << kGenPrelude << "\n"
    << "#define GZERO_RE " << hexd(G.re) << "\n#define GZERO_IM " << hexd(G.im) << "\n";
  for (auto& kt : kernels) o << kSplit << kt;   // compile() builds one NVRTC program per pass
  return o.str();
}

// ---------------------------------------------------------------- compile + cache
struct Module {
  std::vector<CUmodule> mods;
  std::vector<CUfunction> fns;
  std::vector<int> teams;    // compute teams per CTA of each pass kernel (kTeamsTag in its source)
  std::vector<int> stages;   // tile buffers of a one-team pass kernel (kTeamsTag)
};

// One NVRTC program per pass (shared header: prelude + global-phase defines),
// compiled on parallel host threads: program load time scales with the largest
// pass instead of the sum (config 4: 12 passes).
inline bool compile(const std::string& src, int n_passes, int dev, Module& out, std::string& err) {
  Api& A = api();
  if (!A.ok) { err = A.why; return false; }
  if (src.empty()) { err = "program exceeds the generated kernels' limits (noise sites per pass)"; return false; }
  static std::mutex mu;
  static std::map<std::pair<int, std::string>, Module> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, src);
  auto it = cache.find(key);
  if (it != cache.end()) { out = it->second; return true; }
  const std::string split(kSplit);
  std::vector<std::string> parts;
  size_t pos = src.find(split);
  const std::string header = src.substr(0, pos);
  while (pos != std::string::npos) {
    const size_t next = src.find(split, pos + split.size());
    parts.push_back(header + src.substr(pos + split.size(), next == std::string::npos ? std::string::npos
                                                                                       : next - pos - split.size()));
    pos = next;
  }
  if ((int)parts.size() != n_passes) { err = "generated source does not hold one kernel per pass"; return false; }
  std::vector<std::vector<char>> cubins(parts.size());
  std::vector<std::string> errs(parts.size());
  auto build = [&](size_t i) {
    void* prog = nullptr;
    if (A.create(&prog, parts[i].c_str(), "ptsbe_gen.cu", 0, nullptr, nullptr) != 0) {
      errs[i] = "nvrtcCreateProgram failed";
      return;
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--device-as-default-execution-space"};
    if (A.compile(prog, 4, opts) != 0) {
      size_t n = 0;
      A.log_size(prog, &n);
      std::string log(n, '\0');
      if (n) A.get_log(prog, &log[0]);
      errs[i] = "NVRTC compile failed: " + log.substr(0, 2000);
    } else {
      size_t n = 0;
      A.cubin_size(prog, &n);
      cubins[i].resize(n);
      A.get_cubin(prog, cubins[i].data());
    }
    A.destroy(&prog);
  };
  {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> pool;
    std::atomic<size_t> next{0};
    for (unsigned t = 0; t < std::min<unsigned>(hw, (unsigned)parts.size()); ++t)
      pool.emplace_back([&] {
        for (size_t i; (i = next.fetch_add(1)) < parts.size();) build(i);
      });
    for (auto& th : pool) th.join();
  }
  for (auto& e : errs)
    if (!e.empty()) { err = e; return false; }
  Module m;
  for (int i = 0; i < n_passes; ++i) {
    CUmodule mod = nullptr;
    if (A.module_load(&mod, cubins[i].data()) != CUDA_SUCCESS) { err = "cuModuleLoadData failed"; return false; }
    m.mods.push_back(mod);
    CUfunction f = nullptr;
    if (A.get_function(&f, mod, kernel_name(i).c_str()) != CUDA_SUCCESS) { err = "cuModuleGetFunction failed"; return false; }
    A.func_set_attr(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 227 * 1024);
    m.fns.push_back(f);
    const size_t tp = parts[i].find(kTeamsTag, header.size());
    int tv = 1, sv = 0;
    if (tp != std::string::npos) std::sscanf(parts[i].c_str() + tp + std::strlen(kTeamsTag), "%d %d", &tv, &sv);
    m.teams.push_back(std::max(1, tv));
    m.stages.push_back(sv);
  }
  cache[key] = m;
  out = m;
  return true;
}

inline size_t smem_bytes_for(int L, size_t amp_bytes, int teams, int stages) {
  // [1024-B alignment slack for TMA's 128-B swizzle] tile buffers (three for two teams) |
  // mbarriers + stamps | red | emask | hits per team | TMA row table (gen_prelude.cuh run_pass)
  const size_t nbuf = teams > 1 ? 3 : stages > 0 ? (size_t)stages : (size_t)stages_for(L, amp_bytes);
  return 1024 + nbuf * ((size_t)1 << L) * amp_bytes + 64 + 32 * 8 + 16 + 8 * kMaxHitWords * (size_t)teams + 16 * 128;
}
inline size_t smem_bytes(int L, int /*c*/, size_t amp_bytes, int teams = 1, int stages = 0) {
  return smem_bytes_for(L, amp_bytes, teams, stages);
}

}  // namespace gen
}  // namespace ptsbe
