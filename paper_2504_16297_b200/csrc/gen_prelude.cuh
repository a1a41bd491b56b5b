// gen_prelude.cuh -- device prelude of the circuit-specialised pass kernels.
//
// At ptsbe_load_program time engine.cu emits, for every fused pass, a phase
// body in which every gate is a straight-line call with compile-time register
// positions and literal matrix entries (cx / swap become pure register
// renaming), and every noise site is a CTA-uniform test of the trajectory's
// outcome.  NVRTC compiles prelude + bodies for sm_100a; the persistent,
// cp.async double-buffered tile loop below is shared by all passes.
//
// A phase keeps N = 2^GB amplitudes per thread in registers (GB = 4 or 5 tile
// bits); the gate templates deduce N from the register array.
//
// This file is embedded verbatim as a string (gen_prelude.inc, produced by
// build.py) -- it is NOT compiled by nvcc directly.  Keep PassParams identical
// to pass_kernels.cuh.
#if defined(__CUDACC_RTC__)   // NVRTC has no <stdint.h>; nvcc (tools/gen_offline.py) does
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef unsigned char uint8_t;
typedef long long int64_t;
#else
#include <stdint.h>
#endif

namespace ptg {

#ifndef PTG_TEAM_TAIL_SYNC
#define PTG_TEAM_TAIL_SYNC 0   // 1: team barrier after every tile's TMA store (PTSBE_TEAM_TAIL_SYNC)
#endif
#define PTG_MAX_HIT_WORDS 480   // = codegen.h kMaxHitWords (shared-memory room for the hit words)

struct DevOp { int32_t kind, arity, b0, b1, ref, slot, k0, k1; };
struct DevPhase { uint32_t pbits; int32_t op_begin, n_ops, pad; };
struct DevChan { int32_t n_outcomes, mat_base, general, arity; uint64_t identity_mask; };
struct PassParams {
  void* states; int n; int L; int c; uint64_t qmask;
  const DevOp* ops; int n_ops; const DevPhase* phases; int n_phases;
  const uint8_t* sel; int S; const int32_t* site_chan; const DevChan* chans;
  const void* mats; const int32_t* mat_kind; const double* nst; int use_scale; int gen_zero;
  double* partials; const int32_t* status; int B; long long tiles;
  const int4* ent; int E;   // launch entries {trajectory row, src slot, dst slot, 0}
  uint64_t* tsum; long long tsum_stride; int tsum_sbits;   // fused sampler block sums (last pass)
};

template <typename R> struct Cplx;
template <> struct Cplx<float> { typedef float2 V; typedef float4 W; };
template <> struct Cplx<double> { typedef double2 V; typedef double2 W; };

__device__ __forceinline__ float2 mk(float2*, double x, double y) { return make_float2((float)x, (float)y); }
__device__ __forceinline__ double2 mk(double2*, double x, double y) { return make_double2(x, y); }

// Packed (re, im) arithmetic.  complex64 uses Blackwell's FP32x2 instructions
// (FFMA2 / FMUL2 / FADD2).  Complex products are written as
//   d * x = x * d.re + (i x) * d.im,   i x = (-x.im, x.re)
// so that, with a literal d, each term is ONE instruction: the scalar is a
// 32-bit immediate broadcast to both lanes and i*x is an operand modifier
// (FFMA2 Rd, -Rx.F32x2.LO_HI.NP, imm, Rc) -- no register pairs of constants
// (which cost two MOVs per use).  complex128 falls back to scalar DFMA.
__device__ __forceinline__ float2 pfma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 pmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 padd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ double2 pfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, c.x), fma(a.y, b.y, c.y));
}
__device__ __forceinline__ double2 pmul(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
__device__ __forceinline__ double2 padd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
template <typename V, typename S> __device__ __forceinline__ V bc(S s) { V r; r.x = s; r.y = s; return r; }
template <typename V> __device__ __forceinline__ V ix(V x) { V r; r.x = -x.y; r.y = x.x; return r; }   // i * x
template <typename V> __device__ __forceinline__ V neg(V x) { V r; r.x = -x.x; r.y = -x.y; return r; }

template <typename V> __device__ __forceinline__ V cmul(V d, V x) {     // d * x
  typedef decltype(d.x) R;
  return pfma(ix(x), bc<V, R>(d.y), pmul(x, bc<V, R>(d.x)));
}
template <typename V> __device__ __forceinline__ V cmadd2(V m0, V a, V m1, V b) {   // m0*a + m1*b
  typedef decltype(a.x) R;
  return pfma(ix(b), bc<V, R>(m1.y), pfma(b, bc<V, R>(m1.x), pfma(ix(a), bc<V, R>(m0.y), pmul(a, bc<V, R>(m0.x)))));
}
template <typename V> __device__ __forceinline__ V cmadd4(V m0, V m1, V m2, V m3, V a, V b, V c, V d) {
  typedef decltype(a.x) R;
  V r = pmul(a, bc<V, R>(m0.x));
  r = pfma(ix(a), bc<V, R>(m0.y), r);
  r = pfma(b, bc<V, R>(m1.x), r);
  r = pfma(ix(b), bc<V, R>(m1.y), r);
  r = pfma(c, bc<V, R>(m2.x), r);
  r = pfma(ix(c), bc<V, R>(m2.y), r);
  r = pfma(d, bc<V, R>(m3.x), r);
  return pfma(ix(d), bc<V, R>(m3.y), r);
}
// Fixed-point probability of the fused sampler sums (2^-62 units); identical
// definition in sample_kernels.cuh qfix (the resolve step recomputes it).
__device__ __forceinline__ uint64_t qfix(float2 a) {
  return __float2ull_rn(__fmul_rn(__fmaf_rn(a.x, a.x, __fmul_rn(a.y, a.y)), 0x1p62f));
}
__device__ __forceinline__ uint64_t qfix(double2 a) {
  return __double2ull_rn(__dmul_rn(__fma_rn(a.x, a.x, __dmul_rn(a.y, a.y)), 0x1p62));
}
__device__ __forceinline__ double prob64(float2 a) {
  const double x = a.x, y = a.y;
  return __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
}
__device__ __forceinline__ double prob64(double2 a) {
  return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// ---- gate kernels on an N-amplitude register group; K* compile-time bit positions
template <int K, typename V, int N> __device__ __forceinline__ void g1(V (&a)[N], V m00, V m01, V m10, V m11) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = cmadd2(m00, x, m01, y);
      a[j | (1 << K)] = cmadd2(m10, x, m11, y);
    }
}
template <int K, typename V, int N, typename R> __device__ __forceinline__ void g1r(V (&a)[N], R m00, R m01, R m10, R m11) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = pfma(bc<V>(m01), y, pmul(bc<V>(m00), x));
      a[j | (1 << K)] = pfma(bc<V>(m11), y, pmul(bc<V>(m10), x));
    }
}
// [[1, t0], [t1, 1]] -- a pivot-scaled real rotation (ry): one packed FMA per output
template <int K, typename V, int N, typename R> __device__ __forceinline__ void g1rot(V (&a)[N], R t0, R t1) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = pfma(bc<V>(t0), y, x);
      a[j | (1 << K)] = pfma(bc<V>(t1), x, y);
    }
}
// [[1, 1], [1, -1]] -- a pivot-scaled Hadamard: add / subtract butterfly
template <int K, typename V, int N> __device__ __forceinline__ void g1h(V (&a)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = padd(x, y);
      a[j | (1 << K)] = pfma(y, bc<V>(-1.0f), x);
    }
}
template <int K, typename V, int N> __device__ __forceinline__ void g1d(V (&a)[N], V d0, V d1) {
#pragma unroll
  for (int j = 0; j < N; ++j) a[j] = cmul((j & (1 << K)) ? d1 : d0, a[j]);
}
template <int K, typename V, int N> __device__ __forceinline__ void g1p(V (&a)[N], V d1) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j & (1 << K)) a[j] = cmul(d1, a[j]);
}
template <int K, typename V, int N> __device__ __forceinline__ void g1a(V (&a)[N], V m01, V m10) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = cmul(m01, y); a[j | (1 << K)] = cmul(m10, x);
    }
}
template <int K, typename V, int N> __device__ __forceinline__ void g1x(V (&a)[N]) {   // X: renaming only
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << K))) { const V t = a[j]; a[j] = a[j | (1 << K)]; a[j | (1 << K)] = t; }
}
template <int K, typename V, int N> __device__ __forceinline__ void g1neg(V (&a)[N]) {    // diag(1, -1)
  typedef decltype(a[0].x) R;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j & (1 << K)) a[j] = pmul(a[j], bc<V, R>((R)-1));
}
template <int K, typename V, int N> __device__ __forceinline__ void g1pi(V (&a)[N], bool neg) {   // diag(1, ±i)
  typedef decltype(a[0].x) R;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j & (1 << K)) a[j] = pmul(ix(a[j]), bc<V, R>(neg ? (R)-1 : (R)1));
}
template <int KH, int KL, typename V, int N> __device__ __forceinline__ void g2(V (&a)[N], const V* m) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (!(j & (1 << KH)) && !(j & (1 << KL))) {
      const int i1 = j | (1 << KL), i2 = j | (1 << KH), i3 = j | (1 << KH) | (1 << KL);
      const V v0 = a[j], v1 = a[i1], v2 = a[i2], v3 = a[i3];
      a[j] = cmadd4(m[0], m[1], m[2], m[3], v0, v1, v2, v3);
      a[i1] = cmadd4(m[4], m[5], m[6], m[7], v0, v1, v2, v3);
      a[i2] = cmadd4(m[8], m[9], m[10], m[11], v0, v1, v2, v3);
      a[i3] = cmadd4(m[12], m[13], m[14], m[15], v0, v1, v2, v3);
    }
}
template <int KH, int KL, typename V, int N> __device__ __forceinline__ void g2cx(V (&a)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if ((j & (1 << KH)) && !(j & (1 << KL))) { const V t = a[j]; a[j] = a[j | (1 << KL)]; a[j | (1 << KL)] = t; }
}
template <int KH, int KL, typename V, int N> __device__ __forceinline__ void g2sw(V (&a)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if ((j & (1 << KH)) && !(j & (1 << KL))) {
      const int o = (j & ~(1 << KH)) | (1 << KL);
      const V t = a[j]; a[j] = a[o]; a[o] = t;
    }
}
template <int KH, int KL, int S, typename V, int N> __device__ __forceinline__ void g2dsel(V (&a)[N], V d) {
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (((j >> KH) & 1) * 2 + ((j >> KL) & 1) == S) a[j] = cmul(d, a[j]);
}
template <typename V, int N> __device__ __forceinline__ void cscale(V (&a)[N], V d) {
#pragma unroll
  for (int j = 0; j < N; ++j) a[j] = cmul(d, a[j]);
}
template <typename V, int N> __device__ __forceinline__ void rscale(V (&a)[N], double s) {
  typedef decltype(a[0].x) R;
#pragma unroll
  for (int j = 0; j < N; ++j) a[j] = pmul(a[j], bc<V, R>((R)s));
}

// ---- addressing
// (shared-memory swizzles are per pass: codegen.h Swizzle / swizzle_struct)
__device__ __forceinline__ uint32_t ins0(uint32_t p, int bit) {
  const uint32_t lo = p & ((1u << bit) - 1u);
  return ((p ^ lo) << 1) | lo;
}
__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

// ---- TMA tile staging (sm_100a): the state viewed as rows of 128 B (16 x 8-B words), one
// 2-D tensor map over every state slot; a tile's rows are gathered four at a time
// (tile::gather4: four arbitrary row coordinates -> 512 contiguous B of shared memory,
// 128-B swizzled) and written back with tile::scatter4.  Completion of the gathers is
// an mbarrier transaction count; the scatters are bulk groups.
struct __align__(64) TMapDesc { unsigned long long opaque[16]; };
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const TMapDesc* tm, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)), "l"(tm), "r"(0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_scatter4(const TMapDesc* tm, int r0, int r1, int r2, int r3, const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n"
      ::"l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_prefetch4(const TMapDesc* tm, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile::gather4 [%0, {%1, %2, %3, %4, %5}];\n"
               ::"l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
// Warp-uniform issue: the whole (converged) warp executes these with warp-uniform operands;
// elect.sync keeps the copy to one issue, and because the operands are uniform ptxas emits
// a single UTMALDG / UTMASTG from uniform registers (no per-lane ELECT / R2UR.BROADCAST /
// BRA.U.ANY waterfall loop, which the per-lane form above compiles to).
__device__ __forceinline__ void tma_gather4_w(void* dst, const TMapDesc* tm, int r0, int r1, int r2, int r3,
                                              uint64_t* bar) {
  asm volatile(
      "{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n"
      "@P cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n}\n" ::"r"(smem_u32(dst)), "l"(tm), "r"(0), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_scatter4_w(const TMapDesc* tm, int r0, int r1, int r2, int r3, const void* src) {
  asm volatile(
      "{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n"
      "@P cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n}\n"
      ::"l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_prefetch4_w(const TMapDesc* tm, int r0, int r1, int r2, int r3) {
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n"
               "@P cp.async.bulk.prefetch.tensor.2d.L2.global.tile::gather4 [%0, {%1, %2, %3, %4, %5}];\n}\n"
               ::"l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx_w(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n"
               "@P mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_w(uint64_t* bar) {
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n"
               "@P mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

// A CTA runs one or two compute TEAMS of NT threads (run_pass TEAMS): generated code
// addresses its team-local thread index and synchronises its team only (named
// barrier 1 + team; with one team that is the whole CTA).
template <int NT> __device__ __forceinline__ uint32_t gtid() { return threadIdx.x & (uint32_t)(NT - 1); }
template <int NT> __device__ __forceinline__ void gsync() {
  asm volatile("bar.sync %0, %1;\n" ::"r"(1u + threadIdx.x / (uint32_t)NT), "n"(NT) : "memory");
}

template <int NT> __device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const uint32_t t = gtid<NT>();
  if ((t & 31) == 0) red[t >> 5] = v;
  gsync<NT>();
  double r = 0.0;
  if (t == 0) {
    for (int i = 0; i < (NT + 31) / 32; ++i) r += red[i];
  }
  gsync<NT>();
  return r;
}

// ---- phase register load / store (N amplitudes at sg ^ so[j]; so[] literal)
// The swizzle flips only the bits M (codegen.h: OR of its masks), and a phase's register
// offsets are disjoint from the thread's base outside M, so
//   sg ^ so[j] == (sg ^ (so[j] & M)) + (so[j] & ~M):
// one base register per distinct low pattern of the phase and every access an immediate
// offset from it -- no per-access address arithmetic.
template <uint32_t M, typename V>
__device__ __forceinline__ V* slot_ptr(V* cur, uint32_t sg, uint32_t so) {
  return cur + (sg ^ (so & M)) + (so & ~M);
}
template <typename V, int N, int P0, uint32_t M>
__device__ __forceinline__ void ldg(V (&a)[N], const V* cur, uint32_t sg, const uint32_t* so, bool active,
                                    double scale) {
  if (!active) {
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = mk((V*)0, 0.0, 0.0);
    return;
  }
  if (sizeof(V) == 8 && P0 == 0) {      // bit 0 in the phase: adjacent pairs, 16-B accesses
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const float4 w = *reinterpret_cast<const float4*>(slot_ptr<M>(cur, sg, so[j]));
      a[j] = mk((V*)0, w.x, w.y);
      a[j + 1] = mk((V*)0, w.z, w.w);
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = *slot_ptr<M>(cur, sg, so[j]);
  }
  if (scale != 1.0) rscale(a, scale);
}
template <typename V, int N, int P0, uint32_t M>
__device__ __forceinline__ void stg(const V (&a)[N], V* cur, uint32_t sg, const uint32_t* so, bool active) {
  if (!active) return;
  if (sizeof(V) == 8 && P0 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      float4 w; w.x = a[j].x; w.y = a[j].y; w.z = a[j + 1].x; w.w = a[j + 1].y;
      *reinterpret_cast<float4*>(slot_ptr<M>(cur, sg, so[j])) = w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) *slot_ptr<M>(cur, sg, so[j]) = a[j];
  }
}
// A non-default outcome (slow variant of a phase): the thread's N amplitudes are
// stored to their own tile slots, this out-of-line routine applies the outcome's
// operator there, and the caller reloads them.  Keeping the operator off the
// register path means the per-site branch joins with the registers unchanged,
// so the common (no-hit) path pays no register-shuffling moves.  k0 / k1 are
// register-bit positions (first-listed target = MSB of the local index).
template <typename V, int GB, class Sw>
__device__ __noinline__ void err_apply(V* cur, uint32_t gb, uint32_t pbits, int arity, int k0, int k1, const V* m) {
  constexpr int N = 1 << GB;
  uint32_t pos[GB];
#pragma unroll
  for (int q = 0; q < GB; ++q) pos[q] = 1u << ((pbits >> (5 * q)) & 31);
  auto addr = [&](int j) {
    uint32_t off = 0;
#pragma unroll
    for (int q = 0; q < GB; ++q)
      if ((j >> q) & 1) off |= pos[q];
    return Sw()(gb | off);
  };
  if (arity == 1) {
    const V m00 = m[0], m01 = m[1], m10 = m[4], m11 = m[5];
#pragma unroll 1
    for (int j = 0; j < N; ++j)
      if (!(j & (1 << k0))) {
        const uint32_t a0 = addr(j), a1 = addr(j | (1 << k0));
        const V x = cur[a0], y = cur[a1];
        cur[a0] = cmadd2(m00, x, m01, y);
        cur[a1] = cmadd2(m10, x, m11, y);
      }
  } else {
#pragma unroll 1
    for (int j = 0; j < N; ++j)
      if (!(j & (1 << k0)) && !(j & (1 << k1))) {
        const uint32_t a0 = addr(j), a1 = addr(j | (1 << k1)), a2 = addr(j | (1 << k0)),
                       a3 = addr(j | (1 << k0) | (1 << k1));
        const V v0 = cur[a0], v1 = cur[a1], v2 = cur[a2], v3 = cur[a3];
        cur[a0] = cmadd4(m[0], m[1], m[2], m[3], v0, v1, v2, v3);
        cur[a1] = cmadd4(m[4], m[5], m[6], m[7], v0, v1, v2, v3);
        cur[a2] = cmadd4(m[8], m[9], m[10], m[11], v0, v1, v2, v3);
        cur[a3] = cmadd4(m[12], m[13], m[14], m[15], v0, v1, v2, v3);
      }
  }
}

// |0...0> times the program's accumulated global phase G (see codegen.h)
template <typename V, int N>
__device__ __forceinline__ void zerog(V (&a)[N], uint64_t base, uint32_t gb, const uint32_t* off, bool active,
                                      double g_re, double g_im) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const bool one = active && base == 0 && (gb | off[j]) == 0;
    a[j] = mk((V*)0, one ? g_re : 0.0, one ? g_im : 0.0);
  }
}

// Persistent, double-buffered tile loop shared by every generated pass kernel.
// Compile-time: R, tile bits L, contiguous low bits C, TLOG = n - L, threads NT.
// tile_base(tile) / row_off(r) scatter bits onto the pass's fixed qubit masks
// (generated per pass as shift/mask runs).  Each thread's 16-B vectors sit at
// rows r0 + k*RSTEP with a fixed in-row offset, so their shared and global
// offsets are a per-thread base plus compile-time constants (swz and the row
// scatter are linear on disjoint bits).  err_mask(sel_row) runs once per CTA
// per trajectory (and fills the hit words).  body(cur, b, sel_row, tile, base,
// scale, red, emask, hits) runs
// the pass's phases on one tile.
template <typename R, int L, int C, int TLOG, int NT, bool SUMS, bool TMA, bool TMA_ST, int TMA_LANES, int STAGES,
          bool TMA_PF, int TEAMS, class Sw, class SlotInv, class TileBase, class RowOff, class ErrMask, class Body,
          class RowTabC>
__device__ __forceinline__ void run_pass(const PassParams& p, const TMapDesc* tm, Sw swz_, SlotInv slot_inv,
                                         TileBase tile_base, RowOff row_off, ErrMask err_mask, Body body,
                                         RowTabC rowtab_c) {
  typedef typename Cplx<R>::V V;
  typedef typename Cplx<R>::W W;
  constexpr int VPW = sizeof(W) / sizeof(V);
  constexpr uint32_t TL = 1u << L;
  constexpr int THREADS = NT;
  // rows of 2^C contiguous amplitudes longer than the CTA's threads are walked as 2^(C - CE)
  // sub-rows of 2^CE (CE: one 16-B vector per thread per sub-row), so the per-thread vector
  // layout (and the fused sampler sums) works for every pass; roff(r) scatters a sub-row index
  constexpr int CPR_FULL = C - (VPW == 2 ? 1 : 0);
  constexpr int TLOG2 = NT >= 1024 ? 10 : NT >= 512 ? 9 : NT >= 256 ? 8 : NT >= 128 ? 7 : NT >= 64 ? 6 : 5;
  constexpr int CPR_LOG = CPR_FULL < TLOG2 ? CPR_FULL : TLOG2;   // 16-B vectors per (sub-)row, log2
  constexpr int CE = CPR_LOG + (VPW == 2 ? 1 : 0);
  constexpr uint32_t NVEC = TL / VPW;
  constexpr bool FAST = THREADS >= (1 << CPR_LOG) && (NVEC % THREADS) == 0;
  constexpr int ITER = FAST ? (int)(NVEC / THREADS) : 1;
  constexpr int RSTEP = FAST ? (THREADS >> CPR_LOG) : 1;   // row stride between a thread's vectors
  // TMA rows: 128 B = 2^LOGU amplitudes; a tile is 2^(L - LOGU) rows, gathered in groups of 4
  constexpr int LOGU = sizeof(V) == 8 ? 4 : 3;
  constexpr int NGRP = TMA ? (1 << (L - LOGU)) / 4 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // TMA's 128-B swizzle needs 1024-B aligned tiles (the engine adds the slack)
  unsigned char* smem = TMA ? smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) : smem_raw;
  // layout (codegen.h smem_bytes_for): tile buffers | 4 mbarriers + 4 stamps | red[32] | emask[2] |
  // hit words per team | TMA row table
  constexpr int NBUF = TEAMS > 1 ? 3 : STAGES;
  V* buf0 = reinterpret_cast<V*>(smem);
  V* buf1 = STAGES >= 2 ? buf0 + TL : buf0;   // one buffer: tiles load after the previous one is stored
  uint64_t* mbar = reinterpret_cast<uint64_t*>(buf0 + (size_t)NBUF * TL);   // TMA: one transaction barrier per buffer
  volatile int* stamp = reinterpret_cast<volatile int*>(mbar + 4);   // teams: tile counter loaded per buffer
  double* red_all = reinterpret_cast<double*>(mbar + 8);
  uint64_t* emask_all = reinterpret_cast<uint64_t*>(red_all + 32);
  uint64_t* hits_all = emask_all + 2;   // per-phase hit words (codegen.h err_mask_fn), one set per team
  // TMA: tile-relative row coordinates of each gather group (shared-memory slots 4g..4g+3)
  uint4* rowtab = reinterpret_cast<uint4*>(hits_all + TEAMS * PTG_MAX_HIT_WORDS);
  static_assert(TEAMS == 1 || NT <= 512, "two teams: at most 16 warps each (red)");
  const uint32_t team = TEAMS > 1 ? threadIdx.x / (uint32_t)NT : 0u;
  double* red = red_all + team * 16u;
  uint64_t* emask_s = emask_all + team;
  uint64_t* hits_s = hits_all + (size_t)team * PTG_MAX_HIT_WORDS;
  int lb = -1;
  const uint32_t tid = gtid<NT>();   // team-local
  auto roff = [&](uint32_t r) -> uint64_t {
    return ((uint64_t)(r & ((1u << (C - CE)) - 1u)) << CE) | row_off(r >> (C - CE));
  };
  const uint32_t j0 = tid & ((1u << CPR_LOG) - 1u);
  const uint32_t r0 = tid >> CPR_LOG;
  const uint32_t s0 = swz_((r0 << CE) | (j0 * VPW));
  const uint64_t g0 = roff(r0) + (uint64_t)j0 * VPW;
  const long long total = (long long)p.E << TLOG;

  // Launch entries change every 2^TLOG tiles: the entry record, its row's status
  // and scale are cached per entry (separately for the prefetch, which runs one
  // tile ahead), so a tile costs no dependent global loads before its cp.async.
  int le = -1, ce = -1;          // cached entry index: load side / compute side
  const V* lsrc = nullptr;       // load side: source state of entry le (nullptr: skip)
  int4 cen = make_int4(0, 0, 0, 0);
  bool cdead = false;
  double cscale_v = 1.0;
  auto load_tile = [&](long long tt, V* dst) {
    const int e = (int)(tt >> TLOG);
    if (e != le) {
      le = e;
      const int4 en = p.ent[e];
      lsrc = (p.gen_zero || p.status[en.x] != 0) ? nullptr
                                                  : reinterpret_cast<const V*>(p.states) + ((size_t)en.y << p.n);
    }
    if (!lsrc) return;
    const V* src = lsrc + tile_base((uint64_t)(tt & ((1ll << TLOG) - 1)));
    if (FAST) {
#pragma unroll
      for (int k = 0; k < ITER; ++k)
        cp_async16(dst + (s0 ^ swz_((uint32_t)(k * RSTEP) << CE)), src + g0 + roff((uint32_t)(k * RSTEP)));
    } else {
      for (uint32_t u = tid; u < NVEC; u += NT) {
        const uint32_t r = u >> CPR_LOG, j = u & ((1u << CPR_LOG) - 1u);
        cp_async16(dst + swz_((r << CE) | (j * VPW)), src + roff(r) + (uint64_t)j * VPW);
      }
    }
  };

  // TMA path: every warp issues an equal share of the tile's gather4s (NGRP / warps, one per
  // issuing lane, each arming the buffer's transaction barrier with its own 512 B), from a
  // per-CTA table of tile-relative row coordinates (the same for every tile of the pass)
  constexpr int NWARP = NT / 32;
  constexpr int PERW = TMA ? (NGRP + NWARP - 1) / NWARP : 1;   // gather4s per warp
  // TMA_LANES == 0: each warp issues its PERW gather4s as one warp-uniform sequence (one
  // mbarrier arrival per issuing warp); otherwise one gather4 per issuing lane
  constexpr bool WISSUE = TMA_LANES == 0;
  constexpr int NIW = TMA ? (NGRP + PERW - 1) / PERW : 1;   // issuing warps
  constexpr int NISSUE = !TMA ? 1 : WISSUE ? NIW : (NGRP < NWARP * PERW ? NGRP : NWARP * PERW);
  static_assert(WISSUE || PERW <= 32, "TMA: more gather groups per warp than lanes");
  const uint32_t lane = tid & 31u;
  const int wid = __shfl_sync(0xffffffffu, (int)(tid >> 5), 0);   // warp-uniform
  const int gi = wid * PERW + (int)lane;            // this thread's gather group (per-lane issue)
  const bool issuer = TMA && (WISSUE ? wid * PERW < NGRP : (lane < (uint32_t)PERW && gi < NGRP));
  auto tma_load = [&](long long tt, int k) {
    V* dst = buf0 + (size_t)k * TL;   // buffer k (two stages: buf1 = buf0 + TL; teams: three buffers)
    const int e = (int)(tt >> TLOG);
    if (e != le) {
      le = e;
      const int4 en = p.ent[e];
      lsrc = (p.gen_zero || p.status[en.x] != 0) ? nullptr
                                                  : reinterpret_cast<const V*>(p.states) + ((size_t)en.y << p.n);
    }
    if (!issuer) return;
    if (TMA_ST) bulk_wait_read0();
    if constexpr (WISSUE) {
      if (!lsrc) {
        mbar_arrive_w(&mbar[k]);
        return;
      }
      const int g0 = wid * PERW;
      const int cnt = NGRP - g0 < PERW ? NGRP - g0 : PERW;
      mbar_arrive_tx_w(&mbar[k], 512u * (uint32_t)cnt);   // cnt x 4 rows x 128 B
      const unsigned long long row0 = __shfl_sync(0xffffffffu, (unsigned long long)(
          ((uint64_t)(lsrc - reinterpret_cast<const V*>(p.states)) +
           tile_base((uint64_t)(tt & ((1ll << TLOG) - 1)))) >> LOGU), 0);
#pragma unroll 1
      for (int j = 0; j < PERW; ++j) {
        if (NIW * PERW != NGRP && j >= cnt) break;
        const uint4 r = rowtab_c(g0 + j);
        tma_gather4_w(dst + ((size_t)(g0 + j) << (LOGU + 2)), tm, (int)(row0 + r.x), (int)(row0 + r.y),
                      (int)(row0 + r.z), (int)(row0 + r.w), &mbar[k]);
      }
      return;
    }
    if (!lsrc) {
      mbar_arrive(&mbar[k]);
      return;
    }
    mbar_arrive_tx(&mbar[k], 512u);   // 4 rows x 128 B
    const uint64_t row0 = ((uint64_t)(lsrc - reinterpret_cast<const V*>(p.states)) +
                           tile_base((uint64_t)(tt & ((1ll << TLOG) - 1)))) >> LOGU;
    const uint4 r = rowtab[gi];
    tma_gather4(dst + ((size_t)gi << (LOGU + 2)), tm, (int)(row0 + r.x), (int)(row0 + r.y), (int)(row0 + r.z),
                (int)(row0 + r.w), &mbar[k]);
  };
  // single buffer: the tile after this one is prefetched into L2 while this one computes, so
  // its gather (issued once this tile is stored) is served from L2 instead of HBM latency
  auto tma_prefetch = [&](long long tt) {
    if (!issuer) return;
    const int4 en = p.ent[(int)(tt >> TLOG)];
    if (p.gen_zero || p.status[en.x] != 0) return;
    const uint64_t row0 = (((uint64_t)en.y << p.n) + tile_base((uint64_t)(tt & ((1ll << TLOG) - 1)))) >> LOGU;
    if constexpr (WISSUE) {
      const unsigned long long r0u = __shfl_sync(0xffffffffu, (unsigned long long)row0, 0);
#pragma unroll
      for (int j = 0; j < PERW; ++j) {
        if (NIW * PERW != NGRP && wid * PERW + j >= NGRP) break;
        const uint4 r = rowtab_c(wid * PERW + j);
        tma_prefetch4_w(tm, (int)(r0u + r.x), (int)(r0u + r.y), (int)(r0u + r.z), (int)(r0u + r.w));
      }
      return;
    }
    const uint4 r = rowtab[gi];
    tma_prefetch4(tm, (int)(row0 + r.x), (int)(row0 + r.y), (int)(row0 + r.z), (int)(row0 + r.w));
  };
  auto tma_store = [&](const V* src, long long slot_base_amp, uint64_t base) {
    if (!issuer) return;
    if constexpr (WISSUE) {
      const int g0 = wid * PERW;
      const unsigned long long row0 =
          __shfl_sync(0xffffffffu, (unsigned long long)(((uint64_t)slot_base_amp + base) >> LOGU), 0);
#pragma unroll 1
      for (int j = 0; j < PERW; ++j) {
        if (NIW * PERW != NGRP && g0 + j >= NGRP) break;
        const uint4 r = rowtab_c(g0 + j);
        tma_scatter4_w(tm, (int)(row0 + r.x), (int)(row0 + r.y), (int)(row0 + r.z), (int)(row0 + r.w),
                       src + ((size_t)(g0 + j) << (LOGU + 2)));
      }
      bulk_commit();
      return;
    }
    const uint64_t row0 = ((uint64_t)slot_base_amp + base) >> LOGU;
    const uint4 r = rowtab[gi];
    tma_scatter4(tm, (int)(row0 + r.x), (int)(row0 + r.y), (int)(row0 + r.z), (int)(row0 + r.w),
                 src + ((size_t)gi << (LOGU + 2)));
    bulk_commit();
  };

  // One tile: entry bookkeeping, the pass's phases, store (+ fused sampler sums).  Only the
  // calling team takes part (gsync: the whole CTA when TEAMS == 1).
  auto process = [&](long long t, V* cur) {
    if ((int)(t >> TLOG) != ce) {
      ce = (int)(t >> TLOG);
      cen = p.ent[ce];
      cdead = p.status[cen.x] != 0;
      cscale_v = (p.use_scale && !p.gen_zero && !cdead) ? rsqrt(p.nst[cen.x]) : 1.0;
    }
    const int4 en = cen;
    const int b = en.x;                          // trajectory row
    const long long tile = t & ((1ll << TLOG) - 1);
    if (cdead) return;
    if (b != lb) {   // per trajectory, once: which phases see a non-default outcome
      if (tid == 0) *emask_s = err_mask(p.sel + (size_t)b * p.S, hits_s);
      gsync<NT>();
      lb = b;
    }
    const uint64_t emask = *emask_s;
    const uint64_t base = tile_base((uint64_t)tile);
    const double scale = cscale_v;
    // the phases address buf0 + (kofs | slot): tile-buffer offset kofs (a multiple of 2^L) ORed into
    // each phase's per-thread base, so every shared-memory access keeps a fixed base register
    // (opaque to the compiler: it would otherwise split the OR back into a per-access add)
    uint32_t kofs = (uint32_t)(cur - buf0);
    if (NBUF > 1) asm volatile("mov.b32 %0, %0;\n" : "+r"(kofs));
    body(buf0, kofs, b, p.sel + (size_t)b * p.S, tile, base, scale, red, emask, hits_s);
    V* st = reinterpret_cast<V*>(p.states) + ((size_t)en.z << p.n) + base;
    if (TMA && TMA_ST) {
      // the phases' shared-memory writes must be visible to the async proxy before the scatter
      fence_proxy_async();
      gsync<NT>();
      tma_store(cur, (long long)en.z << p.n, base);
      if (SUMS && FAST && p.tsum) {   // fused sampler block sums straight from the tile (see below)
        constexpr int PER_THREAD = ITER * VPW;
        constexpr int LANES = 512 / PER_THREAD;
        uint64_t q = 0;
#pragma unroll
        for (int k = 0; k < ITER; ++k) {
          const W w = *reinterpret_cast<const W*>(cur + (s0 ^ swz_((uint32_t)(k * RSTEP) << CE)));
          const V* pv = reinterpret_cast<const V*>(&w);
#pragma unroll
          for (int e = 0; e < VPW; ++e) q += qfix(pv[e]);
        }
#pragma unroll
        for (int o = LANES / 2; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if ((tid & (LANES - 1)) == 0 && en.x < p.B - 1)
          p.tsum[(size_t)en.x * p.tsum_stride + ((size_t)tile << (L - 9)) + tid / LANES] = q;
      }
    } else if (SUMS && FAST && p.tsum) {
      // Last pass of a unitary program: the sampler's block sums of q = qfix(a)
      // (2^-62 fixed point) are produced here, so sampling needs no separate read
      // of the states.  CDF order inside a tile is THREAD-major (thread, k, vector
      // element): a 512-amplitude block is the amplitudes of 32 (4-bit phases) or
      // 16 (5-bit phases) consecutive threads, so a block sum is one (half-)warp
      // reduction.  The sampler's Philox path maps element indices back through
      // this geometry (sample_kernels.cuh tiled_phys).
      constexpr int PER_THREAD = ITER * VPW;
      constexpr int LANES = 512 / PER_THREAD;        // 32 or 16 (engine checks)
      uint64_t q = 0;
#pragma unroll
      for (int k = 0; k < ITER; ++k) {
        const W w = *reinterpret_cast<const W*>(cur + (s0 ^ swz_((uint32_t)(k * RSTEP) << CE)));
        st_stream(reinterpret_cast<W*>(st + g0 + roff((uint32_t)(k * RSTEP))), w);
        const V* pv = reinterpret_cast<const V*>(&w);
#pragma unroll
        for (int e = 0; e < VPW; ++e) q += qfix(pv[e]);
      }
#pragma unroll
      for (int o = LANES / 2; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if ((tid & (LANES - 1)) == 0 && en.x < p.B - 1)
        p.tsum[(size_t)en.x * p.tsum_stride + ((size_t)tile << (L - 9)) + tid / LANES] = q;
    } else if (FAST) {
#pragma unroll
      for (int k = 0; k < ITER; ++k) {
        const W w = *reinterpret_cast<const W*>(cur + (s0 ^ swz_((uint32_t)(k * RSTEP) << CE)));
        st_stream(reinterpret_cast<W*>(st + g0 + roff((uint32_t)(k * RSTEP))), w);
      }
    } else {
      for (uint32_t u = tid; u < NVEC; u += NT) {
        const uint32_t r = u >> CPR_LOG, j = u & ((1u << CPR_LOG) - 1u);
        const W w = *reinterpret_cast<const W*>(cur + swz_((r << CE) | (j * VPW)));
        st_stream(reinterpret_cast<W*>(st + roff(r) + (uint64_t)j * VPW), w);
      }
    }
    // Compute teams, TMA stores, no fused sums: no team barrier after the store.  Every thread
    // passed the pre-store barrier (done with the tile's phases, hit words and reductions); the
    // buffer is next written only by the gathers of tile i + 3, which each issuing warp issues
    // into the slot groups its own scatters read, after waiting for those reads.
    if (!(TEAMS > 1 && TMA && TMA_ST && !PTG_TEAM_TAIL_SYNC && !(SUMS && FAST && p.tsum))) gsync<NT>();
  };
  auto fill_rowtab = [&]() {   // tile row in shared-memory slot 4g+q: slot^-1, then its row offset
    for (int g = (int)threadIdx.x; g < NGRP; g += NT * TEAMS) {
      uint32_t q4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t u = slot_inv((uint32_t)(4 * g + q));
        q4[q] = (uint32_t)((((uint64_t)(u & ((1u << (C - LOGU)) - 1u)) << LOGU) | row_off(u >> (C - LOGU))) >> LOGU);
      }
      rowtab[g] = make_uint4(q4[0], q4[1], q4[2], q4[3]);
    }
  };

  if constexpr (TEAMS > 1) {
    // Two compute teams share three tile buffers (single-buffered 64-KB tiles, one CTA of
    // 2 x NT threads per SM).  The CTA's i-th tile (t = blockIdx + i * grid) lives in buffer
    // i % 3 and is computed by team i % 2; when a team has stored tile i it loads tile i + 3
    // -- the other team's -- into the freed buffer.  A team therefore finds its next tile
    // already in flight while it computes, instead of exposing the whole load latency as a
    // single-buffered CTA does (ncu, 12-qubit c128 tiles at 2 CTAs/SM: long-scoreboard
    // stalls on the tile barrier 31 % of the warp cycles).
    static_assert(TMA && TMA_ST && STAGES == 1, "compute teams need TMA single-buffered tiles");
    // An mbarrier wait by parity only tells the current phase from the previous one, so a
    // team must not wait for tile i before the load of tile i was issued (the buffer's
    // previous phase -- tile i - 3, the other team's -- may still be open, e.g. when this
    // team raced through dead tiles): the issuing team's thread 0 stamps the buffer with i
    // once it has consumed tile i - 3, and the waiter first spins on the stamp.
    fill_rowtab();
    if (threadIdx.x == 0) {
      for (int k = 0; k < 3; ++k) {
        mbar_init(&mbar[k], NISSUE);
        stamp[k] = k;
      }
    }
    __syncthreads();
    const long long t0 = blockIdx.x, step = gridDim.x;
    if (team == 0) {
      if (t0 < total) tma_load(t0, 0);
      if (t0 + 2 * step < total) tma_load(t0 + 2 * step, 2);
    } else if (t0 + step < total) {
      tma_load(t0 + step, 1);
    }
    for (long long i = team;; i += 2) {
      const long long t = t0 + i * step;
      if (t >= total) break;
      const int k = (int)(i % 3);
      V* cur = buf0 + (size_t)k * TL;
      while (stamp[k] != (int)i) __nanosleep(64);
      mbar_wait(&mbar[k], (uint32_t)(i / 3) & 1u);
      process(t, cur);
      if (t + 3 * step < total) {
        if (tid == 0) stamp[k] = (int)(i + 3);   // this team has consumed tile i (its phase is complete)
        tma_load(t + 3 * step, k);   // issuers: after their scatters have read the buffer
      }
    }
    if (issuer) bulk_wait0();   // the last scatters must be done with shared memory before the CTA exits
    return;
  }

  long long t = blockIdx.x;
  if (TMA && STAGES == 1) {   // single buffer: loads issued at the top of each iteration
    fill_rowtab();
    if (tid == 0) mbar_init(&mbar[0], NISSUE);
    __syncthreads();
  } else if (TMA) {   // STAGES buffers: the next STAGES - 1 tiles are in flight while one computes
    fill_rowtab();
    if (tid == 0)
      for (int k = 0; k < STAGES; ++k) mbar_init(&mbar[k], NISSUE);
    __syncthreads();
    for (int k = 0; k < STAGES - 1; ++k)
      if (t + (long long)k * gridDim.x < total) tma_load(t + (long long)k * gridDim.x, k);
  } else if (STAGES == 2) {
    if (t < total) load_tile(t, buf0);
    cp_async_commit();
  }
  for (int it = 0; t < total; t += gridDim.x, ++it) {
    V* cur = (TMA && STAGES > 2) ? buf0 + (size_t)(it % STAGES) * TL : (it & 1) ? buf1 : buf0;
    V* nxt = (it & 1) ? buf0 : buf1;
    if (STAGES == 1) {
      if (TMA) {
        tma_load(t, 0);
        mbar_wait(&mbar[0], (uint32_t)it & 1u);
        if (TMA_PF && t + gridDim.x < total) tma_prefetch(t + gridDim.x);
      } else {
        load_tile(t, buf0);
        cp_async_commit();
        cp_async_wait0();
        __syncthreads();
      }
    } else if (TMA) {
      // (the buffer of tile it + STAGES - 1 last held tile it - 1, stored in the previous
      // iteration: tma_load's issuers wait for that store's reads first)
      const long long ahead = t + (long long)(STAGES - 1) * gridDim.x;
      if (ahead < total) tma_load(ahead, (it + STAGES - 1) % STAGES);
      mbar_wait(&mbar[it % STAGES], (uint32_t)(it / STAGES) & 1u);
    } else {
      if (t + gridDim.x < total) load_tile(t + gridDim.x, nxt);
      cp_async_commit();
      cp_async_wait1();
      __syncthreads();
    }
    process(t, cur);
  }
  if (TMA && TMA_ST) {
    if (issuer) bulk_wait0();   // the last scatters must be done with shared memory before the CTA exits
  } else {
    cp_async_wait0();
  }
}

}  // namespace ptg
