// common.cuh -- small device helpers shared by the PTSBE kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ptsbe {

// Complex amplitude types: interleaved (re, im), 8 B (c64) or 16 B (c128).
template <typename R> struct Cplx;
template <> struct Cplx<float>  { using V = float2;  using W = float4;  };   // W: one 16-B vector
template <> struct Cplx<double> { using V = double2; using W = double2; };

template <typename V> __device__ __forceinline__ V make_vec2(double x, double y);
template <> __device__ __forceinline__ float2 make_vec2<float2>(double x, double y) { return make_float2((float)x, (float)y); }
template <> __device__ __forceinline__ double2 make_vec2<double2>(double x, double y) { return make_double2(x, y); }

template <typename V>
__device__ __forceinline__ V cmadd2(V m0, V a, V m1, V b) {
  // m0*a + m1*b
  V r;
  r.x = m0.x * a.x - m0.y * a.y + m1.x * b.x - m1.y * b.y;
  r.y = m0.x * a.y + m0.y * a.x + m1.x * b.y + m1.y * b.x;
  return r;
}

template <typename V>
__device__ __forceinline__ V cmadd4(const V* m, V a, V b, V c, V d) {
  V r;
  r.x = m[0].x * a.x - m[0].y * a.y + m[1].x * b.x - m[1].y * b.y +
        m[2].x * c.x - m[2].y * c.y + m[3].x * d.x - m[3].y * d.y;
  r.y = m[0].x * a.y + m[0].y * a.x + m[1].x * b.y + m[1].y * b.x +
        m[2].x * c.y + m[2].y * c.x + m[3].x * d.y + m[3].y * d.x;
  return r;
}

// Scatter the low bits of `src` onto the set bits of `mask` (software PDEP).
__device__ __forceinline__ uint64_t pdep64(uint64_t src, uint64_t mask) {
  uint64_t out = 0;
  while (mask) {
    const uint64_t low = mask & (~mask + 1);
    if (src & 1) out |= low;
    src >>= 1;
    mask ^= low;
  }
  return out;
}

// Insert a zero bit at position `bit` of p.
__device__ __forceinline__ uint32_t insert0(uint32_t p, int bit) {
  const uint32_t lo = p & ((1u << bit) - 1u);
  return ((p ^ lo) << 1) | lo;
}

// |a|^2 in float64 without FMA contraction (identical rounding in every kernel).
__device__ __forceinline__ double prob64(float2 a) {
  const double x = a.x, y = a.y;
  return __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
}
__device__ __forceinline__ double prob64(double2 a) {
  return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
}

// Deterministic CTA-wide fp64 sum; result valid in thread 0.  `red` >= 32 doubles.
__device__ __forceinline__ double block_sum_f64(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) r += red[i];
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
  const uint32_t lo = __shfl_up_sync(0xffffffffu, (uint32_t)v, d);
  const uint32_t hi = __shfl_up_sync(0xffffffffu, (uint32_t)(v >> 32), d);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

// Inclusive warp scan of u64 (integer: order-independent, exact).
__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = shfl_up_u64(v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// Streaming 16-B global load/store (data touched once per pass).
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

// Probability -> unsigned fixed point with 2^-62 resolution.  Integer sums are
// associative, so every scan order yields the same CDF bit for bit.
constexpr double kFixScale = 4611686018427387904.0;  // 2^62
__device__ __forceinline__ uint64_t to_fixed(double p) {
  return (uint64_t)__double2ull_rn(p * kFixScale);
}

}  // namespace ptsbe
