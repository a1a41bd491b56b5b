// exact_cdf.cuh -- the reference sampler's CDF reproduced bit for bit (verification mode).
//
// sample_shots (reference statevector.py:155-162) computes, in float64,
//   p_j   = np.abs(a_j) ** 2        numpy's SIMD complex abs: larger * sqrt(fma(r, r, 1)),
//                                    r = smaller / larger, then one rounded square
//   cum_j = np.cumsum(p)            SEQUENTIAL: cum_j = fl(cum_{j-1} + p_j)
//   cdf_j = fl(cum_j / cum_last)    (cum /= cum[-1])
//   idx   = #{j : cdf_j <= u}       (searchsorted side="right", then clip)
// At 28 qubits the sequential sum drifts ~1e-13 from the exact sum, so an exact
// (fixed-point) CDF picks a neighbouring index for ~1 shot in 10^4.  This file
// reproduces the sequential float64 sum exactly, in parallel:
//
// While the running sum s stays in one binade [2^e, 2^(e+1)) it is a multiple of
// u = 2^(e-52), so fl(s + p) = s + round_u(p): the step adds the INTEGER
// round(p / u) units -- independent of s, except at an exact tie (p / u = k + 1/2)
// where round-half-even looks at the parity of s / u.  Per 512-amplitude sample
// block (binade guessed from the exact fixed-point prefix) the steps compose into
// a map {parity in -> (units added, parity out)}; one warp per trajectory then
// chains the blocks, taking the map when the block provably stays inside the
// binade and summing the block sequentially otherwise (binade crossings, the first
// blocks).  The result is the block-end values C_b = cum_{512(b+1)-1} exactly as
// numpy computes them; the resolve step binary-searches C_b / T and re-walks the
// one hit block sequentially.  Exact integer/IEEE steps only: __ddiv_rn,
// __dsqrt_rn, __fma_rn, __dmul_rn, __dadd_rn.
#pragma once
#include "common.cuh"
#include "sample_kernels.cuh"

namespace ptsbe {

// numpy's np.abs(complex128) ** 2 (loops_arithm_fp: simd_cabsolute), finite inputs.
__device__ __forceinline__ double np_abs2(double re, double im) {
  const double a = fabs(re), b = fabs(im);
  const double larger = fmax(a, b), smaller = fmin(a, b);
  const double ratio = larger == 0.0 ? 0.0 : __ddiv_rn(smaller, larger);
  const double h = __dmul_rn(__dsqrt_rn(__fma_rn(ratio, ratio, 1.0)), larger);
  return __dmul_rn(h, h);
}
__device__ __forceinline__ double np_abs2(float2 a) { return np_abs2((double)a.x, (double)a.y); }
__device__ __forceinline__ double np_abs2(double2 a) { return np_abs2(a.x, a.y); }

struct BlockMap {
  uint64_t inc[2];   // units of u = 2^(e-52) added, for input parity 0 / 1
  int32_t e;         // binade exponent the map is valid for
  uint8_t out[2];    // parity of s / u after the block
  uint8_t valid;
  uint8_t pad;
};

struct ParMap {
  uint64_t inc0, inc1;
  uint32_t out0, out1;
};

__device__ __forceinline__ ParMap parmap_then(const ParMap& a, const ParMap& b) {
  ParMap r;
  r.inc0 = a.inc0 + (a.out0 ? b.inc1 : b.inc0);
  r.inc1 = a.inc1 + (a.out1 ? b.inc1 : b.inc0);
  r.out0 = a.out0 ? b.out1 : b.out0;
  r.out1 = a.out1 ? b.out1 : b.out0;
  return r;
}

// One warp per sample block: the block's parity map for the binade of its start
// value, guessed from the exact 2^-62 fixed-point prefix E (sample_blockscan).
template <typename R>
__global__ void __launch_bounds__(256) exact_blockmaps(SampleParams p, BlockMap* maps) {
  using V = typename Cplx<R>::V;
  const int b = blockIdx.y;
  if (p.status[b] != 0) return;
  const long long blk = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (blk >= p.nblk) return;
  const int lane = threadIdx.x & 31;
  const uint64_t* E = p.bs + (size_t)b * p.nblk;
  BlockMap* out = maps + (size_t)b * p.nblk + blk;
  const double s0 = blk ? (double)E[blk - 1] * 0x1p-62 : 0.0;
  const double s1 = (double)E[blk] * 0x1p-62;
  int e = 0;
  bool ok = s0 > 0.0;
  if (ok) {
    e = ilogb(s0);
    // clear of both binade edges (the fixed-point prefix is within ~1e-12 of numpy's)
    ok = s0 >= ldexp(1.0, e) * (1.0 + 1e-9) && s1 < ldexp(1.0, e + 1) * (1.0 - 1e-9);
  }
  if (!ok) {
    if (lane == 0) out->valid = 0;
    return;
  }
  const uint32_t bsz = 1u << p.sbits;
  const int per = bsz >= 32 ? (int)(bsz >> 5) : 1;
  const V* src = reinterpret_cast<const V*>(p.states) + ((size_t)b << p.n) + (size_t)blk * bsz;
  ParMap m{0, 0, 0, 1};   // identity
  bool big = false;
  for (int k = 0; k < per; ++k) {
    const uint32_t j = (uint32_t)lane * per + k;
    if (j >= bsz) break;
    const double pj = np_abs2(src[j]);
    const double x = ldexp(pj, 52 - e);          // p / u, exact
    if (!(x < 0x1p53)) { big = true; break; }
    const double f = floor(x);
    const double fr = x - f;                      // exact
    const uint64_t fi = (uint64_t)f;
    ParMap s;
    if (fr == 0.5) {                              // tie: round half to even of (K + f)
      s.inc0 = fi + (fi & 1);
      s.inc1 = fi + ((fi + 1) & 1);
      s.out0 = s.out1 = 0;
    } else {
      const uint64_t inc = fi + (fr > 0.5 ? 1 : 0);
      s.inc0 = s.inc1 = inc;
      s.out0 = (uint32_t)(inc & 1);
      s.out1 = (uint32_t)((inc + 1) & 1);
    }
    m = parmap_then(m, s);
  }
  const bool any_big = __any_sync(0xffffffffu, big);
  // compose the 32 lane maps in lane order (lane 0 first)
  ParMap acc = m;
  for (int l = 1; l < 32; ++l) {
    ParMap o;
    o.inc0 = shfl_u64(m.inc0, l);
    o.inc1 = shfl_u64(m.inc1, l);
    o.out0 = __shfl_sync(0xffffffffu, m.out0, l);
    o.out1 = __shfl_sync(0xffffffffu, m.out1, l);
    if (lane == 0) acc = parmap_then(acc, o);
  }
  if (lane == 0) {
    BlockMap r;
    r.inc[0] = acc.inc0;
    r.inc[1] = acc.inc1;
    r.out[0] = (uint8_t)acc.out0;
    r.out[1] = (uint8_t)acc.out1;
    r.e = e;
    r.valid = any_big ? 0 : 1;
    r.pad = 0;
    *out = r;
  }
}

// One warp per trajectory: chain the blocks in order -> C[b][blk] = numpy's cum at the
// block's last element (float64 bits in the u64 buffer), total[b] = cum_last.
// Blocks go 32 at a time: when all 32 maps are valid for the binade of the running sum
// and the group's end stays inside it, a warp scan of the maps gives every block end at
// once (one step per 32 blocks); otherwise the group is chained block by block.
template <typename R>
__global__ void __launch_bounds__(32) exact_chain(SampleParams p, const BlockMap* maps, uint64_t* C) {
  using V = typename Cplx<R>::V;
  __shared__ double pv[1 << 9];
  const int b = blockIdx.x;
  if (p.status[b] != 0) return;
  const int lane = threadIdx.x;
  const uint32_t bsz = 1u << p.sbits;
  const V* st = reinterpret_cast<const V*>(p.states) + ((size_t)b << p.n);
  const BlockMap* mp = maps + (size_t)b * p.nblk;
  uint64_t* Cb = C + (size_t)b * p.nblk;
  double s = 0.0;   // running sum (identical in every lane)
  for (long long g0 = 0; g0 < p.nblk; g0 += 32) {
    const long long blk = g0 + lane;
    const bool have = blk < p.nblk;
    BlockMap m{};
    if (have) m = mp[blk];
    // fast path: one warp scan for the whole group
    const int e0 = __shfl_sync(0xffffffffu, m.e, 0);
    const bool mine_ok = !have || (m.valid && m.e == e0);
    bool fast = __all_sync(0xffffffffu, mine_ok) && s > 0.0 && ilogb(s) == e0;
    if (fast) {
      ParMap pm;
      if (have) { pm.inc0 = m.inc[0]; pm.inc1 = m.inc[1]; pm.out0 = m.out[0]; pm.out1 = m.out[1]; }
      else { pm.inc0 = pm.inc1 = 0; pm.out0 = 0; pm.out1 = 1; }
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {   // inclusive scan: maps of lanes <= this one, in order
        ParMap o;
        o.inc0 = shfl_up_u64(pm.inc0, d);
        o.inc1 = shfl_up_u64(pm.inc1, d);
        o.out0 = __shfl_up_sync(0xffffffffu, pm.out0, d);
        o.out1 = __shfl_up_sync(0xffffffffu, pm.out1, d);
        if (lane >= d) pm = parmap_then(o, pm);
      }
      const uint64_t K = (uint64_t)ldexp(s, 52 - e0);
      const uint64_t Kj = K + ((K & 1) ? pm.inc1 : pm.inc0);
      const uint64_t Kend = shfl_u64(Kj, 31);
      fast = Kend < (1ull << 53);   // the group ends inside the binade
      if (fast) {
        if (have) Cb[blk] = (uint64_t)__double_as_longlong(ldexp((double)Kj, e0 - 52));
        s = ldexp((double)Kend, e0 - 52);
      }
    }
    if (fast) continue;
    // slow path: block by block, map when it provably applies, else sequential sums
    const int nb = (int)min((long long)32, p.nblk - g0);
    for (int j = 0; j < nb; ++j) {
      const int me = __shfl_sync(0xffffffffu, m.e, j);
      const int mv = __shfl_sync(0xffffffffu, (int)m.valid, j);
      const uint64_t i0 = shfl_u64(m.inc[0], j), i1 = shfl_u64(m.inc[1], j);
      int ok = 0;
      if (mv && s > 0.0 && ilogb(s) == me) {
        const uint64_t K = (uint64_t)ldexp(s, 52 - me);
        const uint64_t Kend = K + ((K & 1) ? i1 : i0);
        if (Kend < (1ull << 53)) {
          s = ldexp((double)Kend, me - 52);
          ok = 1;
        }
      }
      if (!ok) {   // the block crosses a binade (or the sum is still tiny)
        const V* src = st + (size_t)(g0 + j) * bsz;
        for (uint32_t t = lane; t < bsz; t += 32) pv[t] = np_abs2(src[t]);
        __syncwarp();
        double acc = s;
        if (lane == 0)
          for (uint32_t t = 0; t < bsz; ++t) acc = __dadd_rn(acc, pv[t]);
        s = __shfl_sync(0xffffffffu, acc, 0);
        __syncwarp();
      }
      if (lane == 0) Cb[g0 + j] = (uint64_t)__double_as_longlong(s);
    }
  }
  if (lane == 0) p.total[b] = (uint64_t)__double_as_longlong(s);
}

// Per shot (sorted keys, 32 per warp as sample_resolve): idx = #{j : fl(cum_j / T) <= u},
// u = K * 2^-53 -- binary search over the block ends, then the hit block re-walked
// sequentially from its exact start value.
template <typename R>
__global__ void __launch_bounds__(256) exact_resolve(SampleParams p, const uint64_t* chunks, long long n_chunks,
                                                      const uint64_t* keys, const uint64_t* C, uint64_t* idx_out) {
  using V = typename Cplx<R>::V;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_chunks) return;
  const int lane = threadIdx.x & 31;
  const uint64_t ch = chunks[w];
  const int b = (int)(ch >> 40);
  const long long i = (long long)(ch & 0xFFFFFFFFFFull) + lane;
  if (p.status[b] != 0 || i >= p.m[b]) return;
  const double u = (double)keys[p.off[b] + i] * 0x1p-53;
  const uint64_t* Cb = C + (size_t)b * p.nblk;
  const double T = __longlong_as_double((long long)p.total[b]);
  long long lo = 0, hi = p.nblk - 1;    // first block whose end has cdf > u (the last one does)
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (__ddiv_rn(__longlong_as_double((long long)Cb[mid]), T) > u) hi = mid; else lo = mid + 1;
  }
  const uint32_t bsz = 1u << p.sbits;
  const V* src = reinterpret_cast<const V*>(p.states) + ((size_t)b << p.n) + (size_t)lo * bsz;
  double s = lo ? __longlong_as_double((long long)Cb[lo - 1]) : 0.0;
  uint64_t idx = (uint64_t)lo * bsz + bsz - 1;
  for (uint32_t j = 0; j < bsz; ++j) {
    s = __dadd_rn(s, np_abs2(src[j]));
    if (__ddiv_rn(s, T) > u) { idx = (uint64_t)lo * bsz + j; break; }
  }
  const uint64_t last = (1ull << p.n) - 1;
  idx_out[p.off[b] + i] = idx < last ? idx : last;
}

}  // namespace ptsbe
