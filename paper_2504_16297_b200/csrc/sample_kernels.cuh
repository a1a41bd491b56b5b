// sample_kernels.cuh -- bulk shot sampling for a batch of prepared states.
//
// Replaces sample_shots (reference statevector.py:148-163: |a|^2, sequential
// fp64 cumsum, /cum[-1], searchsorted(side="right"), np.unique counts).
//
// The CDF is built in 2^-62 fixed point: q_j = rn(|a_j|^2 / N * 2^62) as u64.
// Integer prefix sums are associative, so the two-level (block, element) CDF
// used here is exactly monotone and identical under any scan order, and the
// reference's decision "idx = #{j : cum_j / cum_last <= u}" becomes the exact
// integer test cum_j <= floor(K * T / 2^53) for u = K * 2^-53.
//
// Pipeline per batch (one launch each, all trajectories at once):
//   blocksum  : q-sums of 2^sbits-amplitude sample blocks (one full state read)
//   blockscan : per-trajectory inclusive scan of block sums -> E[], T = E[last]
//   keys      : 53-bit uniform keys per shot -- PCG64 (bit-exact numpy stream),
//               Philox sorted-by-construction (exponential spacings), or host keys
//   sort      : per-trajectory LSD radix sort of keys (PCG64 / host keys only)
//   resolve   : per 32 sorted shots: binary search of E, then ONE re-read of each
//               hit block shared by all shots that land in it
//   rle       : sorted indices -> (index, count) runs  == ShotBatch.from_indices
#pragma once
#include "common.cuh"
#include "rng.cuh"

namespace ptsbe {

struct SampleParams {
  const void* states;
  int n;
  int sbits;               // sample-block bits
  long long nblk;          // blocks per state
  int B;
  const double* nst;       // [B] norm^2 of stored state
  const int32_t* status;   // [B]
  uint64_t* bs;            // [B][nblk] block sums -> inclusive scan
  uint64_t* total;         // [B]
  const int64_t* off;      // [B] shot offsets
  const int64_t* m;        // [B] shots
  // tile-order CDF (block sums written by the last generated pass): element e =
  // (tile, row, column) of that pass's geometry; 0 = plain index order
  int tiled;
  uint64_t tq;             // the pass's tile qubit mask
  int tL, tC;              // its tile bits and contiguous low bits
  int tT;                  // its threads per CTA (thread-major element order)
};

// Fixed-point probability of the fused (tile-order) block sums: must equal
// gen_prelude.cuh qfix bit for bit.
__device__ __forceinline__ uint64_t qfix(float2 a) {
  return __float2ull_rn(__fmul_rn(__fmaf_rn(a.x, a.x, __fmul_rn(a.y, a.y)), 0x1p62f));
}
__device__ __forceinline__ uint64_t qfix(double2 a) {
  return __double2ull_rn(__dmul_rn(__fma_rn(a.x, a.x, __dmul_rn(a.y, a.y)), 0x1p62));
}
// Physical basis index of tile-order element e.  Inside a tile the order is
// thread-major, as the last pass's store loop walks it (gen_prelude.cuh run_pass):
// thread t holds 16-B vectors k = 0..ITER-1 at row (t >> CPR) + k * RSTEP, column
// (t & (2^CPR - 1)) * VPW, with VPW amplitudes per vector (c64: 2, c128: 1).
template <typename V>
__device__ __forceinline__ uint64_t tiled_phys(const SampleParams& p, uint64_t e) {
  constexpr int VPW = sizeof(V) == 8 ? 2 : 1;
  const int cpr = p.tC - (VPW == 2 ? 1 : 0);                 // log2 vectors per row
  const uint64_t nmask = p.n >= 64 ? ~0ull : ((1ull << p.n) - 1);
  const uint64_t lowm = (1ull << p.tC) - 1;
  const uint64_t tile = e >> p.tL, internal = e & ((1ull << p.tL) - 1);
  const uint64_t per_thread = (1ull << p.tL) / (uint64_t)p.tT;   // ITER * VPW
  const uint64_t t = internal / per_thread, r = internal % per_thread;
  const uint64_t k = r / VPW, ev = r % VPW;
  const uint64_t rstep = (uint64_t)p.tT >> cpr;
  const uint64_t row = (t >> cpr) + k * rstep;
  const uint64_t col = (t & ((1ull << cpr) - 1)) * VPW + ev;
  return pdep64(tile, ~p.tq & nmask) | pdep64(row, p.tq & ~lowm) | col;
}

// ---- blocksum: one warp per sample block, coalesced 16-B loads
template <typename R>
__global__ void __launch_bounds__(256) sample_blocksum(SampleParams p) {
  using V = typename Cplx<R>::V;
  const int b = blockIdx.y;
  if (p.status[b] != 0) return;
  const long long blk = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (blk >= p.nblk) return;
  const int lane = threadIdx.x & 31;
  const uint32_t bsz = 1u << p.sbits;
  const V* src = reinterpret_cast<const V*>(p.states) + ((size_t)b << p.n) + (size_t)blk * bsz;
  const double mul = kFixScale / p.nst[b];
  uint64_t acc = 0;
  for (uint32_t i = lane; i < bsz; i += 32) {
    const V a = __ldcs(src + i);
    acc += (uint64_t)__double2ull_rn(prob64(a) * mul);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += shfl_xor_u64(acc, o);
  if (lane == 0) p.bs[(size_t)b * p.nblk + blk] = acc;
}

// ---- blockscan: one CTA (1024 threads) per trajectory, in place
__global__ void __launch_bounds__(1024) sample_blockscan(SampleParams p) {
  __shared__ uint64_t wsum[32];
  __shared__ uint64_t carry_s;
  const int b = blockIdx.x;
  if (p.status[b] != 0) return;
  uint64_t* a = p.bs + (size_t)b * p.nblk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int PER = 4;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (long long base = 0; base < p.nblk; base += 1024 * PER) {
    uint64_t v[PER];
    uint64_t s = 0;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const long long i = base + (long long)threadIdx.x * PER + e;
      v[e] = (i < p.nblk) ? a[i] : 0;
      s += v[e];
      v[e] = s;                      // thread-local inclusive
    }
    const uint64_t incl = warp_incl_scan_u64(s);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = wsum[lane];
      w = warp_incl_scan_u64(w);
      wsum[lane] = w;               // inclusive over warps
    }
    __syncthreads();
    const uint64_t before = carry_s + (warp ? wsum[warp - 1] : 0) + (incl - s);
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const long long i = base + (long long)threadIdx.x * PER + e;
      if (i < p.nblk) a[i] = before + v[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry_s += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) p.total[b] = carry_s;
}

// ---- keys, PCG64 mode: thread per shot, O(log i) jump-ahead to draw i
__global__ void __launch_bounds__(256) keys_pcg64(const uint64_t* chunks, long long n_chunks,
                                                   const uint64_t* rng_state, const int64_t* off,
                                                   const int64_t* m, const int32_t* status,
                                                   uint64_t* keys) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_chunks) return;
  const uint64_t ch = chunks[w];
  const int b = (int)(ch >> 40);
  const long long i = (long long)(ch & 0xFFFFFFFFFFull) + (threadIdx.x & 31);
  if (i >= m[b] || status[b] != 0) return;
  const u128 st = ((u128)rng_state[4 * b] << 64) | rng_state[4 * b + 1];
  const u128 inc = ((u128)rng_state[4 * b + 2] << 64) | rng_state[4 * b + 3];
  const u128 before = pcg_advance(st, inc, (uint64_t)i);
  keys[off[b] + i] = pcg_key53(before, inc);
}

// ---- keys, Philox mode: sorted uniforms u_k = S_k / S_{m+1}, S = prefix of Exp(1)
__global__ void __launch_bounds__(1024) keys_philox_sorted(const uint64_t* seeds, const int64_t* off,
                                                            const int64_t* m, const int32_t* status,
                                                            uint64_t* keys) {
  __shared__ double wsum[32];
  __shared__ double carry_s;
  const int b = blockIdx.x;
  const long long mb = m[b];
  if (status[b] != 0 || mb == 0) return;
  const uint32_t k0 = (uint32_t)seeds[b], k1 = (uint32_t)(seeds[b] >> 32);
  double* S = reinterpret_cast<double*>(keys + off[b]);   // prefix sums staged in place
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0.0;
  __syncthreads();
  // draws 0..m-1 give S_1..S_m; draw m is the extra spacing for the normaliser
  for (long long base = 0; base <= mb; base += 1024) {
    const long long i = base + threadIdx.x;
    double e = 0.0;
    if (i <= mb) {
      Philox4 c{(uint32_t)i, (uint32_t)(i >> 32), 0x53484f54u, 0u};
      const Philox4 r = philox4x32_10(c, k0, k1);
      const uint64_t bits = ((uint64_t)r.x << 21) ^ (uint64_t)(r.y >> 11);
      const double u = ((double)(bits & ((1ull << 53) - 1)) + 0.5) * 0x1p-53;
      e = -log(u);
    }
    double incl = e;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      double w = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += o;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const double val = carry_s + (warp ? wsum[warp - 1] : 0.0) + incl;
    if (i < mb) S[i] = val;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry_s + wsum[31];
    __syncthreads();
  }
  const double tot = carry_s;
  for (long long i = threadIdx.x; i < mb; i += blockDim.x) {
    const double u = S[i] / tot;
    uint64_t k = (uint64_t)(u * 0x1p53);
    if (k > (1ull << 53) - 1) k = (1ull << 53) - 1;
    keys[off[b] + i] = k;
  }
}

// ---- stable LSD radix sort of each trajectory's key segment (one CTA each)
__global__ void __launch_bounds__(1024) seg_radix_sort(uint64_t* keys, uint64_t* tmp, const int64_t* off,
                                                        const int64_t* m, const int32_t* status,
                                                        int key_bits) {
  __shared__ uint32_t base[256];
  __shared__ uint32_t tile_tot[256];
  __shared__ uint32_t wcnt[32][256];
  const int b = blockIdx.x;
  const long long n = m[b];
  if (status[b] != 0 || n <= 1) return;
  uint64_t* src = keys + off[b];
  uint64_t* dst = tmp + off[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) base[i] = 0;
    __syncthreads();
    for (long long i = threadIdx.x; i < n; i += blockDim.x)
      atomicAdd(&base[(src[i] >> shift) & 255u], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t acc = 0;
      for (int d = 0; d < 256; ++d) { const uint32_t c = base[d]; base[d] = acc; acc += c; }
    }
    __syncthreads();
    for (long long t0 = 0; t0 < n; t0 += blockDim.x) {
      for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) (&wcnt[0][0])[i] = 0;
      __syncthreads();
      const long long i = t0 + threadIdx.x;
      const bool valid = i < n;
      const uint64_t key = valid ? src[i] : 0;
      const int d = valid ? (int)((key >> shift) & 255u) : 256 + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t rank = __popc(peers & lt_mask);
      if (valid && rank == 0) wcnt[warp][d] = __popc(peers);
      __syncthreads();
      if (threadIdx.x < 256) {
        uint32_t acc = 0;
        for (int w = 0; w < nw; ++w) { const uint32_t c = wcnt[w][threadIdx.x]; wcnt[w][threadIdx.x] = acc; acc += c; }
        tile_tot[threadIdx.x] = acc;
      }
      __syncthreads();
      if (valid) dst[base[d] + wcnt[warp][d] + rank] = key;
      __syncthreads();
      if (threadIdx.x < 256) base[threadIdx.x] += tile_tot[threadIdx.x];
      __syncthreads();
    }
    uint64_t* t = src; src = dst; dst = t;
  }
  if (passes & 1) {
    uint64_t* out = keys + off[b];
    for (long long i = threadIdx.x; i < n; i += blockDim.x) out[i] = src[i];
  }
}

// ---- resolve: 32 sorted shots per warp -> basis indices
template <typename R>
__global__ void __launch_bounds__(256) sample_resolve(SampleParams p, const uint64_t* chunks, long long n_chunks,
                                                       const uint64_t* keys, uint64_t* idx_out) {
  using V = typename Cplx<R>::V;
  constexpr int EMAX = 16;
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n_chunks) return;
  const int lane = threadIdx.x & 31;
  const uint64_t ch = chunks[w];
  const int b = (int)(ch >> 40);
  const long long i = (long long)(ch & 0xFFFFFFFFFFull) + lane;
  if (p.status[b] != 0) return;
  const bool valid = i < p.m[b];
  const uint64_t* E = p.bs + (size_t)b * p.nblk;
  const uint64_t T = p.total[b];
  uint64_t target = 0;
  long long blk = -1;
  if (valid) {
    const uint64_t K = keys[p.off[b] + i];
    target = (uint64_t)(((u128)K * (u128)T) >> 53);
    long long lo = 0, hi = p.nblk - 1;     // first blk with E[blk] > target (exists: E[last]=T > target)
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (E[mid] > target) hi = mid; else lo = mid + 1;
    }
    blk = lo;
  }
  const uint32_t bsz = 1u << p.sbits;
  const int per = bsz >= 32 ? (int)(bsz >> 5) : 1;     // elements per lane (<= EMAX)
  const V* st = reinterpret_cast<const V*>(p.states) + ((size_t)b << p.n);
  const double mul = kFixScale / p.nst[b];
  uint32_t pending = __ballot_sync(0xffffffffu, valid);
  while (pending) {
    const int leader = __ffs(pending) - 1;
    const long long cur = __shfl_sync(0xffffffffu, blk, leader);
    const uint32_t members = __ballot_sync(0xffffffffu, valid && blk == cur);
    const uint64_t P = cur ? E[cur - 1] : 0;
    uint64_t q[EMAX];
    uint64_t lsum = 0;
    const long long e0 = (long long)cur * bsz + (long long)lane * per;
    // tiled: this lane's elements are one thread's vectors of the last pass, or an
    // aligned half of them (fused sums need a block == the amplitudes of a warp or a
    // half warp): element j = (k0 + k, ev) sits at base | PDEP(k * RSTEP onto the row
    // bits) | ev, k0 aligned so the bits are disjoint -- one full PDEP per lane
    constexpr int VPW_ = sizeof(V) == 8 ? 2 : 1;
    uint64_t tbase = 0, rowmask = 0;
    int lr = 0;
    if (p.tiled) {
      tbase = tiled_phys<V>(p, (uint64_t)e0);
      rowmask = p.tq & ~((1ull << p.tC) - 1);
      lr = 31 - __clz(p.tT >> (p.tC - (VPW_ == 2 ? 1 : 0)));
    }
#pragma unroll
    for (int j = 0; j < EMAX; ++j) {
      q[j] = 0;
      if (j < per && (uint32_t)(lane * per + j) < bsz) {
        if (p.tiled) {
          const uint64_t a = tbase | pdep64((uint64_t)(j / VPW_) << lr, rowmask) | (uint64_t)(j % VPW_);
          q[j] = qfix(st[a]);
        } else {
          q[j] = (uint64_t)__double2ull_rn(prob64(st[e0 + j]) * mul);
        }
      }
      lsum += q[j];
    }
    const uint64_t incl = warp_incl_scan_u64(lsum);
    const uint64_t lane_end = P + incl;
    uint32_t mem = members;
    while (mem) {
      const int s = __ffs(mem) - 1;
      mem &= mem - 1;
      const uint64_t tg = shfl_u64(target, s);
      const uint32_t over = __ballot_sync(0xffffffffu, lane_end > tg);
      const int ls = __ffs(over) - 1;
      if (lane == ls) {
        uint64_t c = P + incl - lsum;
        int jj = per - 1;
        bool found = false;
#pragma unroll
        for (int j = 0; j < EMAX; ++j) {
          c += q[j];
          if (!found && j < per && c > tg) { found = true; jj = j; }
        }
        const long long sh = (long long)(ch & 0xFFFFFFFFFFull) + s;
        idx_out[p.off[b] + sh] = p.tiled ? tiled_phys<V>(p, (uint64_t)(e0 + jj)) : (uint64_t)(e0 + jj);
      }
    }
    pending &= ~members;
  }
}

// ---- rle: sorted indices -> (index, count) runs, one CTA per trajectory.
// Writes runs at the trajectory's shot offset; nuniq[b] = number of runs.
__global__ void __launch_bounds__(1024) sample_rle(const uint64_t* idx, const int64_t* off, const int64_t* m,
                                                    const int32_t* status, uint64_t* run_idx, uint32_t* run_cnt,
                                                    int64_t* nuniq) {
  __shared__ uint32_t wsum[32];
  __shared__ long long carry_s;
  const int b = blockIdx.x;
  const long long n = m[b];
  if (status[b] != 0 || n == 0) { if (threadIdx.x == 0) nuniq[b] = 0; return; }
  const uint64_t* x = idx + off[b];
  uint64_t* ri = run_idx + off[b];
  uint32_t* rc = run_cnt + off[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  // pass 1: run starts -> (index, start position)
  for (long long t0 = 0; t0 < n; t0 += blockDim.x) {
    const long long i = t0 + threadIdx.x;
    const uint32_t f = (i < n && (i == 0 || x[i] != x[i - 1])) ? 1u : 0u;
    uint32_t incl = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t v = wsum[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
      }
      wsum[lane] = v;
    }
    __syncthreads();
    if (f) {
      const long long pos = carry_s + (warp ? wsum[warp - 1] : 0) + incl - 1;
      ri[pos] = x[i];
      rc[pos] = (uint32_t)i;      // start, converted to a count in pass 2
    }
    __syncthreads();
    if (threadIdx.x == 0) carry_s += wsum[31];
    __syncthreads();
  }
  const long long runs = carry_s;
  __syncthreads();
  // pass 2: count = next start - start (each run read/written by one thread)
  for (long long r0 = 0; r0 < runs; r0 += blockDim.x) {
    const long long r = r0 + threadIdx.x;
    uint32_t start = 0, next = 0;
    if (r < runs) { start = rc[r]; next = (r + 1 < runs) ? rc[r + 1] : (uint32_t)n; }
    __syncthreads();
    if (r < runs) rc[r] = next - start;
    __syncthreads();
  }
  if (threadIdx.x == 0) nuniq[b] = runs;
}

// Physical layout -> logical bitstrings.  The state may be stored with logical
// qubit q at physical bit perm[q] (planner.h layout search); shots come out of
// the CDF in physical order and are mapped back here, then re-sorted.
struct BitPerm {
  int8_t src[64];   // logical bit q <- physical bit src[q]
  int n;
};

__device__ __forceinline__ uint64_t permute_bits(uint64_t x, const BitPerm& P) {
  uint64_t out = 0;
  for (int q = 0; q < P.n; ++q) out |= ((x >> P.src[q]) & 1ull) << q;
  return out;
}

__global__ void unpermute_indices(uint64_t* idx, long long total, BitPerm P) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    idx[i] = permute_bits(idx[i], P);
}

// out[logical(i)] = in[i] for one state (parity download / upload of permuted layouts).
// The bit permutation is linear over disjoint bits: perm(i) = OR over the bytes of
// i of a per-byte table (built once per CTA in shared memory), 5 lookups instead
// of a loop over n bits per amplitude.
template <typename V>
__global__ void __launch_bounds__(256) permute_state(const V* in, V* out, int n, BitPerm P) {
  __shared__ uint64_t T[5][256];
  for (int e = threadIdx.x; e < 5 * 256; e += blockDim.x) {
    const int byte = e >> 8, v = e & 255;
    T[byte][v] = permute_bits((uint64_t)v << (8 * byte), P);
  }
  __syncthreads();
  const size_t N = 1ull << n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t j = T[0][i & 255] | T[1][(i >> 8) & 255] | T[2][(i >> 16) & 255] | T[3][(i >> 24) & 255] |
                       T[4][(i >> 32) & 255];
    out[j] = in[i];
  }
}

// The same bit permutation, tiled so that reads AND writes move whole 128-B rows: a CTA
// handles tiles of 2^K amplitudes spanning the input bits Qin (input bits 0..R-1 plus the
// input bits that feed output bits 0..R-1, padded with low bits), loads them row-contiguous
// into shared memory and writes them out row-contiguous in output order.  Element f of the
// output tile takes element e = sum_b bit_b(f) << fmap[b] of the input tile.
struct TilePerm {
  uint64_t qin, qout;   // tile bits on the input / output side
  int8_t fmap[16];      // output-tile bit b <- input-tile bit fmap[b]
  int k;                // tile bits
};

__device__ __forceinline__ uint64_t pdep_loop(uint64_t src, uint64_t mask) {
  uint64_t out = 0;
  while (mask) {
    const uint64_t low = mask & (~mask + 1);
    if (src & 1) out |= low;
    src >>= 1;
    mask ^= low;
  }
  return out;
}

template <typename V>
__global__ void __launch_bounds__(256) permute_tiled(const V* in, V* out, int n, BitPerm P, TilePerm T) {
  extern __shared__ __align__(16) unsigned char psm[];
  const uint32_t K = 1u << T.k;
  V* tile = reinterpret_cast<V*>(psm);
  uint64_t* offin = reinterpret_cast<uint64_t*>(tile + K);    // pdep(e, qin)
  uint64_t* offout = offin + K;                                 // pdep(f, qout)
  uint16_t* emap = reinterpret_cast<uint16_t*>(offout + K);    // input-tile element of output element f
  __shared__ uint64_t base_s[2];
  for (uint32_t e = threadIdx.x; e < K; e += blockDim.x) {       // per-CTA tables, once
    offin[e] = pdep_loop(e, T.qin);
    offout[e] = pdep_loop(e, T.qout);
    uint32_t m = 0;
    for (int b = 0; b < T.k; ++b) m |= ((e >> b) & 1u) << T.fmap[b];
    emap[e] = (uint16_t)m;
  }
  const uint64_t nmask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t outside = ~T.qin & nmask;
  const uint64_t ntiles = 1ull << (n - T.k);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (threadIdx.x == 0) {
      const uint64_t ib = pdep_loop(t, outside);
      base_s[0] = ib;
      base_s[1] = permute_bits(ib, P);
    }
    __syncthreads();
    const uint64_t ibase = base_s[0], jbase = base_s[1];
    for (uint32_t e = threadIdx.x; e < K; e += blockDim.x) tile[e] = in[ibase | offin[e]];
    __syncthreads();
    for (uint32_t f = threadIdx.x; f < K; f += blockDim.x) out[jbase | offout[f]] = tile[emap[f]];
    __syncthreads();
  }
}

// State sharding: the half of a shard whose local bit `bit` equals `value`,
// packed contiguously (index order) for a global<->local qubit swap.
template <typename V>
__global__ void pack_half(const V* st, V* buf, int n, int bit, int value, int unpack) {
  const size_t half = 1ull << (n - 1);
  const size_t lowm = (1ull << bit) - 1ull;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < half; i += (size_t)gridDim.x * blockDim.x) {
    const size_t src = ((i & ~lowm) << 1) | ((size_t)value << bit) | (i & lowm);
    if (unpack) const_cast<V*>(st)[src] = buf[i];
    else buf[i] = st[src];
  }
}

// Exclusive prefix sum of n <= 1024*64 int64 counts (one CTA): CSR offsets on device.
__global__ void __launch_bounds__(1024) exclusive_scan_i64(const int64_t* in, int n, int64_t* out) {
  __shared__ int64_t part[1024];
  constexpr int PER = 64;
  const int t = threadIdx.x;
  int64_t s = 0;
  for (int e = 0; e < PER; ++e) {
    const int i = t * PER + e;
    if (i < n) s += in[i];
  }
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t acc = 0;
    for (int i = 0; i < 1024; ++i) { const int64_t v = part[i]; part[i] = acc; acc += v; }
  }
  __syncthreads();
  int64_t acc = part[t];
  for (int e = 0; e < PER; ++e) {
    const int i = t * PER + e;
    if (i < n) { out[i] = acc; acc += in[i]; }
  }
}

// Gather each trajectory's runs into one contiguous CSR stream.
__global__ void compact_runs(const uint64_t* run_idx, const uint32_t* run_cnt, const int64_t* off,
                             const int64_t* nuniq, const int64_t* uoff, uint64_t* out_idx, uint32_t* out_cnt) {
  const int b = blockIdx.y;
  const long long n = nuniq[b];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    out_idx[uoff[b] + i] = run_idx[off[b] + i];
    out_cnt[uoff[b] + i] = run_cnt[off[b] + i];
  }
}

}  // namespace ptsbe
