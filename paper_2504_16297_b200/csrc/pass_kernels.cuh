// pass_kernels.cuh -- fused gate/Kraus passes over a batch of statevectors.
//
// Replaces the per-op loop of prepare_state (reference execute.py:85-97), which
// costs one full-state numpy pass per gate and per noise site
// (statevector.py:102-109 / :91-99), by P << (#ops + #sites) HBM passes.
//
// Pass = tile sweep.  One CTA owns one TILE of one trajectory's state: the 2^L
// amplitudes whose basis indices agree outside the pass's qubit set Q (|Q| = L).
// Q always contains qubits 0..c-1, so a tile is 2^(L-c) rows of 2^c contiguous
// amplitudes (>= 128 B), moved with coalesced 16-B streaming loads/stores.
// Every op of the pass has its targets inside Q, so it acts block-diagonally on
// tiles; the tile is read from HBM once and written once.
//
// Phase = register sweep.  Inside the tile the pass's ops are grouped (by the
// host, engine.cu) into phases whose targets span at most 4 tile bits.  Each
// thread owns one 16-amplitude group of a phase in registers and applies every
// op of the phase there -- with the gate's kind specialised (real, diagonal,
// phase, anti-diagonal, CX, SWAP, general) and its bit positions compile-time
// so the register file is indexed statically.  Between phases the tile goes
// through XOR-swizzled shared memory once.
//
// Noise sites read the trajectory's outcome from sel[b][site]; exact-identity
// outcomes (U_0 = I of every builtin mixture) are skipped bit-exactly and
// CTA-uniformly.  Non-unitary Kraus ops (general channels, statevector.py:
// 136-145) are applied unnormalised; right after each one the CTA reduces its
// tile's ||.||^2 into a per-tile partial (an op inside Q preserves every other
// tile), norm_finalize turns partials into realized weights, and the
// 1/sqrt(norm^2) rescale is deferred into the next pass's loads.
#pragma once
#include "common.cuh"

namespace ptsbe {

// matrix kinds (engine.cu classifies every matrix of the operator table)
enum : int32_t {
  MK_GEN1 = 0, MK_REAL1 = 1, MK_DIAG1 = 2, MK_PHASE1 = 3, MK_ANTI1 = 4,
  MK_GEN2 = 8, MK_CX2 = 9, MK_SWAP2 = 10, MK_DIAG2 = 11
};

struct DevOp {
  int32_t kind;    // 0 gate, 1 site
  int32_t arity;   // 1 or 2
  int32_t b0;      // tile bit of first target (MSB of matrix index)
  int32_t b1;      // tile bit of second target or -1
  int32_t ref;     // gate: matrix index; site: site id
  int32_t slot;    // general-channel site: norm slot within the pass, else -1
  int32_t k0, k1;  // register-bit positions (0..3) of b0/b1 inside the op's phase
};

struct DevPhase {
  uint32_t pbits;  // 4 tile bit positions, 5 bits each (ascending)
  int32_t op_begin;
  int32_t n_ops;
  int32_t pad;
};

struct DevChan {
  int32_t n_outcomes;
  int32_t mat_base;
  int32_t general;
  int32_t arity;
  uint64_t identity_mask;
};

struct PassParams {
  void* states;              // [B][2^n] amplitudes
  int n;                     // qubits
  int L;                     // tile bits
  int c;                     // contiguous low bits in Q
  uint64_t qmask;            // Q
  const DevOp* ops;          // this pass's ops, phase-major
  int n_ops;
  const DevPhase* phases;    // this pass's phases
  int n_phases;
  const uint8_t* sel;        // [B][S]
  int S;
  const int32_t* site_chan;  // [S]
  const DevChan* chans;
  const void* mats;          // [n_mats][16] V
  const int32_t* mat_kind;   // [n_mats]
  const double* nst;         // [B] norm^2 of the stored state (used when use_scale)
  int use_scale;
  int gen_zero;              // first pass: synthesize |0...0> (1) or the zero vector (2) instead of loading
  double* partials;          // [slot][B][tiles]
  const int32_t* status;     // [B]
  int B;                     // trajectory rows (stride of per-row tables)
  long long tiles;
  const int4* ent;           // [E] launch entries {row, src slot, dst slot, 0}
  int E;
  uint64_t* tsum;            // generated last pass: sampler block sums in tile order (or null)
  long long tsum_stride;     // blocks per trajectory row
  int tsum_sbits;            // log2 amplitudes per sampler block
};

// ---- shared-memory swizzle: spreads the 32 lanes of a phase access over banks
template <typename V> __device__ __forceinline__ uint32_t swz(uint32_t i);
template <> __device__ __forceinline__ uint32_t swz<float2>(uint32_t i) {
  // never flips bit 0: adjacent amplitude pairs stay one aligned 16-B vector
  const uint32_t h = (i >> 3) ^ (i >> 7) ^ ((i >> 7) << 1) ^ (i >> 11);
  return i ^ (h & 14u);
}
template <> __device__ __forceinline__ uint32_t swz<double2>(uint32_t i) {
  const uint32_t h = (i >> 3) ^ (i >> 6) ^ ((i >> 6) << 1) ^ (i >> 9) ^ (i >> 12);
  return i ^ (h & 7u);
}

// ---- register-resident gate kernels on a 16-amplitude group; K* are bit positions
template <int K, typename V>
__device__ __forceinline__ void r1_gen(V* a, const V* m) {
  const V m00 = m[0], m01 = m[1], m10 = m[4], m11 = m[5];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = cmadd2(m00, x, m01, y);
      a[j | (1 << K)] = cmadd2(m10, x, m11, y);
    }
}
template <int K, typename V>
__device__ __forceinline__ void r1_real(V* a, const V* m) {
  const auto m00 = m[0].x, m01 = m[1].x, m10 = m[4].x, m11 = m[5].x;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      V u, v;
      u.x = m00 * x.x + m01 * y.x; u.y = m00 * x.y + m01 * y.y;
      v.x = m10 * x.x + m11 * y.x; v.y = m10 * x.y + m11 * y.y;
      a[j] = u;
      a[j | (1 << K)] = v;
    }
}
template <typename V>
__device__ __forceinline__ V cmul(V d, V x) {
  V r;
  r.x = d.x * x.x - d.y * x.y;
  r.y = d.x * x.y + d.y * x.x;
  return r;
}
template <int K, typename V>
__device__ __forceinline__ void r1_diag(V* a, const V* m) {
  const V d0 = m[0], d1 = m[5];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = cmul((j & (1 << K)) ? d1 : d0, a[j]);
}
template <int K, typename V>
__device__ __forceinline__ void r1_phase(V* a, const V* m) {   // diag(1, d1)
  const V d1 = m[5];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j & (1 << K)) a[j] = cmul(d1, a[j]);
}
template <int K, typename V>
__device__ __forceinline__ void r1_anti(V* a, const V* m) {    // [[0, m01], [m10, 0]]
  const V m01 = m[1], m10 = m[4];
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (!(j & (1 << K))) {
      const V x = a[j], y = a[j | (1 << K)];
      a[j] = cmul(m01, y);
      a[j | (1 << K)] = cmul(m10, x);
    }
}
// 2-qubit ops: KH = register bit of the first-listed target (MSB of local index)
template <int KH, int KL, typename V>
__device__ __forceinline__ void r2_gen(V* a, const V* m) {
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (!(j & (1 << KH)) && !(j & (1 << KL))) {
      const int i1 = j | (1 << KL), i2 = j | (1 << KH), i3 = j | (1 << KH) | (1 << KL);
      const V v0 = a[j], v1 = a[i1], v2 = a[i2], v3 = a[i3];
      a[j] = cmadd4(m + 0, v0, v1, v2, v3);
      a[i1] = cmadd4(m + 4, v0, v1, v2, v3);
      a[i2] = cmadd4(m + 8, v0, v1, v2, v3);
      a[i3] = cmadd4(m + 12, v0, v1, v2, v3);
    }
}
template <int KH, int KL, typename V>
__device__ __forceinline__ void r2_cx(V* a) {    // control = first target (KH), flip KL
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if ((j & (1 << KH)) && !(j & (1 << KL))) {
      const V t = a[j];
      a[j] = a[j | (1 << KL)];
      a[j | (1 << KL)] = t;
    }
}
template <int KH, int KL, typename V>
__device__ __forceinline__ void r2_swap(V* a) {
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if ((j & (1 << KH)) && !(j & (1 << KL))) {
      const int o = (j & ~(1 << KH)) | (1 << KL);
      const V t = a[j];
      a[j] = a[o];
      a[o] = t;
    }
}
template <int KH, int KL, typename V>
__device__ __forceinline__ void r2_diag(V* a, const V* m) {
  const V d0 = m[0], d1 = m[5], d2 = m[10], d3 = m[15];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int s = ((j >> KH) & 1) * 2 + ((j >> KL) & 1);
    a[j] = cmul(s == 0 ? d0 : s == 1 ? d1 : s == 2 ? d2 : d3, a[j]);
  }
}

// ---- one switch over (kind, register positions): a single indirect branch per op
struct CompactOp {
  int32_t code;    // kind * 16 + k0 * 4 + k1
  int32_t mat;     // matrix index
  int32_t slot;    // general-channel norm slot or -1
  int32_t pad;
};

template <typename V>
__device__ __forceinline__ void apply_code(V* a, int code, const V* m) {
#define C1(KIND, FN, K) case KIND * 16 + K * 4: FN<K>(a, m); break;
#define C1ALL(KIND, FN) C1(KIND, FN, 0) C1(KIND, FN, 1) C1(KIND, FN, 2) C1(KIND, FN, 3)
#define C2(KIND, EXPR, H, L) case KIND * 16 + H * 4 + L: EXPR(H, L); break;
#define C2ALL(KIND, EXPR) C2(KIND, EXPR, 0, 1) C2(KIND, EXPR, 0, 2) C2(KIND, EXPR, 0, 3) C2(KIND, EXPR, 1, 0) \
  C2(KIND, EXPR, 1, 2) C2(KIND, EXPR, 1, 3) C2(KIND, EXPR, 2, 0) C2(KIND, EXPR, 2, 1) C2(KIND, EXPR, 2, 3)       \
  C2(KIND, EXPR, 3, 0) C2(KIND, EXPR, 3, 1) C2(KIND, EXPR, 3, 2)
#define E_GEN(H, L) r2_gen<H, L>(a, m)
#define E_CX(H, L) r2_cx<H, L>(a)
#define E_SWAP(H, L) r2_swap<H, L>(a)
#define E_DIAG(H, L) r2_diag<H, L>(a, m)
  switch (code) {
    C1ALL(MK_GEN1, r1_gen)
    C1ALL(MK_REAL1, r1_real)
    C1ALL(MK_DIAG1, r1_diag)
    C1ALL(MK_PHASE1, r1_phase)
    C1ALL(MK_ANTI1, r1_anti)
    C2ALL(MK_GEN2, E_GEN)
    C2ALL(MK_CX2, E_CX)
    C2ALL(MK_SWAP2, E_SWAP)
    C2ALL(MK_DIAG2, E_DIAG)
    default: break;
  }
#undef C1
#undef C1ALL
#undef C2
#undef C2ALL
#undef E_GEN
#undef E_CX
#undef E_SWAP
#undef E_DIAG
}

// Shared-memory layout of the pass kernel (dynamic):
//   buf[2][2^L] V | rowoff [2^(L-c)] u64 | red [32] f64 | cops [n_ops] CompactOp | cph [n_phases] int2
__host__ __device__ inline size_t pass_smem_bytes(int L, int c, size_t amp_bytes, int n_ops, int n_phases) {
  return 2 * ((size_t)1 << L) * amp_bytes + (((size_t)1 << L) >> c) * 8 + 32 * 8 +
         (size_t)n_ops * sizeof(CompactOp) + (size_t)n_phases * 8;
}

__device__ __forceinline__ void cp_async16(void* smem_ptr, const void* gptr) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_ptr);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gptr) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Persistent, double-buffered pass kernel.  The grid walks the flattened
// (trajectory, tile) space; while a CTA runs the phases of tile i out of one
// shared buffer, cp.async streams tile i+gridDim into the other, so HBM
// traffic overlaps the register work.  Threads = max(32, 2^(L-4)): each thread
// owns at most one 16-amplitude group per phase.
template <typename R>
__global__ void __launch_bounds__(sizeof(R) == 8 ? 256 : 512) pass_kernel(PassParams p) {
  using V = typename Cplx<R>::V;
  using W = typename Cplx<R>::W;
  constexpr int VPW = sizeof(W) / sizeof(V);   // amplitudes per 16-B vector
  extern __shared__ __align__(16) unsigned char smem[];

  const int L = p.L, c = p.c;
  const uint32_t TL = 1u << L;
  V* buf0 = reinterpret_cast<V*>(smem);
  V* buf1 = buf0 + TL;
  uint64_t* rowoff = reinterpret_cast<uint64_t*>(buf1 + TL);
  double* red = reinterpret_cast<double*>(rowoff + (TL >> c));
  CompactOp* cops = reinterpret_cast<CompactOp*>(red + 32);
  int2* cph = reinterpret_cast<int2*>(cops + p.n_ops);

  const uint64_t nmask = (p.n >= 64) ? ~0ull : ((1ull << p.n) - 1ull);
  const uint64_t comp = ~p.qmask & nmask;
  const uint64_t hmask = p.qmask & ~((1ull << c) - 1ull);
  const uint32_t rows = TL >> c;
  for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) rowoff[r] = pdep64(r, hmask);
  __syncthreads();

  const int cpr_log = c - (VPW == 2 ? 1 : 0);   // 16-B vectors per row, log2
  const uint32_t nvec = TL / VPW;
  const long long total = (long long)p.E * p.tiles;

  auto issue_load = [&](long long tt, V* dst) {
    const int eb = (int)(tt / p.tiles);
    const int4 en = p.ent[eb];
    if (p.gen_zero || p.status[en.x] != 0) return;
    const uint64_t base = pdep64((uint64_t)(tt - (long long)eb * p.tiles), comp);
    const V* src = reinterpret_cast<const V*>(p.states) + ((size_t)en.y << p.n) + base;
#pragma unroll 4
    for (uint32_t u = threadIdx.x; u < nvec; u += blockDim.x) {
      const uint32_t r = u >> cpr_log;
      const uint32_t j = u & ((1u << cpr_log) - 1u);
      cp_async16(dst + swz<V>((r << c) | (j * VPW)), src + rowoff[r] + (uint64_t)j * VPW);
    }
  };

  long long t = blockIdx.x;
  if (t < total) issue_load(t, buf0);
  cp_async_commit();
  const V* mats = reinterpret_cast<const V*>(p.mats);
  const uint32_t g = threadIdx.x;               // this thread's group
  const bool active = g < (TL >> 4);            // blockDim may exceed 2^(L-4) for L < 8
  int cur_b = -1;
  for (int it = 0; t < total; t += gridDim.x, ++it) {
    V* cur = (it & 1) ? buf1 : buf0;
    V* nxt = (it & 1) ? buf0 : buf1;
    if (t + gridDim.x < total) issue_load(t + gridDim.x, nxt);
    cp_async_commit();
    cp_async_wait<1>();                         // this thread's copies of `cur` landed
    __syncthreads();                            // ... and everyone else's
    const int eb = (int)(t / p.tiles);
    const long long tile = t - (long long)eb * p.tiles;
    const int4 en = p.ent[eb];
    const int b = en.x;                         // trajectory row
    if (p.status[b] != 0) continue;             // annihilated: stop evolving (CTA-uniform)
    if (b != cur_b) {
      // warp 0: this trajectory's op list, identity outcomes dropped, decoded once
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int out = 0;
        for (int ph = 0; ph < p.n_phases; ++ph) {
          const DevPhase P = p.phases[ph];
          const int start = out;
          for (int k0 = 0; k0 < P.n_ops; k0 += 32) {
            const int k = P.op_begin + k0 + lane;
            bool keep = false;
            CompactOp co{0, 0, -1, 0};
            if (k0 + lane < P.n_ops) {
              const DevOp op = p.ops[k];
              int mat = op.ref;
              keep = true;
              if (op.kind == 1) {
                const int outcome = p.sel[(size_t)b * p.S + op.ref];
                const DevChan ch = p.chans[p.site_chan[op.ref]];
                keep = !((ch.identity_mask >> outcome) & 1ull);
                mat = ch.mat_base + outcome;
                if (ch.general) co.slot = op.slot;
              }
              co.mat = mat;
              co.code = p.mat_kind[mat] * 16 + op.k0 * 4 + (op.arity == 2 ? op.k1 : 0);
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) cops[out + __popc(bal & ((1u << lane) - 1u))] = co;
            out += __popc(bal);
          }
          if (lane == 0) cph[ph] = make_int2(start, out - start);
        }
      }
      __syncthreads();
      cur_b = b;
    }
    const uint64_t base = pdep64((uint64_t)tile, comp);
    const R scale = (p.use_scale && !p.gen_zero) ? (R)rsqrt(p.nst[b]) : R(1);

    // ---- phases: shared -> registers, apply, registers -> shared
    for (int ph = 0; ph < p.n_phases; ++ph) {
      const DevPhase P = p.phases[ph];
      const int p0 = P.pbits & 31, p1 = (P.pbits >> 5) & 31, p2 = (P.pbits >> 10) & 31, p3 = (P.pbits >> 15) & 31;
      const uint32_t gb = insert0(insert0(insert0(insert0(g, p0), p1), p2), p3);
      // swz is linear over GF(2) and gb / offsets have disjoint bits: addr_j = swz(gb) ^ swz(off_j)
      const uint32_t sg = swz<V>(gb);
      uint32_t so[16];
      so[0] = 0;
      so[1] = swz<V>(1u << p0);
      so[2] = swz<V>(1u << p1);
      so[4] = swz<V>(1u << p2);
      so[8] = swz<V>(1u << p3);
#pragma unroll
      for (int j = 3; j < 16; ++j)
        if (j & (j - 1)) so[j] = so[j & (j - 1)] ^ so[j & -j];
      V a[16];
      if (ph == 0 && p.gen_zero) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const bool one = p.gen_zero == 1 && base == 0 && active && (gb | ((j & 1) << p0) | (((j >> 1) & 1) << p1) |
                                                     (((j >> 2) & 1) << p2) | (((j >> 3) & 1) << p3)) == 0;
          a[j] = make_vec2<V>(one ? 1.0 : 0.0, 0.0);
        }
      } else if (active) {
        if (VPW == 2 && p0 == 0) {            // bit 0 in the phase: adjacent pairs, 16-B accesses
#pragma unroll
          for (int j = 0; j < 16; j += 2) {
            const float4 w = *reinterpret_cast<const float4*>(cur + (sg ^ so[j]));
            a[j] = make_vec2<V>(w.x, w.y);
            a[j + 1] = make_vec2<V>(w.z, w.w);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) a[j] = cur[sg ^ so[j]];
        }
        if (ph == 0 && p.use_scale) {
#pragma unroll
          for (int j = 0; j < 16; ++j) { a[j].x *= scale; a[j].y *= scale; }
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = make_vec2<V>(0, 0);
      }
      const int2 range = cph[ph];
      for (int k = range.x; k < range.x + range.y; ++k) {
        const CompactOp co = cops[k];
        apply_code(a, co.code, mats + (size_t)co.mat * 16);
        if (co.slot >= 0) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < 16; ++j) s += prob64(a[j]);
          s = block_sum_f64(s, red);
          if (threadIdx.x == 0) p.partials[((size_t)co.slot * p.B + b) * p.tiles + tile] = s;
        }
      }
      if (active) {
        if (VPW == 2 && p0 == 0) {
#pragma unroll
          for (int j = 0; j < 16; j += 2)
            *reinterpret_cast<float4*>(cur + (sg ^ so[j])) = make_float4(a[j].x, a[j].y, a[j + 1].x, a[j + 1].y);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) cur[sg ^ so[j]] = a[j];
        }
      }
      __syncthreads();
    }

    // ---- shared -> HBM
    V* st = reinterpret_cast<V*>(p.states) + ((size_t)en.z << p.n) + base;
#pragma unroll 4
    for (uint32_t u = threadIdx.x; u < nvec; u += blockDim.x) {
      const uint32_t r = u >> cpr_log;
      const uint32_t j = u & ((1u << cpr_log) - 1u);
      const W w = *reinterpret_cast<const W*>(cur + swz<V>((r << c) | (j * VPW)));
      st_stream(reinterpret_cast<W*>(st + rowoff[r] + (uint64_t)j * VPW), w);
    }
    __syncthreads();                            // `cur` is refilled two iterations from now
  }
  cp_async_wait<0>();
}

// Tiny states (L < 4): one op at a time in shared memory.
template <typename R>
__global__ void __launch_bounds__(32) pass_kernel_small(PassParams p) {
  using V = typename Cplx<R>::V;
  __shared__ V tile[16];
  __shared__ double red[32];
  const int4 en = p.ent[blockIdx.y];
  const int b = en.x;
  if (p.status[b] != 0) return;
  const uint32_t TL = 1u << p.L;                 // == 2^n, one tile
  const V* src = reinterpret_cast<const V*>(p.states) + ((size_t)en.y << p.n);
  V* st = reinterpret_cast<V*>(p.states) + ((size_t)en.z << p.n);
  const R scale = (!p.gen_zero && p.use_scale) ? (R)rsqrt(p.nst[b]) : R(1);
  for (uint32_t i = threadIdx.x; i < TL; i += blockDim.x) {
    V v;
    if (p.gen_zero) { v.x = (i == 0 && p.gen_zero == 1) ? R(1) : R(0); v.y = R(0); }
    else { v = src[i]; v.x *= scale; v.y *= scale; }
    tile[i] = v;
  }
  __syncthreads();
  const V* mats = reinterpret_cast<const V*>(p.mats);
  for (int k = 0; k < p.n_ops; ++k) {
    const DevOp op = p.ops[k];
    int mat = op.ref;
    bool general = false;
    if (op.kind == 1) {
      const int outcome = p.sel[(size_t)b * p.S + op.ref];
      const DevChan ch = p.chans[p.site_chan[op.ref]];
      if ((ch.identity_mask >> outcome) & 1ull) continue;
      mat = ch.mat_base + outcome;
      general = ch.general != 0;
    }
    const V* m = mats + (size_t)mat * 16;
    V out = make_vec2<V>(0, 0);
    const uint32_t i = threadIdx.x;
    if (i < TL) {
      if (op.arity == 1) {
        const int bit = (i >> op.b0) & 1;
        const V x0 = tile[i & ~(1u << op.b0)], x1 = tile[i | (1u << op.b0)];
        out = cmadd2(m[bit * 4 + 0], x0, m[bit * 4 + 1], x1);
      } else {
        const int r = ((i >> op.b0) & 1) * 2 + ((i >> op.b1) & 1);
        const uint32_t z = i & ~(1u << op.b0) & ~(1u << op.b1);
        const V v0 = tile[z], v1 = tile[z | (1u << op.b1)], v2 = tile[z | (1u << op.b0)],
                v3 = tile[z | (1u << op.b0) | (1u << op.b1)];
        out = cmadd4(m + 4 * r, v0, v1, v2, v3);
      }
    }
    __syncthreads();
    if (i < TL) tile[i] = out;
    __syncthreads();
    if (general) {
      double s = (i < TL) ? prob64(tile[i]) : 0.0;
      s = block_sum_f64(s, red);
      if (threadIdx.x == 0) p.partials[((size_t)op.slot * p.B + b) * p.tiles + blockIdx.x] = s;
    }
  }
  for (uint32_t i = threadIdx.x; i < TL; i += blockDim.x) st[i] = tile[i];
}

// Per trajectory: fold the pass's per-tile partial norms (fixed order ->
// deterministic), derive realized_j = N_j / N_{j-1} per general site in op
// order (weight *= realized_j, execute.py:97), flag annihilation at
// realized <= 1e-14 (statevector.py:141-144) and record the stored state's
// norm^2 for the deferred rescale.
__global__ void __launch_bounds__(256) norm_finalize(const double* partials, int n_slots, int B,
                                                     long long tiles, const int32_t* slot_site,
                                                     double* nst, double* weight, int32_t* status,
                                                     int32_t* fail_site, const int4* ent) {
  __shared__ double red[32];
  const int b = ent[blockIdx.x].x;
  if (status[b] != 0) return;
  double prev = 1.0;
  double w = weight[b];
  for (int j = 0; j < n_slots; ++j) {
    const double* src = partials + ((size_t)j * B + b) * tiles;
    double s = 0.0;
    for (long long t = threadIdx.x; t < tiles; t += blockDim.x) s += src[t];
    s = block_sum_f64(s, red);
    if (threadIdx.x == 0) red[0] = s;
    __syncthreads();
    const double nj = red[0];
    __syncthreads();
    const double realized = nj / prev;
    if (!(realized > 1e-14)) {        // also catches 0/0
      if (threadIdx.x == 0) {
        status[b] = 2;
        fail_site[b] = slot_site[j];
        weight[b] = realized == realized ? realized : 0.0;   // host reports the offending norm^2
      }
      return;
    }
    w *= realized;
    prev = nj;
  }
  if (threadIdx.x == 0) {
    weight[b] = w;
    nst[b] = prev;
  }
}

// |0...0> for programs with no passes (empty circuits).
template <typename R>
__global__ void init_zero_kernel(void* states, int n, int B, int all_zero = 0) {
  using V = typename Cplx<R>::V;
  V* s = reinterpret_cast<V*>(states);
  const size_t total = (size_t)B << n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    V z; z.x = (!all_zero && (i & ((1ull << n) - 1)) == 0) ? R(1) : R(0); z.y = R(0);
    s[i] = z;
  }
}

__global__ void batch_reset(double* weight, double* nst, int32_t* status, int32_t* fail_site, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) { weight[b] = 1.0; nst[b] = 1.0; status[b] = 0; fail_site[b] = -1; }
}

// Forked trajectories inherit the shared trunk's running weight / norm / status.
__global__ void fork_rows(const int32_t* rows, int n, int trunk, double* weight, double* nst, int32_t* status,
                          int32_t* fail_site) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int r = rows[i];
    weight[r] = weight[trunk]; nst[r] = nst[trunk]; status[r] = status[trunk]; fail_site[r] = fail_site[trunk];
  }
}

// Split-off trajectory groups inherit their parent's running weight / norm / status:
// pairs[2i] (child row) <- pairs[2i+1] (parent row).
__global__ void fork_pairs(const int32_t* pairs, int n, double* weight, double* nst, int32_t* status,
                           int32_t* fail_site) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int r = pairs[2 * i], src = pairs[2 * i + 1];
    weight[r] = weight[src]; nst[r] = nst[src]; status[r] = status[src]; fail_site[r] = fail_site[src];
  }
}

// Multiply state b by 1/sqrt(nst[b]) (normalise before download).
template <typename R>
__global__ void scale_states(void* states, int n, int B, const double* nst, int invert_sqrt) {
  using V = typename Cplx<R>::V;
  V* s = reinterpret_cast<V*>(states);
  const size_t per = 1ull << n;
  const size_t total = (size_t)B * per;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const double f = invert_sqrt ? rsqrt(nst[i / per]) : nst[i / per];
    V v = s[i];
    v.x = (R)(v.x * f); v.y = (R)(v.y * f);
    s[i] = v;
  }
}

}  // namespace ptsbe
