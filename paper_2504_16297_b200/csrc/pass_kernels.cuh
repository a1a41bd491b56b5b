// pass_kernels.cuh -- fused gate/Kraus passes over a batch of statevectors.
//
// Replaces the per-op loop of prepare_state (reference execute.py:85-97), which
// costs one full-state numpy pass per gate and per noise site
// (statevector.py:102-109 / :91-99), by P << (#ops + #sites) HBM passes.
//
// One CTA owns one TILE of one trajectory's state: the 2^L amplitudes whose
// basis indices agree outside the pass's qubit set Q (|Q| = L).  Q always
// contains qubits 0..c-1, so a tile is 2^(L-c) rows of 2^c contiguous
// amplitudes (>= 128 B), moved with coalesced 16-B streaming loads/stores.
// Every op of the pass has its targets inside Q, so it acts block-diagonally on
// tiles: the CTA applies the whole op list in shared memory and writes the tile
// back once.  Noise sites read the trajectory's outcome from sel[b][site];
// exact-identity outcomes (U_0 = I of every builtin mixture) are skipped
// bit-exactly, CTA-uniformly.  Non-unitary Kraus ops (general channels,
// statevector.py:136-145) are applied unnormalised; the CTA writes its tile's
// ||.||^2 right after each one (a unitary inside Q preserves every tile's norm),
// norm_finalize turns the per-tile partials into realized weights, and the
// 1/sqrt(norm^2) rescale is deferred into the next pass's loads.
#pragma once
#include "common.cuh"

namespace ptsbe {

struct DevOp {
  int32_t kind;    // 0 gate, 1 site
  int32_t arity;   // 1 or 2
  int32_t b0;      // local (tile) bit of first target (MSB of matrix index)
  int32_t b1;      // local bit of second target or -1
  int32_t ref;     // gate: matrix index; site: site id
  int32_t slot;    // site of a general channel: norm slot within the pass, else -1
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
  const DevOp* ops;
  int n_ops;
  const uint8_t* sel;        // [B][S]
  int S;
  const int32_t* site_chan;  // [S]
  const DevChan* chans;
  const void* mats;          // [n_mats][16] V
  const double* nst;         // [B] norm^2 of the stored state (used when use_scale)
  int use_scale;
  int gen_zero;              // first pass: synthesize |0...0> instead of loading
  double* partials;          // [slot][B][tiles]
  const int32_t* status;     // [B]
  int B;
  long long tiles;
};

template <typename R>
__global__ void __launch_bounds__(256) pass_kernel(PassParams p) {
  using V = typename Cplx<R>::V;
  using W = typename Cplx<R>::W;
  constexpr int VPW = sizeof(W) / sizeof(V);   // amplitudes per 16-B vector
  extern __shared__ __align__(16) unsigned char smem[];

  const int b = blockIdx.y;
  if (p.status[b] != 0) return;                 // annihilated trajectories stop evolving
  const int L = p.L, c = p.c;
  const uint32_t TL = 1u << L;
  V* tile = reinterpret_cast<V*>(smem);
  uint64_t* rowoff = reinterpret_cast<uint64_t*>(smem + (size_t)TL * sizeof(V));
  double* red = reinterpret_cast<double*>(rowoff + (TL >> c));

  const uint64_t nmask = (p.n >= 64) ? ~0ull : ((1ull << p.n) - 1ull);
  const uint64_t base = pdep64((uint64_t)blockIdx.x, ~p.qmask & nmask);
  const uint64_t hmask = p.qmask & ~((1ull << c) - 1ull);
  const uint32_t rows = TL >> c;
  for (uint32_t r = threadIdx.x; r < rows; r += blockDim.x) rowoff[r] = pdep64(r, hmask);
  __syncthreads();

  V* st = reinterpret_cast<V*>(p.states) + ((size_t)b << p.n);
  const int cpr_log = c - (VPW == 2 ? 1 : 0);   // 16-B vectors per row, log2
  const uint32_t nvec = TL / VPW;

  // ---- load (or synthesize) the tile
  if (p.gen_zero) {
    for (uint32_t i = threadIdx.x; i < TL; i += blockDim.x) {
      V z; z.x = (base == 0 && i == 0) ? R(1) : R(0); z.y = R(0);
      tile[i] = z;
    }
  } else {
    const R scale = p.use_scale ? (R)rsqrt(p.nst[b]) : R(1);
    for (uint32_t u = threadIdx.x; u < nvec; u += blockDim.x) {
      const uint32_t r = u >> cpr_log;
      const uint32_t j = u & ((1u << cpr_log) - 1u);
      const uint64_t g = base + rowoff[r] + (uint64_t)j * VPW;
      W w = ld_stream(reinterpret_cast<const W*>(st + g));
      V* dst = tile + ((r << c) | (j * VPW));
      if constexpr (VPW == 2) {
        dst[0] = make_float2(w.x * scale, w.y * scale);
        dst[1] = make_float2(w.z * scale, w.w * scale);
      } else {
        dst[0] = make_double2(w.x * scale, w.y * scale);
      }
    }
  }
  __syncthreads();

  // ---- apply the pass's op list in shared memory
  const V* mats = reinterpret_cast<const V*>(p.mats);
  for (int k = 0; k < p.n_ops; ++k) {
    const DevOp op = p.ops[k];
    int mat = op.ref;
    bool general = false;
    if (op.kind == 1) {
      const int outcome = p.sel[(size_t)b * p.S + op.ref];
      const DevChan ch = p.chans[p.site_chan[op.ref]];
      if ((ch.identity_mask >> outcome) & 1ull) continue;   // CTA-uniform skip
      mat = ch.mat_base + outcome;
      general = ch.general != 0;
    }
    const V* m = mats + (size_t)mat * 16;
    if (op.arity == 1) {
      const V m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
      const int bit = op.b0;
      const uint32_t step = 1u << bit;
      for (uint32_t q = threadIdx.x; q < (TL >> 1); q += blockDim.x) {
        const uint32_t i0 = insert0(q, bit), i1 = i0 | step;
        const V a0 = tile[i0], a1 = tile[i1];
        tile[i0] = cmadd2(m00, a0, m01, a1);
        tile[i1] = cmadd2(m10, a0, m11, a1);
      }
    } else {
      V mm[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) mm[e] = m[e];
      const int hb = op.b0, lb = op.b1;   // hb: MSB of local index
      const int lo = min(hb, lb), hi = max(hb, lb);
      const uint32_t sh = 1u << hb, sl = 1u << lb;
      for (uint32_t q = threadIdx.x; q < (TL >> 2); q += blockDim.x) {
        const uint32_t i0 = insert0(insert0(q, lo), hi);
        const V v0 = tile[i0], v1 = tile[i0 | sl], v2 = tile[i0 | sh], v3 = tile[i0 | sh | sl];
        tile[i0]           = cmadd4(mm + 0,  v0, v1, v2, v3);
        tile[i0 | sl]      = cmadd4(mm + 4,  v0, v1, v2, v3);
        tile[i0 | sh]      = cmadd4(mm + 8,  v0, v1, v2, v3);
        tile[i0 | sh | sl] = cmadd4(mm + 12, v0, v1, v2, v3);
      }
    }
    __syncthreads();
    if (general) {
      double s = 0.0;
      for (uint32_t i = threadIdx.x; i < TL; i += blockDim.x) s += prob64(tile[i]);
      s = block_sum_f64(s, red);
      if (threadIdx.x == 0)
        p.partials[((size_t)op.slot * p.B + b) * p.tiles + blockIdx.x] = s;
    }
  }

  // ---- store
  for (uint32_t u = threadIdx.x; u < nvec; u += blockDim.x) {
    const uint32_t r = u >> cpr_log;
    const uint32_t j = u & ((1u << cpr_log) - 1u);
    const uint64_t g = base + rowoff[r] + (uint64_t)j * VPW;
    const V* src = tile + ((r << c) | (j * VPW));
    W w;
    if constexpr (VPW == 2) {
      w = make_float4(src[0].x, src[0].y, src[1].x, src[1].y);
    } else {
      w = src[0];
    }
    st_stream(reinterpret_cast<W*>(st + g), w);
  }
}

// Per trajectory: fold the pass's per-tile partial norms (fixed order ->
// deterministic), derive realized_j = N_j / N_{j-1} per general site in op
// order (weight *= realized_j, execute.py:97), flag annihilation at
// realized <= 1e-14 (statevector.py:141-144) and record the stored state's
// norm^2 for the deferred rescale.
__global__ void __launch_bounds__(256) norm_finalize(const double* partials, int n_slots, int B,
                                                     long long tiles, const int32_t* slot_site,
                                                     double* nst, double* weight, int32_t* status,
                                                     int32_t* fail_site) {
  __shared__ double red[32];
  const int b = blockIdx.x;
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
    if (realized <= 1e-14) {
      if (threadIdx.x == 0) {
        status[b] = 2;
        fail_site[b] = slot_site[j];
        weight[b] = realized;     // host reports the offending norm^2
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
__global__ void init_zero_kernel(void* states, int n, int B) {
  using V = typename Cplx<R>::V;
  V* s = reinterpret_cast<V*>(states);
  const size_t total = (size_t)B << n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    V z; z.x = ((i & ((1ull << n) - 1)) == 0) ? R(1) : R(0); z.y = R(0);
    s[i] = z;
  }
}

__global__ void batch_reset(double* weight, double* nst, int32_t* status, int32_t* fail_site, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B) { weight[b] = 1.0; nst[b] = 1.0; status[b] = 0; fail_site[b] = -1; }
}

// Multiply state b by s[b] (used to normalise before download / after set).
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
