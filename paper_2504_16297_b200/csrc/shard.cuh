// shard.cuh -- intra-trajectory state sharding: global<->local qubit swaps and cross-shard
// Kraus norms (drives sharded.py).
//
// A 2^(n+k)-amplitude state is split over 2^k shards by its top k (global) bits; a shard
// holds 2^n local amplitudes.  Swapping k' global bits g_1..g_k' with local bits
// l_1..l_k' is an all-to-all inside each group of 2^k' shards that differ only in those
// global bits: shard s sends its PART c (the amplitudes whose local bits l_j spell c) to
// the shard whose global bits g_j spell c, and stores the part it receives from that shard
// in the same positions (the received amplitudes carry the sender's global bits, which
// become local bits l_j = c).  The part spelling s's own global bits stays in place.
//
// Renormalising (general) Kraus sites need the norm of the WHOLE state: every shard
// reduces its tiles' partials per (slot, trajectory) (norm_slot_sums), the sums are
// added over shards (ncclAllReduce on the engine stream, or the host for shards of one
// process), and norm_finalize_sums turns the global norms into realized weights, the
// stored norm and annihilation status exactly as norm_finalize does unsharded.
#pragma once
#include "common.cuh"

namespace ptsbe {

struct PartMap {
  int kp;               // swapped pairs k'
  int lbit[3];          // local bit of pair j, ascending order of insertion (sorted)
  int lsort[3];         // the same local bits sorted ascending (zero insertion order)
  uint64_t lmask;
};

__device__ __forceinline__ uint64_t part_pos(const PartMap& m, uint64_t j, uint32_t c) {
  uint64_t x = j;
  for (int t = 0; t < m.kp; ++t) {   // open a zero at each swapped local bit, lowest first
    const uint64_t lo = x & ((1ull << m.lsort[t]) - 1ull);
    x = ((x ^ lo) << 1) | lo;
  }
  for (int t = 0; t < m.kp; ++t) x |= (uint64_t)((c >> t) & 1u) << m.lbit[t];
  return x;
}

// Gather (unpack = 0) / scatter (unpack = 1) elements [j0, j0 + len) of part c of one state.
template <typename V>
__global__ void part_copy(V* st, V* buf, PartMap m, uint32_t c, uint64_t j0, uint64_t len, int unpack) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pos = part_pos(m, j0 + i, c);
    if (unpack) st[pos] = buf[i];
    else buf[i] = st[pos];
  }
}

// Shards of one process on one device: swap part c of state a with part d of state b in place.
template <typename V>
__global__ void part_swap(V* a, V* b, PartMap m, uint32_t c, uint32_t d, uint64_t len) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pa = part_pos(m, i, c), pb = part_pos(m, i, d);
    const V t = a[pa];
    a[pa] = b[pb];
    b[pb] = t;
  }
}

// Per launch entry, the shard-local norm^2 of every renormalising slot of the pass:
// sums[j * Bst + b] (same per-tile partials norm_finalize folds).
__global__ void __launch_bounds__(256) norm_slot_sums(const double* partials, int n_slots, int Bst, long long tiles,
                                                      const int4* ent, const int32_t* status, double* sums) {
  __shared__ double red[32];
  const int b = ent[blockIdx.x].x;
  const bool live = status[b] == 0;
  for (int j = 0; j < n_slots; ++j) {
    const double* src = partials + ((size_t)j * Bst + b) * tiles;
    double s = 0.0;
    if (live)
      for (long long t = threadIdx.x; t < tiles; t += blockDim.x) s += src[t];
    s = block_sum_f64(s, red);
    if (threadIdx.x == 0) sums[(size_t)j * Bst + b] = live ? s : 0.0;
  }
}

// norm_finalize over global (all-shard) slot norms: realized_j = N_j / N_{j-1} in
// reference order, weight *= realized_j, annihilation at realized <= 1e-14, stored norm.
__global__ void norm_finalize_sums(const double* sums, int n_slots, int Bst, const int32_t* slot_site,
                                   double* nst, double* weight, int32_t* status, int32_t* fail_site,
                                   const int4* ent, int E) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int b = ent[e].x;
  if (status[b] != 0) return;
  double prev = 1.0, w = weight[b];
  for (int j = 0; j < n_slots; ++j) {
    const double nj = sums[(size_t)j * Bst + b];
    const double realized = nj / prev;
    if (!(realized > 1e-14)) {
      status[b] = 2;
      fail_site[b] = slot_site[j];
      weight[b] = realized == realized ? realized : 0.0;
      return;
    }
    w *= realized;
    prev = nj;
  }
  weight[b] = w;
  nst[b] = prev;
}

// Amplitudes at given physical indices of one state (verification of states too large to download).
template <typename V>
__global__ void gather_amps(const V* st, const uint64_t* idx, int64_t count, V* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = st[idx[i]];
}

}  // namespace ptsbe
