// planner.h -- host-side fusion planner and physical-layout search (no GPU needed).
//
// Partition of the op stream (reference order: each gate, then its noise sites
// in site-id order, execute.py:85-97) into HBM passes.  A pass owns a tile
// qubit set Q of `tile_bits` physical qubits that always contains qubits
// 0..low_bits-1 (coalesced rows) and absorbs, in stream order, every op whose
// targets fit in Q and whose predecessors on those qubits already ran; an op
// that does not fit blocks its qubits for the rest of the pass.  Sites of
// general (renormalising) channels never overtake one another: their realized
// weights are ratios of consecutive norms in reference order.
//
// Layout search: the state may be stored with a permutation logical ->
// physical qubit.  Local search (random transpositions, sideways moves
// accepted) minimises the pass count; the sampler maps physical basis indices
// back to logical bitstrings, so results are layout-independent.
#pragma once
#include <cstdint>
#include <vector>

namespace ptsbe {
namespace plan {

struct Op {
  uint64_t mask;   // logical target mask
  bool general;
  int weight = 0;  // counts toward the per-pass gate budget (gates 1, sites 0)
  bool first = false;  // decision site (conventional Algorithm 1): must be the first op of its
                       // pass, so its outcome can be chosen from the state at the pass boundary
};

inline uint64_t phys_mask(uint64_t logical, const std::vector<int>& perm) {
  uint64_t m = 0;
  while (logical) {
    const int q = __builtin_ctzll(logical);
    m |= 1ull << perm[q];
    logical &= logical - 1;
  }
  return m;
}

// Greedy plan; returns the number of passes.  out_pass / out_masks optional.
inline int greedy(int n, const std::vector<Op>& ops, const std::vector<int>& perm, int L, int c,
                  std::vector<int>* out_pass, std::vector<uint64_t>* out_masks, int max_weight = 0) {
  const int m = (int)ops.size();
  if (m == 0) return 0;
  std::vector<uint64_t> pm(m);
  for (int i = 0; i < m; ++i) pm[i] = phys_mask(ops[i].mask, perm);
  const uint64_t all = n >= 64 ? ~0ull : ((1ull << n) - 1);
  if (out_pass) out_pass->assign(m, -1);
  if (out_masks) out_masks->clear();
  if (n <= L) {   // one tile holds the state: one pass, cut before every decision site
    int p = 0;
    for (int i = 0; i < m; ++i) {
      if (ops[i].first && i > 0) ++p;
      if (out_pass) (*out_pass)[i] = p;
    }
    if (out_masks) out_masks->assign(p + 1, all);
    return p + 1;
  }
  const uint64_t low = c >= 64 ? ~0ull : ((1ull << c) - 1);
  std::vector<int> remaining(m), deferred;
  for (int i = 0; i < m; ++i) remaining[i] = i;
  int passes = 0;
  while (!remaining.empty()) {
    uint64_t q = low, blocked = 0;
    bool gen_blocked = false;
    deferred.clear();
    int taken = 0, weight = 0;
    for (int i : remaining) {
      const uint64_t t = pm[i];
      if ((t & blocked) || (ops[i].general && gen_blocked) || (ops[i].first && taken > 0)) {
        deferred.push_back(i);
        blocked |= t;
        gen_blocked = gen_blocked || ops[i].general;
        continue;
      }
      const uint64_t g = q | t;
      const bool budget = max_weight <= 0 || weight + ops[i].weight <= max_weight || taken == 0;
      if (__builtin_popcountll(g) <= L && budget) {
        q = g;
        ++taken;
        weight += ops[i].weight;
        if (out_pass) (*out_pass)[i] = passes;
      } else {
        deferred.push_back(i);
        blocked |= t;
        gen_blocked = gen_blocked || ops[i].general;
      }
    }
    if (taken == 0) return -1;
    for (int b = 0; b < n && __builtin_popcountll(q) < L; ++b) q |= 1ull << b;   // pad: longer rows
    if (out_masks) out_masks->push_back(q);
    ++passes;
    remaining.swap(deferred);
  }
  return passes;
}

struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed * 0x9E3779B97F4A7C15ull + 1) {}
  uint64_t next() {
    s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
    return s * 0x2545F4914F6CDD1Dull;
  }
};

// Improve `perm` in place; returns the best pass count.
inline int search(int n, const std::vector<Op>& ops, std::vector<int>& perm, int L, int c, int iters,
                  uint64_t seed, int max_weight = 0) {
  int best = greedy(n, ops, perm, L, c, nullptr, nullptr, max_weight);
  if (n <= L || iters <= 0 || best <= 1) return best;
  Rng rng(seed);
  std::vector<int> cand = perm;
  for (int it = 0; it < iters; ++it) {
    const int a = (int)(rng.next() % n), b = (int)(rng.next() % n);
    if (a == b) continue;
    cand = perm;
    std::swap(cand[a], cand[b]);
    const int p = greedy(n, ops, cand, L, c, nullptr, nullptr, max_weight);
    if (p >= 0 && p <= best) {
      best = p;
      perm.swap(cand);
    }
  }
  return best;
}

}  // namespace plan
}  // namespace ptsbe
