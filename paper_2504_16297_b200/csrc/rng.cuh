// rng.cuh -- device random streams for the shot sampler.
//
// PCG64: numpy's default BitGenerator (the stream behind stream_rng,
// reference execute.py:44-45,145-146).  128-bit LCG, XSL-RR output taken from
// the state AFTER the step, random() = (out >> 11) * 2^-53.  Any thread can
// jump to draw i with the O(log i) LCG advance, so the m uniforms of
// Generator(PCG64(seed)).random(m) are produced in parallel bit-exactly.
//
// Philox4x32-10: counter-based production stream keyed by the trajectory's
// 64-bit seed (mix_seed(master, t), execute.py:33-41).
#pragma once
#include <cstdint>

namespace ptsbe {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// State after `delta` LCG steps.
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// Output of the step that starts from `state`; returns 53-bit random() mantissa.
__device__ __forceinline__ uint64_t pcg_key53(u128 state_before, u128 inc) {
  const u128 s = state_before * pcg_mult() + inc;
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  const uint64_t r = (x >> rot) | (x << ((64u - rot) & 63u));
  return r >> 11;
}

struct Philox4 { uint32_t x, y, z, w; };

__device__ __forceinline__ Philox4 philox4x32_10(Philox4 ctr, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    Philox4 n;
    n.x = hi1 ^ ctr.y ^ k0;
    n.y = lo1;
    n.z = hi0 ^ ctr.w ^ k1;
    n.w = lo0;
    ctr = n;
    k0 += W0;
    k1 += W1;
  }
  return ctr;
}

}  // namespace ptsbe
