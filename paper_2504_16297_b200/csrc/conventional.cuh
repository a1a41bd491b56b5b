// conventional.cuh -- state-dependent Kraus selection for conventional (Algorithm 1)
// trajectories on device (reference trajectory.py:40-70 run_trajectory, :138-219 the
// dense ensemble).
//
// At a general-channel site the reference computes every branch probability
// p_k = ||K_k psi||^2 (statevector.py:129-133, one full transform per outcome),
// picks k = select_index(r, p) with the trajectory's next uniform r, then
// applies K_k and renormalises.  Here all branches come from ONE read of the
// state: the reduced density matrix rho of the site's (<= 2) target qubits,
// rho_lm = sum_rest v_l conj(v_m), gives p_k = Re tr(K_k^+ K_k rho) / tr(rho)
// for every outcome at once.  The fused pass that follows applies K_k (the
// planner puts every decision site first in its pass, see planner.h), so the
// selection costs one extra HBM read of each state per general site.
#pragma once
#include "common.cuh"

namespace ptsbe {

constexpr int kRdmVals = 16;   // 4 diagonal + 6 complex off-diagonal (2-qubit); 1-qubit uses 4

__device__ __forceinline__ uint64_t insert0_64(uint64_t p, int bit) {
  const uint64_t lo = p & ((1ull << bit) - 1ull);
  return ((p ^ lo) << 1) | lo;
}

template <int D, typename V>
__device__ __forceinline__ void rdm_accum(double* acc, const V* v) {
  // diagonal, then (l < m) pairs in row-major order: re, im of v_l conj(v_m)
  int o = D;
#pragma unroll
  for (int l = 0; l < D; ++l) {
    const double xr = v[l].x, xi = v[l].y;
    acc[l] += xr * xr + xi * xi;
#pragma unroll
    for (int m = l + 1; m < D; ++m) {
      const double yr = v[m].x, yi = v[m].y;
      acc[o++] += xr * yr + xi * yi;   // Re(v_l conj v_m)
      acc[o++] += xi * yr - xr * yi;   // Im(v_l conj v_m)
    }
  }
}

// Per (state b, block) partial sums of the target qubits' reduced density matrix.
// p0 = physical bit of the first-listed target (MSB of the local index), p1 of the
// second (arity 2) or -1.  partials[(b * nblk + blk) * kRdmVals + j].
template <typename R, int ARITY>
__global__ void __launch_bounds__(256) site_rdm_partials(const void* states, int n, int p0, int p1,
                                                         const int32_t* status, double* partials, int nblk) {
  using V = typename Cplx<R>::V;
  constexpr int arity = ARITY;
  constexpr int nv = arity == 1 ? 4 : kRdmVals;
  __shared__ double red[32];
  const int b = blockIdx.y;
  const bool live = status[b] == 0;
  double acc[kRdmVals];
#pragma unroll
  for (int j = 0; j < kRdmVals; ++j) acc[j] = 0.0;
  if (live) {
    const V* s = reinterpret_cast<const V*>(states) + ((size_t)b << n);
    const uint64_t groups = 1ull << (n - arity);
    const int lo_bit = arity == 1 ? p0 : min(p0, p1), hi_bit = arity == 1 ? p0 : max(p0, p1);
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)nblk * blockDim.x) {
      uint64_t base = insert0_64(g, lo_bit);
      if (arity == 2) base = insert0_64(base, hi_bit);
      V v[4];
      if constexpr (arity == 1) {
        v[0] = s[base];
        v[1] = s[base | (1ull << p0)];
      } else {
#pragma unroll
        for (int l = 0; l < 4; ++l)
          v[l] = s[base | ((l >> 1) ? (1ull << p0) : 0ull) | ((l & 1) ? (1ull << p1) : 0ull)];
      }
      rdm_accum<1 << arity>(acc, v);
    }
  }
#pragma unroll
  for (int j = 0; j < nv; ++j) {
    const double t = block_sum_f64(acc[j], red);
    if (threadIdx.x == 0) partials[((size_t)b * nblk + blockIdx.x) * kRdmVals + j] = t;
  }
}

// One CTA per state: fold the partials in fixed order, p_k = Re tr(G_k rho) / tr(rho)
// with G_k = K_k^+ K_k (mats64: 4x4 padded complex128 per matrix, outcome k at
// mat_base + k), then k = select_index(u, p) (trajectory.py:27-37: the smallest k
// whose running sum exceeds u, else the last) -> sel[b * S + site].
__global__ void __launch_bounds__(128) site_select(const double* partials, int nblk, int arity,
                                                   const double* mats64, int mat_base, int n_outcomes,
                                                   const double* u, int S, int site, uint8_t* sel,
                                                   const int32_t* status, double* probs_out) {
  __shared__ double red[32];
  __shared__ double rv[kRdmVals];
  const int b = blockIdx.x;
  if (status[b] != 0) return;
  const int nv = arity == 1 ? 4 : kRdmVals;
  for (int j = 0; j < nv; ++j) {
    double s = 0.0;
    for (int t = threadIdx.x; t < nblk; t += blockDim.x) s += partials[((size_t)b * nblk + t) * kRdmVals + j];
    s = block_sum_f64(s, red);
    if (threadIdx.x == 0) rv[j] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int d = 1 << arity;
  // rho as full Hermitian d x d (re, im)
  double rr[4][4], ri[4][4];
  int o = d;
  double tr = 0.0;
  for (int l = 0; l < d; ++l) {
    rr[l][l] = rv[l];
    ri[l][l] = 0.0;
    tr += rv[l];
    for (int m = l + 1; m < d; ++m) {
      rr[l][m] = rv[o];
      ri[l][m] = rv[o + 1];
      rr[m][l] = rv[o];
      ri[m][l] = -rv[o + 1];
      o += 2;
    }
  }
  const double r = u[(size_t)b * S + site];
  double run = 0.0;
  int pick = n_outcomes - 1;
  bool found = false;
  for (int k = 0; k < n_outcomes; ++k) {
    const double* K = mats64 + (size_t)(mat_base + k) * 32;
    // ||K v||^2 summed over the ensemble = sum_{l,m} G_lm rho_ml,
    // G_lm = sum_r conj(K_rl) K_rm, rho_ml = sum v_m conj(v_l)
    double p = 0.0;
    for (int l = 0; l < d; ++l)
      for (int m = 0; m < d; ++m) {
        double gr = 0.0, gi = 0.0;
        for (int q = 0; q < d; ++q) {
          const double ar = K[(q * 4 + l) * 2], ai = -K[(q * 4 + l) * 2 + 1];   // conj(K_ql)
          const double br = K[(q * 4 + m) * 2], bi = K[(q * 4 + m) * 2 + 1];
          gr += ar * br - ai * bi;
          gi += ar * bi + ai * br;
        }
        // rho_ml: rho stored as rho_lm = v_l conj(v_m) -> rho_ml = (rr[m][l], ri[m][l])
        p += gr * rr[m][l] - gi * ri[m][l];
      }
    p /= tr;
    if (probs_out) probs_out[(size_t)b * 64 + k] = p;
    run += p;
    if (!found && r < run) {
      pick = k;
      found = true;
    }
  }
  sel[(size_t)b * S + site] = (uint8_t)pick;
}

}  // namespace ptsbe
