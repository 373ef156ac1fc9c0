// Exact-order float64 building blocks shared by the kernels.
//
// Every helper pins the rounding sequence of the numpy/OpenBLAS expression it
// replaces (SURVEY.md §8(c) "exact recipes"), using explicit _rn intrinsics so
// nvcc can neither contract a*b+c into an FMA nor reassociate.
#pragma once
#include <stdint.h>

namespace bzg {

// OpenBLAS dgemm/dgemm-like products V @ F.T for V >= 2 rows: FMA chain over k
// starting from the plain product of the first term (reference graph.py:174-175,
// geometry.py:148).
__device__ __forceinline__ double fma_chain(const double* __restrict__ v, const double* __restrict__ f, int n) {
  double acc = __dmul_rn(v[0], f[0]);
  for (int k = 1; k < n; ++k) acc = __fma_rn(v[k], f[k], acc);
  return acc;
}

template <int N>
__device__ __forceinline__ double fma_chain_n(const double* __restrict__ v, const double* __restrict__ f) {
  double acc = __dmul_rn(v[0], f[0]);
#pragma unroll
  for (int k = 1; k < N; ++k) acc = __fma_rn(v[k], f[k], acc);
  return acc;
}

// Output control points of edge (xi -> xj): np.einsum("pq,eqm->emp", D, bv)
// (graph.py:193-196), a sequential non-fused sum over q that starts from +0.0.
// D is (2G) x (2G) row-major; P[k][j] for k < M, j < 2G.
template <int G, int M>
__device__ __forceinline__ void control_points(const double* __restrict__ xi, const double* __restrict__ xj,
                                               const double* __restrict__ D, double (&P)[M][2 * G]) {
#pragma unroll
  for (int k = 0; k < M; ++k) {
#pragma unroll
    for (int j = 0; j < 2 * G; ++j) {
      if (M == 1) {
        // m = 1 makes both einsum operands contiguous along q, and numpy's contiguous kernel
        // accumulates in two lanes (even q, odd q) and adds them at the end (measured)
        double ev = 0.0, od = 0.0;
#pragma unroll
        for (int q = 0; q < 2 * G; q += 2) {
          const double b0 = q < G ? xi[q] : xj[q - G];
          const double b1 = q + 1 < G ? xi[q + 1] : xj[q + 1 - G];
          ev = __dadd_rn(ev, __dmul_rn(D[j * 2 * G + q], b0));
          od = __dadd_rn(od, __dmul_rn(D[j * 2 * G + q + 1], b1));
        }
        P[k][j] = __dadd_rn(ev, od);
      } else {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < 2 * G; ++q) {
          const double bq = q < G ? xi[q * M + k] : xj[(q - G) * M + k];
          acc = __dadd_rn(acc, __dmul_rn(D[j * 2 * G + q], bq));
        }
        P[k][j] = acc;
      }
    }
  }
}

// np.linalg.norm(np.diff(P, axis=2), axis=1).sum(axis=1) (graph.py:197):
// per segment sqrt of the sequential sum of squares over m, then a left fold.
template <int G, int M>
__device__ __forceinline__ double polygon_length(const double (&P)[M][2 * G]) {
  double total = 0.0;
#pragma unroll
  for (int s = 0; s < 2 * G - 1; ++s) {
    double d0 = __dsub_rn(P[0][s + 1], P[0][s]);
    double sq = __dmul_rn(d0, d0);
#pragma unroll
    for (int k = 1; k < M; ++k) {
      double dk = __dsub_rn(P[k][s + 1], P[k][s]);
      sq = __dadd_rn(sq, __dmul_rn(dk, dk));
    }
    const double seg = __dsqrt_rn(sq);
    total = (s == 0) ? seg : __dadd_rn(total, seg);
  }
  return total;
}

// ---------------------------------------------------------------- PCG64
// numpy's PCG64 (pcg_setseq_128_xsl_rr_64): step s = s*MULT + inc, then XSL-RR
// output of the NEW state; next_double = (x >> 11) * 2^-53.
typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// LCG jump-ahead by `delta` steps (Brown, "Random number generation with arbitrary strides").
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
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

__device__ __forceinline__ uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__device__ __forceinline__ double pcg_next_double(u128& s, u128 inc) {
  s = s * pcg_mult() + inc;
  return (double)(pcg_output(s) >> 11) * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

}  // namespace bzg
