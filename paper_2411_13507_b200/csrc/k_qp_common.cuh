// Batched Cut-QP on device: shared pieces of the dense ADMM (k_admm.cuh) and the
// active-set polish (k_polish.cuh).  Included by k_cut.cu.
//
// Problem (reference graph.py:268-282, _cut_qp_problem), per (edge, obstacle):
//   x = [lambda (J); delta (C)],  min delta' delta
//   s.t.  Q lambda - delta <= b  (C rows, Q = A_O P),  lambda >= 0 (J rows),  sum lambda = 1
// solved by the dense ADMM of qpsolver.py:129-233 and polished by qpsolver.py:236-279.
//
// C is the padded obstacle row count of the launch: obstacles with fewer rows carry zero
// rows with b = 1e300.  A padding row is exactly neutral: its delta_c, z_c, y_c stay 0.0
// through every ADMM step (all their updates are sums of products with 0), it never enters
// the polish active set, and it adds 0 to ||delta||.
#pragma once

namespace bzg {
namespace {

// Work-list length known only on the device (cut_graph keeps the heuristic's pending count
// there): n = min(*d_n, cap); d_n == nullptr means n = cap (the host knows it).
__device__ __forceinline__ long long dev_count(long long cap, const unsigned long long* __restrict__ d_n) {
  if (!d_n) return cap;
  const unsigned long long n = *d_n;
  return (long long)n < cap ? (long long)n : cap;
}

struct QpParams {
  double rho, rho_eq, sigma, alpha, one_m_alpha, eps_abs, eps_rel, eps_pinf;
  int max_iter;
  int batch;  // iterations between lane refills in k_qp_admm
};

// Q = A_O @ points (graph.py:276): BLAS product, FMA chain over the m output dimensions.
template <int G, int M, int C>
__device__ __forceinline__ void cut_q_matrix(const ObsRec<M, obs_cap<C>()>& o, const double (&P)[M][2 * G],
                                             double (&Q)[C][2 * G]) {
#pragma unroll
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int j = 0; j < 2 * G; ++j) {
      double acc = __dmul_rn(o.A[c][0], P[0][j]);
#pragma unroll
      for (int k = 1; k < M; ++k) acc = __fma_rn(o.A[c][k], P[k][j], acc);
      Q[c][j] = acc;
    }
}

template <int G, int M, int C>
__device__ __forceinline__ void load_instance(const DParams& dp, const double* __restrict__ Vx,
                                              const int* __restrict__ src, const int* __restrict__ dst,
                                              const ObsRec<M, obs_cap<C>()>* __restrict__ obs, unsigned long long pk,
                                              double (&Q)[C][2 * G], double (&b)[C]) {
  constexpr int N = G * M;
  const long long e = (long long)(pk >> 20);
  const ObsRec<M, obs_cap<C>()>& o = obs[(int)(pk & 0xFFFFF)];
  double xi[N], xj[N], P[M][2 * G];
  const long long a = src[e], c = dst[e];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    xi[k] = Vx[a * N + k];
    xj[k] = Vx[c * N + k];
  }
  control_points<G, M>(xi, xj, dp.D, P);
  cut_q_matrix<G, M, C>(o, P, Q);
#pragma unroll
  for (int k = 0; k < C; ++k) b[k] = o.b[k];
}

}  // namespace
}  // namespace bzg
