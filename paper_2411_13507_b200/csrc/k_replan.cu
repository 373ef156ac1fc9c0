// Replanning helper on device: the receding-horizon anchor of the reference simulator,
// sim.py:220-239 (_project_on_path) -- the grid time along the path's curve chain that is
// positionally closest to the vehicle state.  Same arithmetic as the reference:
//   hop i joins path states a_i -> a_{i+1}: output control points (D @ bv).T (bezier.py:210-223;
//     BLAS gemm: an FMA chain over the 2*gamma boundary values, first term a product);
//   tau_k = k * h, i = min(int(tau_k / T + 1e-9), hops - 1), s = (tau_k - i*T) / T;
//   x(s) by de Casteljau (bezier.py:142-148: (1 - s) * w_j + s * w_{j+1}, unfused) on the m
//     position rows; d_k = ||x - state[:m]|| (1-D norm: sqrt of an FMA chain);
//   the first k with the smallest d_k (strict <, sim.py:235-237) -> best tau.
// One block; the k's are independent, the argmin is a (d, k) block reduction.
#include <cmath>
#include <vector>

#include "bzg_internal.cuh"

namespace bzg {
namespace {

constexpr int kProjThreads = 256;
constexpr int kMaxP = 8;  // p + 1 <= 8 (gamma <= 4)

struct ProjParams {
  double D[64];  // (p+1) x 2*gamma, row-major
  double state[3];
  double T, h;
  int m, gamma, p, hops, total;
};

__global__ void __launch_bounds__(kProjThreads) k_project_on_path(ProjParams pp, const double* __restrict__ path,
                                                                  double* __restrict__ out) {
  BZG_PDL_ENTRY();
  const int n = pp.m * pp.gamma, J = pp.p + 1, G2 = 2 * pp.gamma;
  double best_d = INFINITY;
  int best_k = 0x7fffffff;
  for (int k = threadIdx.x; k < pp.total; k += blockDim.x) {
    const double tau = (double)k * pp.h;
    int i = (int)(tau / pp.T + 1e-9);  // int() truncates toward zero, tau >= 0
    if (i > pp.hops - 1) i = pp.hops - 1;
    const double t = tau - (double)i * pp.T;
    const double s = t / pp.T;
    const double oms = 1.0 - s;
    const double* a = path + (size_t)i * n;
    const double* b = path + (size_t)(i + 1) * n;
    double d2 = 0.0;
    double xs[3];
    for (int r = 0; r < pp.m; ++r) {
      // output control points of row r: P[r][j] = sum_q D[j][q] bv[q][r], bv = [a; b] as (2 gamma, m)
      double w[kMaxP];
      for (int j = 0; j < J; ++j) {
        double acc = 0.0;
        for (int q = 0; q < G2; ++q) {
          const double bq = q < pp.gamma ? a[q * pp.m + r] : b[(q - pp.gamma) * pp.m + r];
          acc = q == 0 ? __dmul_rn(pp.D[j * G2 + q], bq) : __fma_rn(pp.D[j * G2 + q], bq, acc);
        }
        w[j] = acc;
      }
      for (int kk = 0; kk < pp.p; ++kk)
        for (int j = 0; j < pp.p - kk; ++j) w[j] = __dadd_rn(__dmul_rn(oms, w[j]), __dmul_rn(s, w[j + 1]));
      xs[r] = __dsub_rn(w[0], pp.state[r]);
    }
    d2 = __dmul_rn(xs[0], xs[0]);
    for (int r = 1; r < pp.m; ++r) d2 = __fma_rn(xs[r], xs[r], d2);
    const double d = __dsqrt_rn(d2);
    if (d < best_d) {  // k increases within a thread, so the first minimum is kept
      best_d = d;
      best_k = k;
    }
  }
  // block argmin on (d, k): the smallest d, the lowest k among equals (the sequential scan's pick)
  __shared__ double sd[kProjThreads];
  __shared__ int sk[kProjThreads];
  sd[threadIdx.x] = best_d;
  sk[threadIdx.x] = best_k;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) {
      const double od = sd[threadIdx.x + off];
      const int ok = sk[threadIdx.x + off];
      if (od < sd[threadIdx.x] || (od == sd[threadIdx.x] && ok < sk[threadIdx.x])) {
        sd[threadIdx.x] = od;
        sk[threadIdx.x] = ok;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sk[0] == 0x7fffffff ? 0.0 : (double)sk[0] * pp.h;
}

}  // namespace

double project_on_path(Ctx* c, int m, int gamma, double T, const double* D, long long L, const double* path_states,
                       double h, int spt, const double* state) {
  BZG_REQUIRE(m >= 1 && m <= 3 && gamma >= 1 && gamma <= 4, BZG_EUNSUPPORTED, "m in 1..3 and gamma in 1..4");
  BZG_REQUIRE(L >= 0 && h > 0.0 && T > 0.0 && spt >= 0, BZG_EINVAL, "bad path / step");
  const long long hops = L > 0 ? L - 1 : 0;
  if (hops == 0) return 0.0;  // sim.py:229-230
  BZG_REQUIRE(hops * (long long)spt < (1ll << 31), BZG_EINVAL, "path too long");
  ProjParams pp{};
  const int p = 2 * gamma - 1;
  for (int k = 0; k < (p + 1) * 2 * gamma; ++k) pp.D[k] = D[k];
  for (int k = 0; k < m; ++k) pp.state[k] = state[k];
  pp.T = T;
  pp.h = h;
  pp.m = m;
  pp.gamma = gamma;
  pp.p = p;
  pp.hops = (int)hops;
  pp.total = (int)(hops * spt);
  const int n = m * gamma;
  DevBuf& d_path = c->ws[WS_PROJ];
  d_path.alloc((size_t)L * n * sizeof(double) + sizeof(double), c->stream);
  BZG_CHECK_CUDA(cudaMemcpyAsync(d_path.ptr, path_states, (size_t)L * n * sizeof(double), cudaMemcpyHostToDevice,
                                 c->stream));
  double* d_out = reinterpret_cast<double*>(d_path.as<char>() + (size_t)L * n * sizeof(double));
  launch(c, "k_project_on_path", k_project_on_path, dim3(1), dim3(kProjThreads), 0, pp,
         (const double*)d_path.as<double>(), d_out);
  double* h_out = static_cast<double*>(c->host_scratch(sizeof(double)));
  BZG_CHECK_CUDA(cudaMemcpyAsync(h_out, d_out, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  return h_out[0];
}

}  // namespace bzg
