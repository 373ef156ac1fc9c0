// Obstacle cut on device: box heuristic screen over every (edge, obstacle) pair,
// batched Cut-QP (dense ADMM + active-set polish) for the indeterminate pairs,
// and CutMask aggregation (alive, first-kill provenance, counters).
//
// Replaces reference graph.py:224-265 (_heuristic_batch, box branch),
// graph.py:268-299 (_cut_qp_problem / cut_qp), graph.py:302-350 (cut_graph) and the
// dense ADMM of qpsolver.py:129-304 it calls.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "bzg_internal.cuh"
#include "bzg_math.cuh"

namespace bzg {

namespace {

constexpr int kMaxM = 3;
constexpr int kMaxObsRows = 2 * kMaxM;

struct DParams {
  double D[64];
};

// Per-obstacle record staged in shared memory (box obstacles only).
template <int M>
struct ObsRec {
  double A[2 * M][M];   // normalised rows (geometry.py:135-137)
  double b[2 * M];
  double b_eps[2 * M];  // fl(b + eps_geo)   (graph.py:234)
  double lo[M], hi[M];  // Polytope.as_box bounds (geometry.py:155-185)
};

struct CutScalars {
  double margin;  // CutConfig.heur_margin
  int n_obs;
};

// Heuristic code of one edge against one box obstacle: 0 unsafe, 1 safe, 2 indeterminate
// (graph.py:232-264).  Arithmetic follows the numpy expressions term by term.
template <int G, int M>
__device__ __forceinline__ int box_code(const double (&P)[M][2 * G], const ObsRec<M>& o, double margin) {
  constexpr int J = 2 * G, NC = 2 * M;
  // branch 1: a control point inside the obstacle; vals = einsum("cm,emj->ecj") (sequential from 0)
  bool hit = false;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    bool in = true;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) acc = __dadd_rn(acc, __dmul_rn(o.A[c][k], P[k][j]));
      in = in && (acc <= o.b_eps[c]);
    }
    hit = hit || in;
  }
  if (hit) return 0;
  // branch 2 (box): anchor = first argmin of the squared clamp distance
  int anchor = 0;
  double best = 0.0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double t = __dadd_rn(fmax(__dsub_rn(o.lo[k], P[k][j]), 0.0), fmax(__dsub_rn(P[k][j], o.hi[k]), 0.0));
      const double sq = __dmul_rn(t, t);
      d2 = (k == 0) ? sq : __dadd_rn(d2, sq);
    }
    if (j == 0 || d2 < best) { best = d2; anchor = j; }
  }
  double v[M], pr[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    double vk = P[k][0];
#pragma unroll
    for (int j = 1; j < J; ++j) if (anchor == j) vk = P[k][j];
    v[k] = vk;
    pr[k] = fmin(fmax(vk, o.lo[k]), o.hi[k]);  // np.clip(v, lo, hi)
  }
  // deepest separating face among faces active at the projection; first row on ties
  int face = 0;
  double fbest = -INFINITY;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double sep = __dsub_rn(fma_chain_n<M>(v, o.A[c]), o.b[c]);            // v @ A.T - b
    const double res = fabs(__dsub_rn(fma_chain_n<M>(pr, o.A[c]), o.b[c]));     // |proj @ A.T - b|
    const double val = (res <= 1e-7) ? sep : -INFINITY;
    if (c == 0 || val > fbest) { fbest = val; face = c; }
  }
  double h[M], off = o.b[0];
#pragma unroll
  for (int k = 0; k < M; ++k) h[k] = o.A[0][k];
#pragma unroll
  for (int c = 1; c < NC; ++c)
    if (face == c) {
#pragma unroll
      for (int k = 0; k < M; ++k) h[k] = o.A[c][k];
      off = o.b[c];
    }
  bool clear = true;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double acc = 0.0;  // einsum("em,emj->ej") then - off
#pragma unroll
    for (int k = 0; k < M; ++k) acc = __dadd_rn(acc, __dmul_rn(h[k], P[k][j]));
    clear = clear && (__dsub_rn(acc, off) > margin);
  }
  return clear ? 1 : 2;
}

// One thread per edge, all obstacles of the chunk [o0, o1) in list order.
// Tracks the first heuristic kill, counts codes, and appends indeterminate pairs
// to the QP work list with warp-aggregated atomics.
template <int G, int M>
__global__ void k_cut_heuristic(DParams dp, const double* __restrict__ Vx, long long E, const int* __restrict__ src,
                                const int* __restrict__ dst, const ObsRec<M>* __restrict__ obs, int o0, int o1,
                                double margin, int* __restrict__ first_kill, unsigned long long* __restrict__ counters,
                                unsigned long long* __restrict__ n_pend, unsigned long long cap,
                                unsigned long long* __restrict__ pend) {
  constexpr int N = G * M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ObsRec<M>* s_obs = reinterpret_cast<ObsRec<M>*>(smem_raw);
  const int nob = o1 - o0;
  {
    const double* srcp = reinterpret_cast<const double*>(obs + o0);
    double* dstp = reinterpret_cast<double*>(s_obs);
    const int nd = nob * (int)(sizeof(ObsRec<M>) / sizeof(double));
    for (int t = threadIdx.x; t < nd; t += blockDim.x) dstp[t] = srcp[t];
  }
  __syncthreads();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool valid = e < E;
  double P[M][2 * G];
  int kill = 0x7fffffff;
  if (valid) {
    double xi[N], xj[N];
    const long long a = src[e], b = dst[e];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      xi[k] = Vx[a * N + k];
      xj[k] = Vx[b * N + k];
    }
    control_points<G, M>(xi, xj, dp.D, P);
    kill = first_kill[e];
  }
  unsigned c0 = 0, c1 = 0, c2 = 0;
  const int lane = threadIdx.x & 31;
  for (int oi = 0; oi < nob; ++oi) {
    int code = 1;
    if (valid) code = box_code<G, M>(P, s_obs[oi], margin);
    if (valid) {
      c0 += code == 0;
      c1 += code == 1;
      c2 += code == 2;
      if (code == 0 && kill > o0 + oi) kill = o0 + oi;
    }
    const unsigned want = __ballot_sync(0xffffffffu, valid && code == 2);
    if (want) {
      unsigned long long base = 0;
      const int leader = __ffs(want) - 1;
      if (lane == leader) base = atomicAdd(n_pend, (unsigned long long)__popc(want));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (valid && code == 2) {
        const unsigned long long slot = base + __popc(want & ((1u << lane) - 1u));
        if (slot < cap) pend[slot] = ((unsigned long long)e << 20) | (unsigned long long)(o0 + oi);
      }
    }
  }
  if (valid) first_kill[e] = kill;
  // block reduction of the three counters
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long t0 = BR(tmp).Sum((unsigned long long)c0);
  __syncthreads();
  unsigned long long t1 = BR(tmp).Sum((unsigned long long)c1);
  __syncthreads();
  unsigned long long t2 = BR(tmp).Sum((unsigned long long)c2);
  if (threadIdx.x == 0) {
    atomicAdd(counters + 0, t0);
    atomicAdd(counters + 1, t1);
    atomicAdd(counters + 2, t2);
  }
}

// ------------------------------------------------------------------ Cut-QP ADMM
struct QpParams {
  double rho, rho_eq, sigma, alpha, one_m_alpha, eps_abs, eps_rel, eps_pinf;
  int max_iter;
};

// Dense ADMM on the cut QP (graph.py:268-282 -> qpsolver.py:129-233), one thread per
// instance, persistent lanes that fetch new instances as theirs terminate.
//
// Variables x = [lambda (J); delta (C)], constraints z = [Q lambda - delta (C); lambda (J);
// sum lambda], l = [-inf; 0; 1], u = [b; +inf; 1], rho = [rho..; rho*1e3 on the equality row].
// The reference inverts the (n+mc)^2 KKT matrix per instance; the KKT solve is equivalent to
// xt = (P + sigma I + A'RA)^{-1} (sigma x + A'(R z - y)), zt = A xt, which the structure of A
// reduces to one J x J SPD solve (Schur complement of the diagonal delta block), done here by
// a per-instance Cholesky factor.  Iterates agree with the reference to rounding; termination,
// the infeasibility certificate and MAX_ITER follow qpsolver.py:179-231 line by line.
template <int G, int M>
__global__ void __launch_bounds__(128) k_qp_admm(QpParams qp, DParams dp, const double* __restrict__ Vx,
                                                 const int* __restrict__ src, const int* __restrict__ dst,
                                                 const ObsRec<M>* __restrict__ obs,
                                                 const unsigned long long* __restrict__ pend, long long n_inst,
                                                 unsigned long long* __restrict__ next, int8_t* __restrict__ st_out,
                                                 int* __restrict__ it_out, double* __restrict__ x_out,
                                                 double* __restrict__ res_out) {
  constexpr int J = 2 * G, C = 2 * M, N = G * M, NV = J + C, MC = C + J + 1;
  const int lane = threadIdx.x & 31;
  long long inst = -1;  // -1: needs work, -2: exhausted
  int it = 0;
  double Q[C][J], L[J][J], b[C];
  double lam[J], del[C], z[MC], y[MC];
  const double rho = qp.rho, req = qp.rho_eq, ri = 1.0 / qp.rho, rieq = 1.0 / qp.rho_eq;
  const double kdd = 2.0 + qp.sigma + rho;  // delta-delta diagonal of P + sigma I + A'RA
  while (true) {
    const unsigned need = __ballot_sync(0xffffffffu, inst == -1);
    if (need) {
      unsigned long long base = 0;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base = atomicAdd(next, (unsigned long long)__popc(need));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (inst == -1) {
        const unsigned long long my = base + __popc(need & ((1u << lane) - 1u));
        if ((long long)my >= n_inst) {
          inst = -2;
        } else {
          inst = (long long)my;
          const unsigned long long pk = pend[my];
          const long long e = (long long)(pk >> 20);
          const int oi = (int)(pk & 0xFFFFF);
          const ObsRec<M>& o = obs[oi];
          double xi[N], xj[N], P[M][J];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            xi[k] = Vx[(long long)src[e] * N + k];
            xj[k] = Vx[(long long)dst[e] * N + k];
          }
          control_points<G, M>(xi, xj, dp.D, P);
          // Q = A_O @ points (graph.py:276), BLAS product: FMA chain over m
#pragma unroll
          for (int c = 0; c < C; ++c) {
            b[c] = o.b[c];
#pragma unroll
            for (int j = 0; j < J; ++j) {
              double acc = __dmul_rn(o.A[c][0], P[0][j]);
#pragma unroll
              for (int k = 1; k < M; ++k) acc = __fma_rn(o.A[c][k], P[k][j], acc);
              Q[c][j] = acc;
            }
          }
          // S = (sigma + rho) I + (rho - rho^2/kdd) Q'Q + rho_eq 11'  ->  Cholesky L L'
          const double kap = rho - rho * rho / kdd;
#pragma unroll
          for (int r = 0; r < J; ++r)
#pragma unroll
            for (int s = 0; s <= r; ++s) {
              double qq = 0.0;
#pragma unroll
              for (int c = 0; c < C; ++c) qq = __fma_rn(Q[c][r], Q[c][s], qq);
              L[r][s] = kap * qq + req + (r == s ? qp.sigma + rho : 0.0);
            }
#pragma unroll
          for (int r = 0; r < J; ++r) {
#pragma unroll
            for (int s = 0; s < r; ++s) {
              double t = L[r][s];
#pragma unroll
              for (int k = 0; k < s; ++k) t -= L[r][k] * L[s][k];
              L[r][s] = t / L[s][s];
            }
            double d = L[r][r];
#pragma unroll
            for (int k = 0; k < r; ++k) d -= L[r][k] * L[r][k];
            L[r][r] = sqrt(d);
          }
#pragma unroll
          for (int j = 0; j < J; ++j) lam[j] = 0.0;
#pragma unroll
          for (int c = 0; c < C; ++c) del[c] = 0.0;
#pragma unroll
          for (int i = 0; i < MC; ++i) { z[i] = 0.0; y[i] = 0.0; }
          it = 0;
        }
      }
    }
    if (__all_sync(0xffffffffu, inst == -2)) break;
    if (inst < 0) continue;

    // ---- one ADMM iteration (qpsolver.py:164-174)
    ++it;
    double w[MC];
#pragma unroll
    for (int i = 0; i < MC; ++i) w[i] = (i < MC - 1 ? rho : req) * z[i] - y[i];  // R z - y
    double rl[J], rd_[C];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double acc = qp.sigma * lam[j] + w[C + j] + w[MC - 1];
#pragma unroll
      for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], w[c], acc);
      rl[j] = acc;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) rd_[c] = qp.sigma * del[c] - w[c];
    // S a = rl + rho Q' rd / kdd
    double a[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], rd_[c], acc);
      a[j] = rl[j] + rho * acc / kdd;
    }
#pragma unroll
    for (int r = 0; r < J; ++r) {  // forward L
      double t = a[r];
#pragma unroll
      for (int k = 0; k < r; ++k) t -= L[r][k] * a[k];
      a[r] = t / L[r][r];
    }
#pragma unroll
    for (int r = J - 1; r >= 0; --r) {  // backward L'
      double t = a[r];
#pragma unroll
      for (int k = r + 1; k < J; ++k) t -= L[k][r] * a[k];
      a[r] = t / L[r][r];
    }
    double dd[C], zt[MC];
    double sa = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) sa += a[j];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double qa = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) qa = __fma_rn(Q[c][j], a[j], qa);
      dd[c] = (rd_[c] + rho * qa) / kdd;
      zt[c] = qa - dd[c];
    }
#pragma unroll
    for (int j = 0; j < J; ++j) zt[C + j] = a[j];
    zt[MC - 1] = sa;

    double ln[J], dn[C], zn[MC], yn[MC], zr[MC];
#pragma unroll
    for (int j = 0; j < J; ++j) ln[j] = __dadd_rn(__dmul_rn(qp.alpha, a[j]), __dmul_rn(qp.one_m_alpha, lam[j]));
#pragma unroll
    for (int c = 0; c < C; ++c) dn[c] = __dadd_rn(__dmul_rn(qp.alpha, dd[c]), __dmul_rn(qp.one_m_alpha, del[c]));
#pragma unroll
    for (int i = 0; i < MC; ++i) {
      zr[i] = __dadd_rn(__dmul_rn(qp.alpha, zt[i]), __dmul_rn(qp.one_m_alpha, z[i]));
      const double rinv = i < MC - 1 ? ri : rieq;
      double t = __dadd_rn(zr[i], __dmul_rn(rinv, y[i]));
      // clip to [l, u]
      if (i < C) t = fmin(t, b[i]);
      else if (i < C + J) t = fmax(t, 0.0);
      else t = 1.0;
      zn[i] = t;
      yn[i] = __dadd_rn(y[i], __dmul_rn(i < MC - 1 ? rho : req, __dsub_rn(zr[i], zn[i])));
    }
    // residuals (qpsolver.py:176-186)
    double Ax[MC];
    double sl = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) acc = __dadd_rn(acc, __dmul_rn(Q[c][j], ln[j]));
      Ax[c] = __dsub_rn(acc, dn[c]);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) { Ax[C + j] = ln[j]; sl = __dadd_rn(sl, ln[j]); }
    Ax[MC - 1] = sl;
    double rp = 0.0, maxAx = 0.0, maxz = 0.0;
#pragma unroll
    for (int i = 0; i < MC; ++i) {
      rp = fmax(rp, fabs(__dsub_rn(Ax[i], zn[i])));
      maxAx = fmax(maxAx, fabs(Ax[i]));
      maxz = fmax(maxz, fabs(zn[i]));
    }
    double rdl = 0.0, maxPx = 0.0, maxATy = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < C; ++c) acc = __dadd_rn(acc, __dmul_rn(Q[c][j], yn[c]));
      acc = __dadd_rn(__dadd_rn(acc, yn[C + j]), yn[MC - 1]);
      rdl = fmax(rdl, fabs(acc));
      maxATy = fmax(maxATy, fabs(acc));
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double px = __dmul_rn(2.0, dn[c]);
      maxPx = fmax(maxPx, fabs(px));
      maxATy = fmax(maxATy, fabs(yn[c]));
      rdl = fmax(rdl, fabs(__dsub_rn(px, yn[c])));
    }
    const double eps_p = qp.eps_abs + qp.eps_rel * fmax(maxAx, maxz);
    const double eps_d = qp.eps_abs + qp.eps_rel * fmax(maxPx, maxATy);
    int status = -1;
    if (rp <= eps_p && rdl <= eps_d) {
      status = BZG_SOLVED;
    } else {
      // primal infeasibility certificate (qpsolver.py:193-209)
      double dyn = 0.0;
#pragma unroll
      for (int i = 0; i < MC; ++i) dyn = fmax(dyn, fabs(__dsub_rn(yn[i], y[i])));
      if (dyn > 1e-13) {
        double atd = 0.0, supp = 0.0;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int c = 0; c < C; ++c) acc = __dadd_rn(acc, __dmul_rn(Q[c][j], __dsub_rn(yn[c], y[c])));
          acc = __dadd_rn(__dadd_rn(acc, __dsub_rn(yn[C + j], y[C + j])), __dsub_rn(yn[MC - 1], y[MC - 1]));
          atd = fmax(atd, fabs(acc));
        }
#pragma unroll
        for (int c = 0; c < C; ++c) atd = fmax(atd, fabs(__dsub_rn(yn[c], y[c])));
#pragma unroll
        for (int i = 0; i < MC; ++i) {
          const double dy = __dsub_rn(yn[i], y[i]);
          const double lo = i < C ? -INFINITY : (i < C + J ? 0.0 : 1.0);
          const double hi = i < C ? b[i] : (i < C + J ? INFINITY : 1.0);
          const double t = (dy > 0 ? __dmul_rn(hi, dy) : 0.0) + (dy < 0 ? __dmul_rn(lo, dy) : 0.0);
          supp = __dadd_rn(supp, t);
        }
        if (atd <= qp.eps_pinf * dyn && supp <= -qp.eps_pinf * dyn) status = BZG_INFEASIBLE;
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) lam[j] = ln[j];
#pragma unroll
    for (int c = 0; c < C; ++c) del[c] = dn[c];
#pragma unroll
    for (int i = 0; i < MC; ++i) { z[i] = zn[i]; y[i] = yn[i]; }
    if (status < 0 && it >= qp.max_iter) status = BZG_MAX_ITER;
    if (status >= 0) {
      st_out[inst] = (int8_t)status;
      it_out[inst] = it;
#pragma unroll
      for (int j = 0; j < J; ++j) x_out[inst * NV + j] = lam[j];
#pragma unroll
      for (int c = 0; c < C; ++c) x_out[inst * NV + J + c] = del[c];
      res_out[inst * 2 + 0] = rp;
      res_out[inst * 2 + 1] = rdl;
      inst = -1;
    }
  }
}

// ------------------------------------------------------------------ polish
// Active-set polish (qpsolver.py:236-279), one warp per instance: builds the regularised
// reduced KKT system in shared memory, LU with partial pivoting (lane = row), solve plus two
// steps of iterative refinement, and the acceptance test.  Then ||delta|| and the verdict
// safe = SOLVED and ||delta|| > eps_cut (graph.py:328-329).
constexpr int kPolishWarps = 4;

template <int G, int M>
__global__ void __launch_bounds__(32 * kPolishWarps) k_qp_polish(
    DParams dp, const double* __restrict__ Vx, const int* __restrict__ src, const int* __restrict__ dst,
    const ObsRec<M>* __restrict__ obs, const unsigned long long* __restrict__ pend, long long n_inst, int polish,
    double eps_cut, const int8_t* __restrict__ st, double* __restrict__ x_io, const double* __restrict__ res,
    double* __restrict__ delta_out, uint8_t* __restrict__ safe_out) {
  constexpr int J = 2 * G, C = 2 * M, N = G * M, NV = J + C, MC = C + J + 1, NK = NV + MC;
  static_assert(NK <= 32, "polish system must fit a warp");
  __shared__ double sA[kPolishWarps][MC][NV];
  __shared__ double sK[kPolishWarps][NK][NK + 1];
  __shared__ double sU[kPolishWarps][NK][NK + 1];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long inst = (long long)blockIdx.x * kPolishWarps + wib;
  if (inst >= n_inst) return;
  const int status = st[inst];
  double x[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) x[i] = x_io[inst * NV + i];
  const double rp = res[inst * 2], rd = res[inst * 2 + 1];
  double (&A)[MC][NV] = sA[wib];
  double lo_[MC], hi_[MC];
  const unsigned long long pk = pend[inst];
  const long long e = (long long)(pk >> 20);
  const ObsRec<M>& o = obs[(int)(pk & 0xFFFFF)];
  bool do_polish = polish && (status == BZG_SOLVED || status == BZG_MAX_ITER);
  if (do_polish) {
    // rebuild the constraint matrix (graph.py:275-281)
    double xi[N], xj[N], P[M][J];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      xi[k] = Vx[(long long)src[e] * N + k];
      xj[k] = Vx[(long long)dst[e] * N + k];
    }
    control_points<G, M>(xi, xj, dp.D, P);
    for (int t = lane; t < MC * NV; t += 32) {
      const int r = t / NV, k = t % NV;
      double v = 0.0;
      if (r < C) {
        if (k < J) {
          double acc = __dmul_rn(o.A[r][0], P[0][k]);
          for (int q = 1; q < M; ++q) acc = __fma_rn(o.A[r][q], P[q][k], acc);
          v = acc;
        } else {
          v = (k - J == r) ? -1.0 : 0.0;
        }
      } else if (r < C + J) {
        v = (k == r - C) ? 1.0 : 0.0;
      } else {
        v = k < J ? 1.0 : 0.0;
      }
      A[r][k] = v;
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < MC; ++i) {
      lo_[i] = i < C ? -INFINITY : (i < C + J ? 0.0 : 1.0);
      hi_[i] = i < C ? o.b[i] : (i < C + J ? INFINITY : 1.0);
    }
    // active set at z = A x
    const double tol = fmax(1e-7, 10.0 * rp);
    unsigned act = 0, atlo = 0;
    int k = 0;
#pragma unroll
    for (int i = 0; i < MC; ++i) {
      double zi = 0.0;
#pragma unroll
      for (int q = 0; q < NV; ++q) zi = __fma_rn(A[i][q], x[q], zi);
      const bool l_ = __dsub_rn(zi, lo_[i]) <= tol, u_ = __dsub_rn(hi_[i], zi) <= tol;
      if (l_ || u_) { act |= 1u << i; if (l_) atlo |= 1u << i; ++k; }
    }
    if (k > 0) {
      const int nk = NV + k;
      const double reg = 1e-8;
      double (&K)[NK][NK + 1] = sK[wib];
      double (&U)[NK][NK + 1] = sU[wib];
      int rowmap[MC];
      {
        int a = 0;
#pragma unroll
        for (int i = 0; i < MC; ++i) if (act >> i & 1u) rowmap[a++] = i;
      }
      double rhs_r = 0.0;  // this lane's rhs entry
      if (lane < nk) {
        for (int cidx = 0; cidx < nk; ++cidx) {
          double v;
          if (lane < NV) {
            if (cidx < NV) v = (lane == cidx) ? ((lane >= J ? 2.0 : 0.0) + reg) : 0.0;
            else v = A[rowmap[cidx - NV]][lane];
          } else {
            const int r = rowmap[lane - NV];
            v = cidx < NV ? A[r][cidx] : ((cidx == lane) ? -reg : 0.0);
          }
          K[lane][cidx] = v;
          U[lane][cidx] = v;
        }
        if (lane >= NV) {
          const int r = rowmap[lane - NV];
          rhs_r = (atlo >> r & 1u) ? lo_[r] : hi_[r];
        }
      }
      __syncwarp();
      // LU with partial pivoting; perm[r] tracked per lane as the original row now in slot r
      int perm = lane;
      bool singular = false;
      for (int cc = 0; cc < nk; ++cc) {
        double val = (lane >= cc && lane < nk) ? fabs(U[lane][cc]) : -1.0;
        int idx = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, val, off);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
          if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
        }
        const int piv = idx;
        if (val == 0.0) singular = true;
        if (piv != cc) {
          for (int t = lane; t < nk; t += 32) {
            const double tmp = U[cc][t];
            U[cc][t] = U[piv][t];
            U[piv][t] = tmp;
          }
          const int pc = __shfl_sync(0xffffffffu, perm, cc), pp = __shfl_sync(0xffffffffu, perm, piv);
          if (lane == cc) perm = pp;
          if (lane == piv) perm = pc;
        }
        __syncwarp();
        if (lane > cc && lane < nk && !singular) {
          const double l = U[lane][cc] / U[cc][cc];
          U[lane][cc] = l;
          for (int t = cc + 1; t < nk; ++t) U[lane][t] = __fma_rn(-l, U[cc][t], U[lane][t]);
        }
        __syncwarp();
      }
      if (!singular) {
        // solve K w = rhs with the factors; then two refinement steps on the residual
        auto lu_solve = [&](double bvec) -> double {
          // bvec: this lane's entry of the right-hand side (original row order)
          double yv = __shfl_sync(0xffffffffu, bvec, perm);  // apply the row permutation
          for (int cc = 0; cc < nk; ++cc) {
            const double yc = __shfl_sync(0xffffffffu, yv, cc);
            if (lane > cc && lane < nk) yv = __fma_rn(-U[lane][cc], yc, yv);
          }
          for (int cc = nk - 1; cc >= 0; --cc) {
            double wc = 0.0;
            if (lane == cc) yv = yv / U[cc][cc];
            wc = __shfl_sync(0xffffffffu, yv, cc);
            if (lane < cc) yv = __fma_rn(-U[lane][cc], wc, yv);
          }
          return yv;
        };
        double wv = lu_solve(rhs_r);
        for (int rep = 0; rep < 2; ++rep) {
          double kw = 0.0;
          for (int t = 0; t < nk; ++t) {
            const double wt = __shfl_sync(0xffffffffu, wv, t);
            if (lane < nk) kw = __fma_rn(K[lane][t], wt, kw);
          }
          const double r = lane < nk ? __dsub_rn(rhs_r, kw) : 0.0;
          const double dw = lu_solve(r);
          wv = __dadd_rn(wv, dw);
        }
        // candidate x_pol, y_pol and acceptance (qpsolver.py:271-279)
        double xp[NV], yp[MC];
#pragma unroll
        for (int i = 0; i < NV; ++i) xp[i] = __shfl_sync(0xffffffffu, wv, i);
#pragma unroll
        for (int i = 0; i < MC; ++i) yp[i] = 0.0;
        for (int a = 0; a < k; ++a) {
          const double ya = __shfl_sync(0xffffffffu, wv, NV + a);
#pragma unroll
          for (int i = 0; i < MC; ++i) if (rowmap[a] == i) yp[i] = ya;
        }
        double up_v = 0.0, lo_v = 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) {
          double zi = 0.0;
#pragma unroll
          for (int q = 0; q < NV; ++q) zi = __fma_rn(A[i][q], xp[q], zi);
          up_v = fmax(up_v, fmax(__dsub_rn(zi, hi_[i]), 0.0));
          lo_v = fmax(lo_v, fmax(__dsub_rn(lo_[i], zi), 0.0));
        }
        const double rpp = __dadd_rn(up_v, lo_v);
        double rdp = 0.0;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          double acc = q >= J ? __dmul_rn(2.0, xp[q]) : 0.0;
#pragma unroll
          for (int i = 0; i < MC; ++i) acc = __fma_rn(A[i][q], yp[i], acc);
          rdp = fmax(rdp, fabs(acc));
        }
        if (fmax(rpp, rdp) < fmax(rp, rd)) {
#pragma unroll
          for (int i = 0; i < NV; ++i) x[i] = xp[i];
        }
      }
    }
  }
  if (lane == 0) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) s = __fma_rn(x[J + c], x[J + c], s);
    const double dl = sqrt(s);
    delta_out[inst] = dl;
    safe_out[inst] = (uint8_t)(status == BZG_SOLVED && dl > eps_cut);
#pragma unroll
    for (int i = 0; i < NV; ++i) x_io[inst * NV + i] = x[i];
  }
}

// ------------------------------------------------------------------ aggregation
__global__ void k_qp_verdicts(const unsigned long long* __restrict__ pend, long long n_inst,
                              const uint8_t* __restrict__ safe, int* __restrict__ qp_kill,
                              uint8_t* __restrict__ qp_saved, unsigned long long* __restrict__ counters) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned s = 0, u = 0;
  if (t < n_inst) {
    const unsigned long long pk = pend[t];
    const long long e = (long long)(pk >> 20);
    const int o = (int)(pk & 0xFFFFF);
    if (safe[t]) { qp_saved[e] = 1; s = 1; }
    else { atomicMin(qp_kill + e, o); u = 1; }
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long ts = BR(tmp).Sum((unsigned long long)s);
  __syncthreads();
  unsigned long long tu = BR(tmp).Sum((unsigned long long)u);
  if (threadIdx.x == 0) {
    if (ts) atomicAdd(counters + 3, ts);
    if (tu) atomicAdd(counters + 4, tu);
  }
}

// alive / provenance from the first killing obstacle (graph.py:316-340)
__global__ void k_mask_finalize(long long E, int n_obs, const int* __restrict__ first_kill,
                                const int* __restrict__ qp_kill, const uint8_t* __restrict__ qp_saved,
                                uint8_t* __restrict__ alive, uint8_t* __restrict__ prov) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int kh = first_kill[e], kq = qp_kill[e];
  const bool dead = kh < n_obs || kq < n_obs;
  alive[e] = dead ? 0 : 1;
  uint8_t p;
  if (dead) p = kh < kq ? BZG_HEURISTIC_UNSAFE : BZG_QP_UNSAFE;
  else p = qp_saved[e] ? BZG_QP_SAFE : BZG_HEURISTIC_SAFE;
  prov[e] = p;
}

__global__ void k_unpack_pend(const unsigned long long* __restrict__ pend, long long n, long long* __restrict__ e,
                              int* __restrict__ o) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  e[t] = (long long)(pend[t] >> 20);
  o[t] = (int)(pend[t] & 0xFFFFF);
}

__global__ void k_fill_int(int* p, long long n, int v) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < n) p[t] = v;
}

template <typename F>
void dispatch_cut(int G, int M, F&& f) {
#define BZG_GM(g, m) \
  if (G == g && M == m) { f(std::integral_constant<int, g>{}, std::integral_constant<int, m>{}); return; }
  BZG_GM(1, 1) BZG_GM(1, 2) BZG_GM(1, 3) BZG_GM(2, 1) BZG_GM(2, 2) BZG_GM(2, 3)
  BZG_GM(3, 1) BZG_GM(3, 2) BZG_GM(3, 3)
#undef BZG_GM
  throw Error(BZG_EUNSUPPORTED, "device cut supports gamma in 1..3 and m in 1..3");
}

}  // namespace

void cut_graph(Ctx* c, Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
               const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
               Mask* mk) {
  const long long E = g->E;
  const int m = g->m;
  BZG_REQUIRE(n_obs >= 0 && n_obs < (1 << 20), BZG_EINVAL, "obstacle count out of range");
  BZG_REQUIRE(E < (1ll << 43), BZG_EUNSUPPORTED, "edge count too large for the QP work list");
  for (int o = 0; o < n_obs; ++o) {
    BZG_REQUIRE(is_box[o], BZG_EUNSUPPORTED,
                "obstacle " + std::to_string(o) + " is not an axis-aligned box: the general-polytope "
                "heuristic (graph.py:202-221) is not implemented on device");
    BZG_REQUIRE(row_off[o + 1] - row_off[o] == 2 * m, BZG_EINVAL, "box obstacle must have 2m rows");
  }
  mk->g = g;
  mk->E = E;
  mk->n_obs = n_obs;
  mk->alive.alloc(std::max(E, 1ll), c->stream);
  mk->prov.alloc(std::max(E, 1ll), c->stream);
  for (int i = 0; i < 6; ++i) mk->counters[i] = 0;
  mk->counters[0] = E * (long long)n_obs;
  mk->tree_v0 = -1;
  mk->reach_vg = -1;
  mk->n_qp = 0;

  DParams dp{};
  for (size_t k = 0; k < g->D.size(); ++k) dp.D[k] = g->D[k];
  dispatch_cut(g->gamma, m, [&](auto G_, auto M_) {
    constexpr int Gc = decltype(G_)::value, Mc = decltype(M_)::value;
    using Rec = ObsRec<Mc>;
    std::vector<Rec> h(std::max(n_obs, 1));
    for (int o = 0; o < n_obs; ++o) {
      Rec& r = h[o];
      for (int q = 0; q < 2 * Mc; ++q) {
        const int row = row_off[o] + q;
        for (int k = 0; k < Mc; ++k) r.A[q][k] = A[(size_t)row * Mc + k];
        r.b[q] = b[row];
        r.b_eps[q] = b[row] + cfg->eps_geo;  // O.b + eps_geo (graph.py:234)
      }
      for (int k = 0; k < Mc; ++k) {
        r.lo[k] = box_lo[(size_t)o * Mc + k];
        r.hi[k] = box_hi[(size_t)o * Mc + k];
      }
    }
    DevBuf d_obs, d_kill, d_qkill, d_saved, d_cnt;
    d_obs.alloc(sizeof(Rec) * h.size(), c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_obs.ptr, h.data(), sizeof(Rec) * h.size(), cudaMemcpyHostToDevice, c->stream));
    d_kill.alloc(std::max(E, 1ll) * sizeof(int), c->stream);
    d_qkill.alloc(std::max(E, 1ll) * sizeof(int), c->stream);
    d_saved.alloc(std::max(E, 1ll), c->stream);
    d_cnt.alloc(8 * sizeof(unsigned long long), c->stream);
    BZG_CHECK_CUDA(cudaMemsetAsync(d_cnt.ptr, 0, 8 * sizeof(unsigned long long), c->stream));
    BZG_CHECK_CUDA(cudaMemsetAsync(d_saved.ptr, 0, std::max(E, 1ll), c->stream));
    launch(c, "k_fill_int", k_fill_int, dim3(div_up(E, 256)), dim3(256), 0, d_kill.as<int>(), E, n_obs);
    launch(c, "k_fill_int", k_fill_int, dim3(div_up(E, 256)), dim3(256), 0, d_qkill.as<int>(), E, n_obs);

    // ---- heuristic screen (obstacle chunks sized to shared memory)
    unsigned long long cap = (unsigned long long)std::max<long long>(1 << 20, E * (long long)n_obs / 32);
    DevBuf d_pend;
    unsigned long long* hcnt = static_cast<unsigned long long*>(c->host_scratch(8 * sizeof(unsigned long long)));
    const int chunk = std::max(1, (int)(96 * 1024 / sizeof(Rec)));
    for (int attempt = 0; attempt < 2; ++attempt) {
      d_pend.alloc(cap * sizeof(unsigned long long), c->stream);
      for (int o0 = 0; o0 < n_obs; o0 += chunk) {
        const int o1 = std::min(n_obs, o0 + chunk);
        const size_t smem = sizeof(Rec) * (o1 - o0);
        auto kern = k_cut_heuristic<Gc, Mc>;
        BZG_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        launch(c, "k_cut_heuristic", kern, dim3(div_up(E, 256)), dim3(256), smem, dp, g->vertices.as<double>(), E,
               g->src.as<int>(), g->dst.as<int>(), d_obs.as<Rec>(), o0, o1, cfg->heur_margin, d_kill.as<int>(),
               d_cnt.as<unsigned long long>(), d_cnt.as<unsigned long long>() + 5, cap,
               d_pend.as<unsigned long long>());
      }
      BZG_CHECK_CUDA(cudaMemcpyAsync(hcnt, d_cnt.ptr, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
      BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
      if (hcnt[5] <= cap) break;
      // work list overflowed: grow it and rerun the screen from a clean state
      cap = hcnt[5] + 1024;
      BZG_CHECK_CUDA(cudaMemsetAsync(d_cnt.ptr, 0, 8 * sizeof(unsigned long long), c->stream));
      launch(c, "k_fill_int", k_fill_int, dim3(div_up(E, 256)), dim3(256), 0, d_kill.as<int>(), E, n_obs);
    }
    const long long n_inst = (long long)hcnt[5];
    mk->counters[1] = (long long)hcnt[0];
    mk->counters[2] = (long long)hcnt[1];
    mk->counters[3] = (long long)hcnt[2];

    // ---- QP fallback on every indeterminate pair (graph.py:320-337)
    mk->n_qp = n_inst;
    if (n_inst > 0) {
      constexpr int NV = 2 * Gc + 2 * Mc;
      mk->qp_status.alloc(n_inst, c->stream);
      mk->qp_iters.alloc(n_inst * sizeof(int), c->stream);
      mk->qp_delta.alloc(n_inst * sizeof(double), c->stream);
      DevBuf d_x, d_res, d_safe, d_next;
      d_x.alloc(n_inst * NV * sizeof(double), c->stream);
      d_res.alloc(n_inst * 2 * sizeof(double), c->stream);
      d_safe.alloc(n_inst, c->stream);
      d_next.alloc(sizeof(unsigned long long), c->stream);
      BZG_CHECK_CUDA(cudaMemsetAsync(d_next.ptr, 0, sizeof(unsigned long long), c->stream));
      QpParams qp{};
      qp.rho = cfg->qp_rho;
      qp.rho_eq = cfg->qp_rho * 1e3;  // equality rows (qpsolver.py:100-103, 137)
      qp.sigma = cfg->qp_sigma;
      qp.alpha = cfg->qp_alpha;
      qp.one_m_alpha = 1.0 - cfg->qp_alpha;
      qp.eps_abs = cfg->qp_eps_abs;
      qp.eps_rel = cfg->qp_eps_rel;
      qp.eps_pinf = cfg->qp_eps_pinf;
      qp.max_iter = cfg->qp_max_iter;
      // persistent grid: enough resident warps to cover the SMs several times
      const long long blocks = std::min<long long>(div_up(n_inst, 128), (long long)c->num_sms * 16);
      launch(c, "k_qp_admm", k_qp_admm<Gc, Mc>, dim3((unsigned)blocks), dim3(128), 0, qp, dp,
             g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(), d_obs.as<Rec>(),
             d_pend.as<unsigned long long>(), n_inst, d_next.as<unsigned long long>(), mk->qp_status.as<int8_t>(),
             mk->qp_iters.as<int>(), d_x.as<double>(), d_res.as<double>());
      launch(c, "k_qp_polish", k_qp_polish<Gc, Mc>, dim3(div_up(n_inst, kPolishWarps)), dim3(32 * kPolishWarps), 0,
             dp, g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(), d_obs.as<Rec>(),
             d_pend.as<unsigned long long>(), n_inst, (int)cfg->qp_polish, cfg->eps_cut,
             mk->qp_status.as<int8_t>(), d_x.as<double>(), d_res.as<double>(), mk->qp_delta.as<double>(),
             d_safe.as<uint8_t>());
      launch(c, "k_qp_verdicts", k_qp_verdicts, dim3(div_up(n_inst, 256)), dim3(256), 0,
             d_pend.as<unsigned long long>(), n_inst, d_safe.as<uint8_t>(), d_qkill.as<int>(), d_saved.as<uint8_t>(),
             d_cnt.as<unsigned long long>());
      mk->qp_edge.alloc(n_inst * sizeof(long long), c->stream);
      mk->qp_obs.alloc(n_inst * sizeof(int), c->stream);
      launch(c, "k_unpack_pend", k_unpack_pend, dim3(div_up(n_inst, 256)), dim3(256), 0,
             d_pend.as<unsigned long long>(), n_inst, mk->qp_edge.as<long long>(), mk->qp_obs.as<int>());
    }
    launch(c, "k_mask_finalize", k_mask_finalize, dim3(div_up(E, 256)), dim3(256), 0, E, n_obs, d_kill.as<int>(),
           d_qkill.as<int>(), d_saved.as<uint8_t>(), mk->alive.as<uint8_t>(), mk->prov.as<uint8_t>());
    BZG_CHECK_CUDA(cudaMemcpyAsync(hcnt, d_cnt.ptr, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
    mk->counters[4] = (long long)hcnt[3];
    mk->counters[5] = (long long)hcnt[4];
  });
}

}  // namespace bzg
