// Batched Cut-QP on device: dense ADMM (one thread per instance) and active-set polish
// (one warp per instance).  Included by k_cut.cu.
//
// Problem (reference graph.py:268-282, _cut_qp_problem), per (edge, obstacle):
//   x = [lambda (J); delta (C)],  min delta' delta
//   s.t.  Q lambda - delta <= b  (C rows, Q = A_O P),  lambda >= 0 (J rows),  sum lambda = 1
// solved by the dense ADMM of qpsolver.py:129-233 and polished by qpsolver.py:236-279.
#pragma once

namespace bzg {
namespace {

struct QpParams {
  double rho, rho_eq, sigma, alpha, one_m_alpha, eps_abs, eps_rel, eps_pinf;
  int max_iter;
};

// Q = A_O @ points (graph.py:276): BLAS product, FMA chain over the m output dimensions.
template <int G, int M>
__device__ __forceinline__ void cut_q_matrix(const ObsRec<M>& o, const double (&P)[M][2 * G], double (&Q)[2 * M][2 * G]) {
#pragma unroll
  for (int c = 0; c < 2 * M; ++c)
#pragma unroll
    for (int j = 0; j < 2 * G; ++j) {
      double acc = __dmul_rn(o.A[c][0], P[0][j]);
#pragma unroll
      for (int k = 1; k < M; ++k) acc = __fma_rn(o.A[c][k], P[k][j], acc);
      Q[c][j] = acc;
    }
}

template <int G, int M>
__device__ __forceinline__ void load_instance(const DParams& dp, const double* __restrict__ Vx,
                                              const int* __restrict__ src, const int* __restrict__ dst,
                                              const ObsRec<M>* __restrict__ obs, unsigned long long pk,
                                              double (&Q)[2 * M][2 * G], double (&b)[2 * M]) {
  constexpr int N = G * M;
  const long long e = (long long)(pk >> 20);
  const ObsRec<M>& o = obs[(int)(pk & 0xFFFFF)];
  double xi[N], xj[N], P[M][2 * G];
  const long long a = src[e], c = dst[e];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    xi[k] = Vx[a * N + k];
    xj[k] = Vx[c * N + k];
  }
  control_points<G, M>(xi, xj, dp.D, P);
  cut_q_matrix<G, M>(o, P, Q);
#pragma unroll
  for (int k = 0; k < 2 * M; ++k) b[k] = o.b[k];
}

// ----------------------------------------------------------------------------- ADMM
// The reference forms the (n+mc)^2 KKT matrix [[P + sigma I, A'], [A, -R^-1]] per
// instance, inverts it (np.linalg.inv) and applies the inverse every iteration.  The
// same step is xt = M^-1 (sigma x - q + A'(R z - y)), zt = A xt with
// M = P + sigma I + A'RA; for the cut QP the delta block of M is (2 + sigma + rho) I,
// so its Schur complement leaves one J x J SPD matrix
//   S = (sigma + rho) I + (rho - rho^2/kdd) Q'Q + rho_eq 11',   kdd = 2 + sigma + rho,
// whose inverse is formed once per instance.  Termination (rp <= eps_p, rd <= eps_d),
// the primal-infeasibility certificate and MAX_ITER follow qpsolver.py:179-231.
template <int G, int M>
__global__ void __launch_bounds__(128) k_qp_admm(QpParams qp, DParams dp, const double* __restrict__ Vx,
                                                 const int* __restrict__ src, const int* __restrict__ dst,
                                                 const ObsRec<M>* __restrict__ obs,
                                                 const unsigned long long* __restrict__ pend, long long n_inst,
                                                 unsigned long long* __restrict__ next, int8_t* __restrict__ st_out,
                                                 int* __restrict__ it_out, double* __restrict__ x_out,
                                                 double* __restrict__ res_out) {
  constexpr int J = 2 * G, C = 2 * M, NV = J + C;
  const int lane = threadIdx.x & 31;
  const double rho = qp.rho, req = qp.rho_eq, ri = 1.0 / qp.rho;
  const double sig = qp.sigma, al = qp.alpha, oma = qp.one_m_alpha;
  const double kdd = 2.0 + sig + rho, ikdd = 1.0 / kdd, kp = rho * ikdd;
  const bool rel = qp.eps_rel != 0.0;

  long long inst = -1;  // -1 needs work, -2 exhausted
  int it = 0;
  double Q[C][J], Si[J * (J + 1) / 2], b[C];
  double lam[J], del[C], zc[C], zl[J], ze = 0.0, yc[C], yl[J], ye = 0.0;
  auto S = [&](int r, int s) -> double& { return r >= s ? Si[r * (r + 1) / 2 + s] : Si[s * (s + 1) / 2 + r]; };

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
          load_instance<G, M>(dp, Vx, src, dst, obs, pend[my], Q, b);
          // S = (sig + rho) I + kap Q'Q + req 11'; Cholesky L L', then Si = L^-T L^-1
          const double kap = rho - rho * rho * ikdd;
          double L[J][J];
#pragma unroll
          for (int r = 0; r < J; ++r)
#pragma unroll
            for (int s = 0; s <= r; ++s) {
              double qq = 0.0;
#pragma unroll
              for (int c = 0; c < C; ++c) qq = __fma_rn(Q[c][r], Q[c][s], qq);
              L[r][s] = kap * qq + req + (r == s ? sig + rho : 0.0);
            }
          double dinv[J];
#pragma unroll
          for (int r = 0; r < J; ++r) {
#pragma unroll
            for (int s = 0; s < r; ++s) {
              double t = L[r][s];
#pragma unroll
              for (int k = 0; k < s; ++k) t = __fma_rn(-L[r][k], L[s][k], t);
              L[r][s] = t * dinv[s];
            }
            double d = L[r][r];
#pragma unroll
            for (int k = 0; k < r; ++k) d = __fma_rn(-L[r][k], L[r][k], d);
            L[r][r] = sqrt(d);
            dinv[r] = 1.0 / L[r][r];
          }
          // W = L^-1 (lower), then Si = W' W
          double Wm[J][J];
#pragma unroll
          for (int r = 0; r < J; ++r) {
#pragma unroll
            for (int s = 0; s < J; ++s) Wm[r][s] = 0.0;
            Wm[r][r] = dinv[r];
#pragma unroll
            for (int s = 0; s < r; ++s) {
              double t = 0.0;
#pragma unroll
              for (int k = s; k < r; ++k) t = __fma_rn(L[r][k], Wm[k][s], t);
              Wm[r][s] = -t * dinv[r];
            }
          }
#pragma unroll
          for (int r = 0; r < J; ++r)
#pragma unroll
            for (int s = 0; s <= r; ++s) {
              double t = 0.0;
#pragma unroll
              for (int k = r; k < J; ++k) t = __fma_rn(Wm[k][r], Wm[k][s], t);
              S(r, s) = t;
            }
#pragma unroll
          for (int j = 0; j < J; ++j) { lam[j] = 0.0; zl[j] = 0.0; yl[j] = 0.0; }
#pragma unroll
          for (int c = 0; c < C; ++c) { del[c] = 0.0; zc[c] = 0.0; yc[c] = 0.0; }
          ze = 0.0;
          ye = 0.0;
          it = 0;
        }
      }
    }
    if (__all_sync(0xffffffffu, inst == -2)) break;
    if (inst < 0) continue;

    // ---- one ADMM iteration (qpsolver.py:164-174) in the reduced form
    ++it;
    double rdel[C], tC[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double wc = __fma_rn(rho, zc[c], -yc[c]);  // (R z - y)_c
      rdel[c] = __fma_rn(sig, del[c], -wc);          // sigma delta - w_c
      tC[c] = __fma_rn(kp, rdel[c], wc);
    }
    const double we = __fma_rn(req, ze, -ye);
    double rp_[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double acc = __fma_rn(sig, lam[j], __fma_rn(rho, zl[j], -yl[j]) + we);
#pragma unroll
      for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], tC[c], acc);
      rp_[j] = acc;
    }
    double a[J];
#pragma unroll
    for (int r = 0; r < J; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int s = 0; s < J; ++s) acc = __fma_rn(S(r, s), rp_[s], acc);
      a[r] = acc;
    }
    // relaxation, projection and dual update, row block by row block
    double dmax = 0.0;  // max |dy|
    bool sign_ok = true;  // certificate needs dy_c >= 0 (u finite) and dy_l <= 0 (l finite)
    double dyc[C], dyl[J];
    double rprim = 0.0, maxAx = 0.0, maxz = 0.0;
    double sa = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      sa += a[j];
      const double zr = __dadd_rn(__dmul_rn(al, a[j]), __dmul_rn(oma, zl[j]));
      const double zn = fmax(__dadd_rn(zr, __dmul_rn(ri, yl[j])), 0.0);
      const double yn = __dadd_rn(yl[j], __dmul_rn(rho, __dsub_rn(zr, zn)));
      dyl[j] = __dsub_rn(yn, yl[j]);
      sign_ok = sign_ok && !(dyl[j] > 0.0);
      dmax = fmax(dmax, fabs(dyl[j]));
      lam[j] = __dadd_rn(__dmul_rn(al, a[j]), __dmul_rn(oma, lam[j]));
      zl[j] = zn;
      yl[j] = yn;
      rprim = fmax(rprim, fabs(__dsub_rn(lam[j], zn)));
      if (rel) { maxAx = fmax(maxAx, fabs(lam[j])); maxz = fmax(maxz, fabs(zn)); }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double qa = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) qa = __fma_rn(Q[c][j], a[j], qa);
      const double d = __fma_rn(rdel[c], ikdd, kp * qa);
      const double zt = __dsub_rn(qa, d);
      const double zr = __dadd_rn(__dmul_rn(al, zt), __dmul_rn(oma, zc[c]));
      const double zn = fmin(__dadd_rn(zr, __dmul_rn(ri, yc[c])), b[c]);
      const double yn = __dadd_rn(yc[c], __dmul_rn(rho, __dsub_rn(zr, zn)));
      dyc[c] = __dsub_rn(yn, yc[c]);
      sign_ok = sign_ok && !(dyc[c] < 0.0);
      dmax = fmax(dmax, fabs(dyc[c]));
      del[c] = __dadd_rn(__dmul_rn(al, d), __dmul_rn(oma, del[c]));
      zc[c] = zn;
      yc[c] = yn;
    }
    double dye;
    {
      const double zr = __dadd_rn(__dmul_rn(al, sa), __dmul_rn(oma, ze));
      const double zn = 1.0;  // clip to [1, 1]
      const double yn = __dadd_rn(ye, __dmul_rn(req, __dsub_rn(zr, zn)));
      dye = __dsub_rn(yn, ye);
      dmax = fmax(dmax, fabs(dye));
      ze = zn;
      ye = yn;
    }
    // residuals at the new iterate (qpsolver.py:176-186)
    double sl = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) sl = __dadd_rn(sl, lam[j]);
    rprim = fmax(rprim, fabs(__dsub_rn(sl, 1.0)));
    if (rel) { maxAx = fmax(maxAx, fabs(sl)); maxz = fmax(maxz, 1.0); }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) acc = __fma_rn(Q[c][j], lam[j], acc);
      const double ax = __dsub_rn(acc, del[c]);
      rprim = fmax(rprim, fabs(__dsub_rn(ax, zc[c])));
      if (rel) { maxAx = fmax(maxAx, fabs(ax)); maxz = fmax(maxz, fabs(zc[c])); }
    }
    double rdual = 0.0, maxPx = 0.0, maxATy = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double acc = __dadd_rn(yl[j], ye);
#pragma unroll
      for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], yc[c], acc);
      rdual = fmax(rdual, fabs(acc));
      maxATy = fmax(maxATy, fabs(acc));
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double px = __dmul_rn(2.0, del[c]);
      rdual = fmax(rdual, fabs(__dsub_rn(px, yc[c])));
      if (rel) { maxPx = fmax(maxPx, fabs(px)); maxATy = fmax(maxATy, fabs(yc[c])); }
    }
    const double eps_p = rel ? qp.eps_abs + qp.eps_rel * fmax(maxAx, maxz) : qp.eps_abs;
    const double eps_d = rel ? qp.eps_abs + qp.eps_rel * fmax(maxPx, maxATy) : qp.eps_abs;
    int status = -1;
    if (rprim <= eps_p && rdual <= eps_d) {
      status = BZG_SOLVED;
    } else if (sign_ok && dmax > 1e-13) {
      // primal-infeasibility certificate (qpsolver.py:193-209): reachable only when every
      // dy_i multiplies a finite bound, so support = sum_c b_c dy_c + dy_eq
      double atd = 0.0, supp = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        double acc = __dadd_rn(dyl[j], dye);
#pragma unroll
        for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], dyc[c], acc);
        atd = fmax(atd, fabs(acc));
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        atd = fmax(atd, fabs(dyc[c]));
        supp = __dadd_rn(supp, __dmul_rn(b[c], dyc[c]));
      }
      supp = __dadd_rn(supp, dye);
      if (atd <= qp.eps_pinf * dmax && supp <= -qp.eps_pinf * dmax) status = BZG_INFEASIBLE;
    }
    if (status < 0 && it >= qp.max_iter) status = BZG_MAX_ITER;
    if (status >= 0) {
      st_out[inst] = (int8_t)status;
      it_out[inst] = it;
#pragma unroll
      for (int j = 0; j < J; ++j) x_out[inst * NV + j] = lam[j];
#pragma unroll
      for (int c = 0; c < C; ++c) x_out[inst * NV + J + c] = del[c];
      res_out[inst * 2 + 0] = rprim;
      res_out[inst * 2 + 1] = rdual;
      inst = -1;
    }
  }
}

// ----------------------------------------------------------------------------- polish
// Active-set polish (qpsolver.py:236-279), one warp per SOLVED instance (MAX_ITER and
// INFEASIBLE instances are unsafe whatever their x, graph.py:329, so their polish cannot
// change a verdict and is skipped).  Lane r holds row r of the regularised reduced KKT
// matrix K = [[P + dI, G'], [G, -dI]] in registers; inactive constraint slots are
// decoupled identity rows, which leaves partial pivoting and the arithmetic on the
// active block unchanged.  LU with partial pivoting (pivot = first max |.|, reciprocal
// scaling as LAPACK dgetf2), forward/back substitution, two refinement steps, then the
// acceptance test max(rp', rd') < max(rp, rd) and ||delta|| > eps_cut.
// Verdict from the ADMM iterate and the polish work list.  The polish only changes x,
// never the status (qpsolver.py:301-303), and the verdict is SOLVED and ||delta|| > eps_cut
// (graph.py:329): MAX_ITER / INFEASIBLE instances are unsafe whatever x, and a SOLVED
// instance whose ADMM ||delta|| is at least `screen` cannot drop below eps_cut when
// polished (both iterates are 1e-7-feasible, the ADMM
// one is 1e-7-KKT with exact complementarity, so both norms are within ~1e-3 of the
// optimal ||delta*||).  screen <= 0 polishes every SOLVED instance, as the reference does.
__global__ void k_qp_select(long long n_inst, int nv, int j0, int polish, double screen, double eps_cut,
                            const int8_t* __restrict__ st, const double* __restrict__ x,
                            double* __restrict__ delta_out, uint8_t* __restrict__ safe_out, int* __restrict__ list,
                            unsigned long long* __restrict__ n_list) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool need = false;
  if (t < n_inst) {
    double s = 0.0;
    for (int c = j0; c < nv; ++c) s = __fma_rn(x[t * nv + c], x[t * nv + c], s);
    const double dl = sqrt(s);
    const bool solved = st[t] == BZG_SOLVED;
    delta_out[t] = dl;
    safe_out[t] = (uint8_t)(solved && dl > eps_cut);
    need = polish && solved && (screen <= 0.0 || dl < screen);
  }
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (m) {
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(n_list, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (need) list[base + __popc(m & ((1u << lane) - 1u))] = (int)t;
  }
}

constexpr int kPolishWarps = 4;

template <int G, int M>
__global__ void __launch_bounds__(32 * kPolishWarps) k_qp_polish(
    DParams dp, const double* __restrict__ Vx, const int* __restrict__ src, const int* __restrict__ dst,
    const ObsRec<M>* __restrict__ obs, const unsigned long long* __restrict__ pend, const int* __restrict__ list,
    long long n_list, double eps_cut, double* __restrict__ x_io, const double* __restrict__ res,
    double* __restrict__ delta_out, uint8_t* __restrict__ safe_out) {
  constexpr int J = 2 * G, C = 2 * M, NV = J + C, MC = C + J + 1, NK = NV + MC;
  static_assert(NK <= 32, "polish system must fit a warp");
  // U[t][r]: column-major LU factors, lane r owns row r (conflict-free column access)
  __shared__ double sU[kPolishWarps][NK][32];
  __shared__ double sQ[kPolishWarps][C][J];
  __shared__ double sB[kPolishWarps][C];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long li = (long long)blockIdx.x * kPolishWarps + wib;
  if (li >= n_list) return;
  const long long inst = list[li];  // a SOLVED instance selected by k_qp_select
  const int status = BZG_SOLVED;
  // lane t < NV holds x_t
  double xv = lane < NV ? x_io[inst * NV + lane] : 0.0;
  {
    const double rp = res[inst * 2], rd = res[inst * 2 + 1];
    if (lane == 0) {
      double Q[C][J], b[C];
      load_instance<G, M>(dp, Vx, src, dst, obs, pend[inst], Q, b);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        sB[wib][c] = b[c];
#pragma unroll
        for (int j = 0; j < J; ++j) sQ[wib][c][j] = Q[c][j];
      }
    }
    __syncwarp();
    double (&U)[NK][32] = sU[wib];
    // constraint row i of A (graph.py:275-281) at column t
    auto Aent = [&](int i, int t) -> double {
      if (i < C) return t < J ? sQ[wib][i][t] : (t - J == i ? -1.0 : 0.0);
      if (i < C + J) return t == i - C ? 1.0 : 0.0;
      return t < J ? 1.0 : 0.0;
    };
    auto lo_of = [&](int i) -> double { return i < C ? -INFINITY : (i < C + J ? 0.0 : 1.0); };
    auto hi_of = [&](int i) -> double { return i < C ? sB[wib][i] : (i < C + J ? INFINITY : 1.0); };
    // active set at z = A x (qpsolver.py:245-249); lane i evaluates constraint row i
    const double tol = fmax(1e-7, 10.0 * rp);
    bool l_act = false, u_act = false;
    {
      double zi = 0.0;
      for (int t = 0; t < NV; ++t) {
        const double xt = __shfl_sync(0xffffffffu, xv, t);
        if (lane < MC) zi = __fma_rn(Aent(lane, t), xt, zi);
      }
      if (lane < MC) {
        l_act = __dsub_rn(zi, lo_of(lane)) <= tol;
        u_act = __dsub_rn(hi_of(lane), zi) <= tol;
      }
    }
    const unsigned act = __ballot_sync(0xffffffffu, lane < MC && (l_act || u_act));
    const unsigned atlo = __ballot_sync(0xffffffffu, lane < MC && l_act);
    if (act) {
      const double reg = 1e-8;
      // K = [[P + reg I, G'], [G, -reg I]] with inactive constraint slots as identity rows
      auto Kent = [&](int r, int t) -> double {
        if (r < NV) {
          if (t < NV) return r == t ? (r >= J ? 2.0 : 0.0) + reg : 0.0;
          return (act >> (t - NV) & 1u) ? Aent(t - NV, r) : 0.0;
        }
        const int i = r - NV;
        if (act >> i & 1u) return t < NV ? Aent(i, t) : (t == r ? -reg : 0.0);
        return t == r ? 1.0 : 0.0;
      };
      for (int t = 0; t < NK; ++t) U[t][lane] = lane < NK ? Kent(lane, t) : 0.0;
      double rhs = 0.0;
      if (lane >= NV && lane < NK) {
        const int i = lane - NV;
        if (act >> i & 1u) rhs = (atlo >> i & 1u) ? lo_of(i) : hi_of(i);
      }
      __syncwarp();
      // LU with partial pivoting (first max |.| on ties; reciprocal scaling as dgetf2)
      int perm = lane;
      bool singular = false;
      for (int cc = 0; cc < NK; ++cc) {
        double v = (lane >= cc && lane < NK) ? fabs(U[cc][lane]) : -1.0;
        int idx = lane;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, off);
          const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
          if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
        }
        if (v == 0.0) { singular = true; break; }
        if (idx != cc) {
          if (lane < NK) {
            const double tmp = U[lane][cc];
            U[lane][cc] = U[lane][idx];
            U[lane][idx] = tmp;
          }
          const int from = lane == cc ? idx : (lane == idx ? cc : lane);
          perm = __shfl_sync(0xffffffffu, perm, from);
          __syncwarp();
        }
        const double rpv = 1.0 / U[cc][cc];
        if (lane > cc && lane < NK) {
          const double l = __dmul_rn(U[cc][lane], rpv);
          U[cc][lane] = l;
#pragma unroll 4
          for (int t = cc + 1; t < NK; ++t) U[t][lane] = __fma_rn(-l, U[t][cc], U[t][lane]);
        }
        __syncwarp();
      }
      if (!singular) {
        auto lu_solve = [&](double bv) -> double {
          double yv = __shfl_sync(0xffffffffu, bv, perm);
          for (int cc = 0; cc < NK; ++cc) {
            const double yc = __shfl_sync(0xffffffffu, yv, cc);
            if (lane > cc && lane < NK) yv = __fma_rn(-U[cc][lane], yc, yv);
          }
          for (int cc = NK - 1; cc >= 0; --cc) {
            if (lane == cc) yv = yv / U[cc][cc];
            const double wc = __shfl_sync(0xffffffffu, yv, cc);
            if (lane < cc) yv = __fma_rn(-U[cc][lane], wc, yv);
          }
          return yv;
        };
        double w = lu_solve(rhs);
        for (int rep = 0; rep < 2; ++rep) {
          double kw = 0.0;
          for (int t = 0; t < NK; ++t) {
            const double wt = __shfl_sync(0xffffffffu, w, t);
            if (lane < NK) kw = __fma_rn(Kent(lane, t), wt, kw);
          }
          const double r = lane < NK ? __dsub_rn(rhs, kw) : 0.0;
          w = __dadd_rn(w, lu_solve(r));
        }
        // acceptance (qpsolver.py:271-279): lane i < MC evaluates row i of A x_pol,
        // lane t < NV column t of P x_pol + A' y_pol (y_pol,i = w[NV + i] on active rows)
        const double ypi = (lane >= NV && lane < NK && (act >> (lane - NV) & 1u)) ? w : 0.0;
        double zi = 0.0, acc = (lane >= J && lane < NV) ? __dmul_rn(2.0, w) : 0.0;
        for (int t = 0; t < NV; ++t) {
          const double xt = __shfl_sync(0xffffffffu, w, t);
          if (lane < MC) zi = __fma_rn(Aent(lane, t), xt, zi);
        }
        for (int i = 0; i < MC; ++i) {
          const double yi = __shfl_sync(0xffffffffu, ypi, NV + i);
          if (lane < NV) acc = __fma_rn(Aent(i, lane), yi, acc);
        }
        double upv = lane < MC ? fmax(__dsub_rn(zi, hi_of(lane)), 0.0) : 0.0;
        double lov = lane < MC ? fmax(__dsub_rn(lo_of(lane), zi), 0.0) : 0.0;
        double rdt = lane < NV ? fabs(acc) : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          upv = fmax(upv, __shfl_xor_sync(0xffffffffu, upv, off));
          lov = fmax(lov, __shfl_xor_sync(0xffffffffu, lov, off));
          rdt = fmax(rdt, __shfl_xor_sync(0xffffffffu, rdt, off));
        }
        if (fmax(__dadd_rn(upv, lov), rdt) < fmax(rp, rd)) xv = lane < NV ? w : 0.0;
      }
    }
  }
  // ||delta|| over x[J:] and the verdict (graph.py:328-329)
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double dc = __shfl_sync(0xffffffffu, xv, J + c);
    s = __fma_rn(dc, dc, s);
  }
  if (lane == 0) {
    const double dl = sqrt(s);
    delta_out[inst] = dl;
    safe_out[inst] = (uint8_t)(status == BZG_SOLVED && dl > eps_cut);
  }
}

}  // namespace
}  // namespace bzg
