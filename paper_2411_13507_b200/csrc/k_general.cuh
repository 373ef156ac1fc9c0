// General (non-box) convex obstacles: the scalar screen of reference graph.py:202-221
// (cut_heuristic), which _heuristic_batch applies per edge to non-box polytopes
// (graph.py:242-247).  Included by k_cut.cu.  SURVEY.md §8 row a8.
//
//   inside  = O.contains_many(P.T, eps)                           -> UNSAFE
//   y_j     = closest_point(O, P_j)  (geometry.py:202-230: a dense ADMM QP, 20000 iterations,
//             eps 1e-10, polish), d_j = ||y_j - P_j||, anchor = first argmin d_j
//   hp      = adjacent_hyperplane(O, P_anchor) (geometry.py:233-252): deepest face active at
//             the projection (residual <= 1e-7), first row on ties
//   SAFE iff hp.normal @ P - hp.offset > margin for every control point, else INDETERMINATE.
//
// BLAS orders of the small products (measured on the reference host, OpenBLAS 0.3.30
// SkylakeX kernels): gemm (pts @ A.T) is an FMA chain from the first term (m = 2, 3); gemv
// (A @ x) is fma(a0, x0, a1 x1), and fma(a2, x2, fma(a0, x0, a1 x1)) for m = 3; vector @
// matrix (normal @ pts) is fma(a0, x0, a1 x1) (m = 2) / a2 x2 + fma(a0, x0, a1 x1) (m = 3) on
// columns in blocks of four and the FMA chain on the tail columns; the 1-D norm is the FMA
// chain sqrt(fma(v1, v1, v0 v0)) (m = 2, 3).  The ADMM itself agrees with the reference to rounding, so
// this row's parity class is the epsilon band.
#pragma once

namespace bzg {
namespace {

constexpr double kGenEpsAbs = 1e-10, kGenEpsRel = 1e-10, kGenRho = 0.1, kGenSigma = 1e-6, kGenAlpha = 1.6;
constexpr int kGenMaxIter = 20000;

template <int M>
__device__ __forceinline__ double gemv_row(const double* a, const double* x) {  // A_c @ x (gemv order)
  if (M == 2) return __fma_rn(a[0], x[0], __dmul_rn(a[1], x[1]));
  if (M == 3) return __fma_rn(a[2], x[2], __fma_rn(a[0], x[0], __dmul_rn(a[1], x[1])));
  double acc = __dmul_rn(a[0], x[0]);
#pragma unroll
  for (int k = 1; k < M; ++k) acc = __fma_rn(a[k], x[k], acc);
  return acc;
}

// column of vector @ matrix inside a block of four columns (the tail columns take the chain)
template <int M>
__device__ __forceinline__ double vecmat_block(const double* n, const double* p) {
  if (M == 2) return __fma_rn(n[0], p[0], __dmul_rn(n[1], p[1]));
  if (M == 3) return __dadd_rn(__dmul_rn(n[2], p[2]), __fma_rn(n[0], p[0], __dmul_rn(n[1], p[1])));
  double acc = __dmul_rn(n[0], p[0]);
#pragma unroll
  for (int k = 1; k < M; ++k) acc = __fma_rn(n[k], p[k], acc);
  return acc;
}

template <int M>
__device__ __forceinline__ double gemm_row(const double* a, const double* x) {  // FMA chain from the first term
  double acc = __dmul_rn(a[0], x[0]);
#pragma unroll
  for (int k = 1; k < M; ++k) acc = __fma_rn(a[k], x[k], acc);
  return acc;
}

template <int M>
__device__ __forceinline__ double norm1d(const double* v) {  // np.linalg.norm of a 1-D vector
  double s = __dmul_rn(v[0], v[0]);
#pragma unroll
  for (int k = 1; k < M; ++k) s = __fma_rn(v[k], v[k], s);
  return sqrt(s);
}

// closest_point(O, x) (geometry.py:202-230): x when inside, the clamp for boxes, else the
// projection QP.  Returns false when the solver certifies infeasibility (the reference raises).
template <int M, int RC>
__device__ bool closest_point_general(const ObsRec<M, RC>& o, const double (&x)[M], double eps, double (&y)[M]) {
  const int R = (int)o.rows;
  bool inside = true;
  for (int c = 0; c < R; ++c) inside &= gemv_row<M>(o.A[c], x) <= __dadd_rn(o.b[c], eps);
  if (inside || o.is_box != 0.0) {  // x itself, or Box.clamp = np.clip(x, lo, hi) (geometry.py:50-51)
#pragma unroll
    for (int k = 0; k < M; ++k) y[k] = inside ? x[k] : fmin(fmax(x[k], o.lo[k]), o.hi[k]);
    return true;
  }
  // QP: min |y|^2 - 2 x'y  s.t. A y <= b;  P = 2I, q = -2x, l = -inf, u = b, rho = 0.1 on every row
  const double rho = kGenRho, ri = 1.0 / kGenRho, sig = kGenSigma, al = kGenAlpha, oma = 1.0 - kGenAlpha;
  // M = (2 + sigma) I + rho A'A, inverted once (Cholesky, M x M)
  double Mm[M][M], L[M][M];
#pragma unroll
  for (int r = 0; r < M; ++r)
#pragma unroll
    for (int s = 0; s < M; ++s) {
      double acc = 0.0;
      for (int c = 0; c < R; ++c) acc = __fma_rn(o.A[c][r], o.A[c][s], acc);
      Mm[r][s] = rho * acc + (r == s ? 2.0 + sig : 0.0);
    }
#pragma unroll
  for (int r = 0; r < M; ++r) {
#pragma unroll
    for (int s = 0; s < r; ++s) {
      double t = Mm[r][s];
#pragma unroll
      for (int k = 0; k < s; ++k) t -= L[r][k] * L[s][k];
      L[r][s] = t / L[s][s];
    }
    double d = Mm[r][r];
#pragma unroll
    for (int k = 0; k < r; ++k) d -= L[r][k] * L[r][k];
    L[r][r] = sqrt(d);
  }
  double xs[M], z[RC], yv[RC];
#pragma unroll
  for (int k = 0; k < M; ++k) xs[k] = 0.0;
  for (int c = 0; c < RC; ++c) { z[c] = 0.0; yv[c] = 0.0; }
  double qn = 0.0;
#pragma unroll
  for (int k = 0; k < M; ++k) qn = fmax(qn, fabs(2.0 * x[k]));
  int status = BZG_MAX_ITER;
  double rp = 0.0, rd = 0.0;
  for (int it = 1; it <= kGenMaxIter; ++it) {
    double rhs[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double acc = __fma_rn(sig, xs[k], 2.0 * x[k]);
      for (int c = 0; c < R; ++c) acc = __fma_rn(o.A[c][k], __fma_rn(rho, z[c], -yv[c]), acc);
      rhs[k] = acc;
    }
#pragma unroll
    for (int r = 0; r < M; ++r) {  // L L' xt = rhs
      double t = rhs[r];
#pragma unroll
      for (int k = 0; k < r; ++k) t -= L[r][k] * rhs[k];
      rhs[r] = t / L[r][r];
    }
#pragma unroll
    for (int r = M - 1; r >= 0; --r) {
      double t = rhs[r];
#pragma unroll
      for (int k = r + 1; k < M; ++k) t -= L[k][r] * rhs[k];
      rhs[r] = t / L[r][r];
    }
    double xn[M];
#pragma unroll
    for (int k = 0; k < M; ++k) xn[k] = __dadd_rn(__dmul_rn(al, rhs[k]), __dmul_rn(oma, xs[k]));
    double maxAx = 0.0, maxz = 0.0, maxATy = 0.0, maxPx = 0.0;
    double ATy[M], ATdy[M];
#pragma unroll
    for (int k = 0; k < M; ++k) { ATy[k] = 0.0; ATdy[k] = 0.0; }
    double dmax = 0.0, supp = 0.0;
    bool sign_ok = true;
    rp = 0.0;
    for (int c = 0; c < R; ++c) {
      const double zt = gemm_row<M>(o.A[c], rhs);
      const double zr = __dadd_rn(__dmul_rn(al, zt), __dmul_rn(oma, z[c]));
      const double zn = fmin(__dadd_rn(zr, __dmul_rn(ri, yv[c])), o.b[c]);
      const double yn = __dadd_rn(yv[c], __dmul_rn(rho, __dsub_rn(zr, zn)));
      const double dy = __dsub_rn(yn, yv[c]);
      dmax = fmax(dmax, fabs(dy));
      sign_ok &= !(dy < 0.0);  // l = -inf: a negative dy makes the support +inf
      supp = __dadd_rn(supp, dy > 0.0 ? __dmul_rn(o.b[c], dy) : 0.0);
      z[c] = zn;
      yv[c] = yn;
      const double ax = gemm_row<M>(o.A[c], xn);
      rp = fmax(rp, fabs(__dsub_rn(ax, zn)));
      maxAx = fmax(maxAx, fabs(ax));
      maxz = fmax(maxz, fabs(zn));
#pragma unroll
      for (int k = 0; k < M; ++k) {
        ATy[k] = __fma_rn(o.A[c][k], yn, ATy[k]);
        ATdy[k] = __fma_rn(o.A[c][k], dy, ATdy[k]);
      }
    }
    rd = 0.0;
    double atd = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      xs[k] = xn[k];
      const double px = __dmul_rn(2.0, xn[k]);
      rd = fmax(rd, fabs(__dadd_rn(__dsub_rn(px, 2.0 * x[k]), ATy[k])));
      maxPx = fmax(maxPx, fabs(px));
      maxATy = fmax(maxATy, fabs(ATy[k]));
      atd = fmax(atd, fabs(ATdy[k]));
    }
    const double eps_p = kGenEpsAbs + kGenEpsRel * fmax(maxAx, maxz);
    const double eps_d = kGenEpsAbs + kGenEpsRel * fmax(fmax(maxPx, maxATy), qn);
    if (rp <= eps_p && rd <= eps_d) { status = BZG_SOLVED; break; }
    if (sign_ok && dmax > 1e-13 && atd <= 1e-4 * dmax && __dadd_rn(supp, 0.0) <= -1e-4 * dmax) {
      status = BZG_INFEASIBLE;
      break;
    }
  }
  if (status == BZG_INFEASIBLE) return false;
  // polish (qpsolver.py:236-279): equality solve on the rows with b - A x <= tol
  const double tol = fmax(1e-7, 10.0 * rp);
  int act[RC];
  int k = 0;
  for (int c = 0; c < R; ++c)
    if (__dsub_rn(o.b[c], gemm_row<M>(o.A[c], xs)) <= tol) act[k++] = c;
  if (k > 0) {
    constexpr int NK = M + RC;
    const int nk = M + k;
    const double reg = 1e-8;
    double K0[NK][NK], U[NK][NK], rhs0[NK], w[NK];
    for (int r = 0; r < NK; ++r)
      for (int t = 0; t < NK; ++t) K0[r][t] = 0.0;
    for (int r = 0; r < M; ++r) {
      K0[r][r] = 2.0 + reg;
      rhs0[r] = 2.0 * x[r];
    }
    for (int a = 0; a < k; ++a) {
      for (int r = 0; r < M; ++r) {
        K0[r][M + a] = o.A[act[a]][r];
        K0[M + a][r] = o.A[act[a]][r];
      }
      K0[M + a][M + a] = -reg;
      rhs0[M + a] = o.b[act[a]];
    }
    int perm[NK];
    for (int r = 0; r < nk; ++r) {
      perm[r] = r;
      for (int t = 0; t < nk; ++t) U[r][t] = K0[r][t];
    }
    bool singular = false;
    for (int cc = 0; cc < nk && !singular; ++cc) {
      int piv = cc;
      for (int r = cc + 1; r < nk; ++r)
        if (fabs(U[r][cc]) > fabs(U[piv][cc])) piv = r;
      if (U[piv][cc] == 0.0) { singular = true; break; }
      if (piv != cc) {
        for (int t = 0; t < nk; ++t) { const double s = U[cc][t]; U[cc][t] = U[piv][t]; U[piv][t] = s; }
        const int s = perm[cc]; perm[cc] = perm[piv]; perm[piv] = s;
      }
      const double rpv = 1.0 / U[cc][cc];
      for (int r = cc + 1; r < nk; ++r) {
        const double l = U[r][cc] * rpv;
        U[r][cc] = l;
        for (int t = cc + 1; t < nk; ++t) U[r][t] = __fma_rn(-l, U[cc][t], U[r][t]);
      }
    }
    if (!singular) {
      auto solve = [&](const double* bvec, double* out) {
        for (int r = 0; r < nk; ++r) {
          double t = bvec[perm[r]];
          for (int c2 = 0; c2 < r; ++c2) t = __fma_rn(-U[r][c2], out[c2], t);
          out[r] = t;
        }
        for (int r = nk - 1; r >= 0; --r) {
          double t = out[r];
          for (int c2 = r + 1; c2 < nk; ++c2) t = __fma_rn(-U[r][c2], out[c2], t);
          out[r] = t / U[r][r];
        }
      };
      solve(rhs0, w);
      for (int rep = 0; rep < 2; ++rep) {
        double res[NK], dw[NK];
        for (int r = 0; r < nk; ++r) {
          double t = 0.0;
          for (int c2 = 0; c2 < nk; ++c2) t = __fma_rn(K0[r][c2], w[c2], t);
          res[r] = __dsub_rn(rhs0[r], t);
        }
        solve(res, dw);
        for (int r = 0; r < nk; ++r) w[r] = __dadd_rn(w[r], dw[r]);
      }
      // acceptance: primal violation and dual residual of (x_pol, y_pol)
      double rpp = 0.0, aty[M];
#pragma unroll
      for (int kk = 0; kk < M; ++kk) aty[kk] = 0.0;
      for (int c = 0; c < R; ++c) rpp = fmax(rpp, fmax(__dsub_rn(gemm_row<M>(o.A[c], w), o.b[c]), 0.0));
      for (int a = 0; a < k; ++a)
#pragma unroll
        for (int kk = 0; kk < M; ++kk) aty[kk] = __fma_rn(o.A[act[a]][kk], w[M + a], aty[kk]);
      double rdp = 0.0;
#pragma unroll
      for (int kk = 0; kk < M; ++kk) rdp = fmax(rdp, fabs(__dadd_rn(__dsub_rn(2.0 * w[kk], 2.0 * x[kk]), aty[kk])));
      if (fmax(rpp, rdp) < fmax(rp, rd)) {
#pragma unroll
        for (int kk = 0; kk < M; ++kk) xs[kk] = w[kk];
      }
    }
  }
#pragma unroll
  for (int kk = 0; kk < M; ++kk) y[kk] = xs[kk];
  return true;
}

// cut_heuristic (graph.py:202-221) on the control points P (M x J): 0 unsafe, 1 safe, 2 indeterminate;
// -1 when a projection QP certifies an empty polytope (the reference raises).
template <int G, int M, int RC>
__device__ int general_code(const double (&P)[M][2 * G], const ObsRec<M, RC>& o, double margin, double eps) {
  constexpr int J = 2 * G;
  const int R = (int)o.rows;
  // O.contains_many(pts.T, eps): gemm order
  for (int j = 0; j < J; ++j) {
    double p[M];
#pragma unroll
    for (int k = 0; k < M; ++k) p[k] = P[k][j];
    bool in = true;
    for (int c = 0; c < R; ++c) in &= gemm_row<M>(p, o.A[c]) <= o.b_eps[c];
    if (in) return 0;
  }
  int anchor = 0;
  double best = 0.0, yan[M];
  for (int j = 0; j < J; ++j) {
    double p[M], y[M], dv[M];
#pragma unroll
    for (int k = 0; k < M; ++k) p[k] = P[k][j];
    if (!closest_point_general<M, RC>(o, p, eps, y)) return -1;
#pragma unroll
    for (int k = 0; k < M; ++k) dv[k] = __dsub_rn(y[k], p[k]);
    const double dj = norm1d<M>(dv);
    if (j == 0 || dj < best) {
      best = dj;
      anchor = j;
#pragma unroll
      for (int k = 0; k < M; ++k) yan[k] = y[k];
    }
  }
  double x[M];
#pragma unroll
  for (int k = 0; k < M; ++k) x[k] = P[k][anchor];
  // adjacent_hyperplane (geometry.py:233-252); y = closest_point(O, x) is the anchor's projection
  bool any_act = false;
  for (int c = 0; c < R; ++c) any_act |= __ddiv_rn(__dsub_rn(o.b[c], gemv_row<M>(o.A[c], yan)), o.norm2[c]) <= 1e-7;
  int idx = 0;
  double bs = -INFINITY;
  for (int c = 0; c < R; ++c) {
    const bool active = !any_act || __ddiv_rn(__dsub_rn(o.b[c], gemv_row<M>(o.A[c], yan)), o.norm2[c]) <= 1e-7;
    const double slack = __ddiv_rn(__dsub_rn(o.b[c], gemv_row<M>(o.A[c], x)), o.norm2[c]);
    const double sep = active ? -slack : -INFINITY;
    if (c == 0 || sep > bs) { bs = sep; idx = c; }
  }
  // Hyperplane(A[idx], b[idx]): unit normal and offset (geometry.py:94-100)
  const double nn = norm1d<M>(o.A[idx]);
  double normal[M];
#pragma unroll
  for (int k = 0; k < M; ++k) normal[k] = __ddiv_rn(o.A[idx][k], nn);
  const double off = __ddiv_rn(o.b[idx], nn);
  const int tail0 = (J / 4) * 4;  // vector @ matrix: blocks of four columns, then the tail
  bool clear = true;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double p[M];
#pragma unroll
    for (int k = 0; k < M; ++k) p[k] = P[k][j];
    const double hp = j < tail0 ? vecmat_block<M>(normal, p) : gemm_row<M>(normal, p);
    clear &= __dsub_rn(hp, off) > margin;
  }
  return clear ? 1 : 2;
}

}  // namespace
}  // namespace bzg
