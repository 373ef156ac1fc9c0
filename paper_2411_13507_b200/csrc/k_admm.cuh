// Cut-QP dense ADMM, one thread per instance.  Included by k_cut.cu.
//
// The reference (qpsolver.py:129-233, _dense_kernel) forms the (n+mc)^2 KKT matrix
// [[P + sigma I, A'], [A, -R^-1]] per instance, inverts it (np.linalg.inv) and applies the
// inverse every iteration.  The same step is
//   xt = M^-1 (sigma x - q + A'(R z - y)),  zt = A xt,   M = P + sigma I + A'RA.
// For the cut QP (graph.py:268-282) the delta block of M is kdd I, kdd = 2 + sigma + rho,
// so its Schur complement leaves one J x J SPD matrix
//   S = (sigma + rho) I + (rho - rho^2/kdd) Q'Q + rho_eq 11',
// inverted once per instance.  Relaxation, projection, dual update, the termination test
// (rp <= eps_p and rd <= eps_d), the primal-infeasibility certificate and MAX_ITER follow
// qpsolver.py:164-231 operation by operation; only the linear solve differs from the
// reference by rounding.
//
// Scheduling: persistent lanes.  Each lane owns one instance; between batches of
// kBatch iterations, lanes whose instance terminated fetch the next one with one
// warp-aggregated atomic, so the 500-iteration MAX_ITER instances do not idle the warp.
#pragma once

namespace bzg {
namespace {

constexpr int kAdmmBatch = 8;

template <int G, int M>
__device__ __forceinline__ void admm_setup(double (&Q)[2 * M][2 * G], double (&Si)[G * (2 * G + 1)], double rho,
                                           double req, double sig, double ikdd) {
  constexpr int J = 2 * G, C = 2 * M;
  const double kap = rho - rho * rho * ikdd;
  double L[J][J], dinv[J];
#pragma unroll
  for (int r = 0; r < J; ++r)
#pragma unroll
    for (int s = 0; s <= r; ++s) {
      double qq = 0.0;
#pragma unroll
      for (int c = 0; c < C; ++c) qq = __fma_rn(Q[c][r], Q[c][s], qq);
      L[r][s] = kap * qq + req + (r == s ? sig + rho : 0.0);
    }
#pragma unroll
  for (int r = 0; r < J; ++r) {  // Cholesky L L'
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
  double W[J][J];  // W = L^-1
#pragma unroll
  for (int r = 0; r < J; ++r) {
    W[r][r] = dinv[r];
#pragma unroll
    for (int s = 0; s < r; ++s) {
      double t = 0.0;
#pragma unroll
      for (int k = s; k < r; ++k) t = __fma_rn(L[r][k], k == s ? dinv[s] : W[k][s], t);
      W[r][s] = -t * dinv[r];
    }
  }
#pragma unroll
  for (int r = 0; r < J; ++r)  // S^-1 = W'W, packed lower triangle
#pragma unroll
    for (int s = 0; s <= r; ++s) {
      double t = 0.0;
#pragma unroll
      for (int k = r; k < J; ++k) t = __fma_rn(W[k][r], W[k][s], t);
      Si[r * (r + 1) / 2 + s] = t;
    }
}

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
  double lam[J], del[C], zc[C], zl[J], ze, yc[C], yl[J], ye;
#define SI(r, s) Si[(r) >= (s) ? (r) * ((r) + 1) / 2 + (s) : (s) * ((s) + 1) / 2 + (r)]

  while (true) {
    // ---- refill lanes whose instance terminated (one atomic per warp)
    const unsigned need = __ballot_sync(0xffffffffu, inst == -1);
    if (need) {
      unsigned long long base = 0;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base = atomicAdd(next, (unsigned long long)__popc(need));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (inst == -1) {
        const unsigned long long my = base + __popc(need & ((1u << lane) - 1u));
        inst = (long long)my < n_inst ? (long long)my : -2;
        if (inst >= 0) {
          load_instance<G, M>(dp, Vx, src, dst, obs, pend[inst], Q, b);
          admm_setup<G, M>(Q, Si, rho, req, sig, ikdd);
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
    if (__all_sync(0xffffffffu, inst == -2)) break;

    // ---- a batch of iterations (qpsolver.py:164-211)
#pragma unroll 1
    for (int k = 0; k < kAdmmBatch; ++k) {
      if (inst < 0) break;
      ++it;
      double rdel[C], tC[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double wc = __fma_rn(rho, zc[c], -yc[c]);  // (R z - y)_c
        rdel[c] = __fma_rn(sig, del[c], -wc);          // sigma delta - w_c
        tC[c] = __fma_rn(kp, rdel[c], wc);
      }
      const double we = __fma_rn(req, ze, -ye);
      double rv[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        double acc = __fma_rn(sig, lam[j], __fma_rn(rho, zl[j], -yl[j]) + we);
#pragma unroll
        for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], tC[c], acc);
        rv[j] = acc;
      }
      double a[J];
#pragma unroll
      for (int r = 0; r < J; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < J; ++s) acc = __fma_rn(SI(r, s), rv[s], acc);
        a[r] = acc;
      }
      // relaxation, projection onto [l, u] and dual update, row block by row block
      bool sign_ok = true;  // the certificate needs dy_c >= 0 and dy_lambda <= 0 (finite bounds)
      bool pbad = false;    // some |(A x - z)_i| > eps_p
      double dyc[C], dyl[J];
      double sa = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        sa += a[j];
        const double zr = __dadd_rn(__dmul_rn(al, a[j]), __dmul_rn(oma, zl[j]));
        const double zn = fmax(__dadd_rn(zr, __dmul_rn(ri, yl[j])), 0.0);
        const double yn = __dadd_rn(yl[j], __dmul_rn(rho, __dsub_rn(zr, zn)));
        dyl[j] = __dsub_rn(yn, yl[j]);
        sign_ok = sign_ok && !(dyl[j] > 0.0);
        lam[j] = __dadd_rn(__dmul_rn(al, a[j]), __dmul_rn(oma, lam[j]));
        zl[j] = zn;
        yl[j] = yn;
        pbad = pbad || !(fabs(__dsub_rn(lam[j], zn)) <= qp.eps_abs);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double qa = 0.0;
#pragma unroll
        for (int j = 0; j < J; ++j) qa = __fma_rn(Q[c][j], a[j], qa);
        const double d = __fma_rn(rdel[c], ikdd, kp * qa);
        const double zr = __dadd_rn(__dmul_rn(al, __dsub_rn(qa, d)), __dmul_rn(oma, zc[c]));
        const double zn = fmin(__dadd_rn(zr, __dmul_rn(ri, yc[c])), b[c]);
        const double yn = __dadd_rn(yc[c], __dmul_rn(rho, __dsub_rn(zr, zn)));
        dyc[c] = __dsub_rn(yn, yc[c]);
        sign_ok = sign_ok && !(dyc[c] < 0.0);
        del[c] = __dadd_rn(__dmul_rn(al, d), __dmul_rn(oma, del[c]));
        zc[c] = zn;
        yc[c] = yn;
      }
      double dye;
      {
        const double zr = __dadd_rn(__dmul_rn(al, sa), __dmul_rn(oma, ze));
        const double yn = __dadd_rn(ye, __dmul_rn(req, __dsub_rn(zr, 1.0)));  // z clipped to [1, 1]
        dye = __dsub_rn(yn, ye);
        ze = 1.0;
        ye = yn;
      }
      // termination test at the new iterate (qpsolver.py:176-188)
      double sl = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) sl = __dadd_rn(sl, lam[j]);
      pbad = pbad || !(fabs(__dsub_rn(sl, 1.0)) <= qp.eps_abs);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < J; ++j) acc = __fma_rn(Q[c][j], lam[j], acc);
        pbad = pbad || !(fabs(__dsub_rn(__dsub_rn(acc, del[c]), zc[c])) <= qp.eps_abs);
      }
      bool dbad = false;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        double acc = __dadd_rn(yl[j], ye);
#pragma unroll
        for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], yc[c], acc);
        dbad = dbad || !(fabs(acc) <= qp.eps_abs);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) dbad = dbad || !(fabs(__dsub_rn(__dmul_rn(2.0, del[c]), yc[c])) <= qp.eps_abs);

      int status = -1;
      double rprim = 0.0, rdual = 0.0;
      if (rel || !(pbad || dbad) || sign_ok || it >= qp.max_iter) {
        // rare path: exact residual maxima (qpsolver.py:179-186) and the relative tolerances
        double maxAx = 0.0, maxz = 1.0, maxPx = 0.0, maxATy = 0.0;
        rprim = fabs(__dsub_rn(sl, 1.0));
        maxAx = fabs(sl);
#pragma unroll
        for (int j = 0; j < J; ++j) {
          rprim = fmax(rprim, fabs(__dsub_rn(lam[j], zl[j])));
          maxAx = fmax(maxAx, fabs(lam[j]));
          maxz = fmax(maxz, fabs(zl[j]));
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < J; ++j) acc = __fma_rn(Q[c][j], lam[j], acc);
          const double ax = __dsub_rn(acc, del[c]);
          rprim = fmax(rprim, fabs(__dsub_rn(ax, zc[c])));
          maxAx = fmax(maxAx, fabs(ax));
          maxz = fmax(maxz, fabs(zc[c]));
        }
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
          maxPx = fmax(maxPx, fabs(px));
          maxATy = fmax(maxATy, fabs(yc[c]));
        }
        const double eps_p = rel ? qp.eps_abs + qp.eps_rel * fmax(maxAx, maxz) : qp.eps_abs;
        const double eps_d = rel ? qp.eps_abs + qp.eps_rel * fmax(maxPx, maxATy) : qp.eps_abs;
        if (rprim <= eps_p && rdual <= eps_d) {
          status = BZG_SOLVED;
        } else if (sign_ok) {
          // primal-infeasibility certificate (qpsolver.py:193-209): with every dy_i on a finite
          // bound, support = sum_c b_c dy_c + dy_eq
          double dmax = fabs(dye), atd = 0.0, supp = 0.0;
#pragma unroll
          for (int j = 0; j < J; ++j) {
            dmax = fmax(dmax, fabs(dyl[j]));
            double acc = __dadd_rn(dyl[j], dye);
#pragma unroll
            for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], dyc[c], acc);
            atd = fmax(atd, fabs(acc));
          }
#pragma unroll
          for (int c = 0; c < C; ++c) {
            dmax = fmax(dmax, fabs(dyc[c]));
            atd = fmax(atd, fabs(dyc[c]));
            supp = __dadd_rn(supp, __dmul_rn(b[c], dyc[c]));
          }
          supp = __dadd_rn(supp, dye);
          if (dmax > 1e-13 && atd <= qp.eps_pinf * dmax && supp <= -qp.eps_pinf * dmax) status = BZG_INFEASIBLE;
        }
        if (status < 0 && it >= qp.max_iter) status = BZG_MAX_ITER;
      }
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
#undef SI
}

}  // namespace
}  // namespace bzg
