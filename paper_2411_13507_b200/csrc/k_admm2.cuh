// Cut-QP dense ADMM with TWO lanes per instance (a lane pair), for launches with few
// instances per resident lane.  Included by k_qp_impl.cuh after k_admm.cuh.
//
// Why: k_qp_admm runs one instance per lane, so an instance's iterations are a serial chain
// of ~280 FP64 instructions each; when the work list holds only a few instances per lane
// (cfg2's 107 k instances on 56.8 k lanes, one row block of an 8-way split) the kernel's time
// is set by the 500-iteration MAX_ITER chains in the tail.  Splitting each iteration over two
// lanes halves that chain.
//
// Bitwise contract: every iterate equals k_qp_admm<G, M, C, false, true, CANON>'s.  Each
// quantity is formed by the same operations in the same order; only WHO forms it changes:
//   * lane p of the pair owns the lambda rows j in [p*G, (p+1)*G) (the S^-1 rows, the
//     lambda/z/y block and the Q columns of those j), and the stored obstacle rows r with
//     r % 2 == p (the delta/z/y of their constraint rows c = r and, for a canonical box,
//     c = r + M, and the Q row r);
//   * whenever a sum runs over rows the lane does not own (Q'f over r, S^-1 rv over s,
//     Q a and Q lambda over j, sum(a), sum(lambda), the certificate's b'dy over c), the
//     partner's terms arrive by shuffle and the sum is folded in the original index order
//     on both lanes (sums over all j are computed redundantly, so both lanes hold them);
//   * the termination and certificate tests are per-lane partial ANDs/maxima combined
//     across the pair (exact: AND and max are order-free).
// Only the UNIT (rho = 1), absolute-tolerance (eps_rel = 0) configuration -- the
// CutConfig default -- has this variant; the host falls back to k_qp_admm otherwise.
#pragma once

namespace bzg {
namespace {

// k_qp_admm2 is chosen for work lists of at most kAdmm2MaxInst instances: every instance is
// then a lone chain on its SM sub-partition and two lanes shorten it (cfg1: 0.195 -> 0.178 ms);
// with more instances the extra shuffles and the redundant sums cost more than they save
// (cfg2 0.57 -> 0.62 ms, cfg3 9.2 -> 12.7 ms).  BZG_ADMM_LANES=1|2 forces one.
constexpr long long kAdmm2MaxInst = 4096;

template <int G, int M, int C, bool CANON>
__global__ void __launch_bounds__(128, 2) k_qp_admm2(QpParams qp, const double* __restrict__ consts, long long n_inst,
                                                  unsigned long long* __restrict__ next, int8_t* __restrict__ st_out,
                                                  int* __restrict__ it_out, double* __restrict__ x_out,
                                                  double* __restrict__ zy_out,
                                                  const unsigned long long* __restrict__ d_n) {
  BZG_PDL_ENTRY();
  using K = QpConsts<G, M, C, CANON>;
  constexpr int J = 2 * G, JH = G, NV = J + C, MC = C + J + 1;
  constexpr int R = K::R;          // stored Q rows
  constexpr int RH = (R + 1) / 2;  // stored rows per lane: r = 2 i + p
  constexpr int CPR = CANON ? 2 : 1;
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, p = lane & 1, pair0 = lane & ~1;
  const double req = qp.rho_eq, sig = qp.sigma, al = qp.alpha, oma = qp.one_m_alpha, eps = qp.eps_abs;
  const double kdd = 2.0 + sig + 1.0, ikdd = 1.0 / kdd, kp = 1.0 * ikdd;  // rho = 1 (UNIT)
#define RELAX(a, b) __fma_rn(al, (a), __dmul_rn(oma, (b)))
#define XCH(v) __shfl_xor_sync(FULL, (v), 1)

  const long long n_lim = dev_count(n_inst, d_n);
  long long inst = -1;  // pair-uniform: -1 needs work, -2 exhausted
  int it = 0;
  double si[JH][J];              // S^-1 rows of the owned lambda rows
  double qcol[R][JH];            // Q[r][j] for every r and the owned j
  double qrow[RH][J];            // Q[r][j] for the owned stored rows r and every j
  double bb[RH][CPR];
  double lam[JH], zl[JH], yl[JH];
  double del[RH][CPR], zc[RH][CPR], yc[RH][CPR];
  double ze = 0.0, ye = 0.0;
  // pipelining state: pend = the current state is an iterate whose termination test is due;
  // cu / su / dy* = the partial convergence test, sign test and dual steps of its update
  bool pend = false, cu = true, su = true;
  double dyl[JH], dyc[RH][CPR], dye = 0.0;

  while (true) {
    // ---- refill pairs whose instance terminated (one atomic per warp)
    const unsigned need = __ballot_sync(FULL, inst == -1);
    if (need) {
      unsigned long long base = 0;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base = atomicAdd(next, (unsigned long long)(__popc(need) >> 1));
      base = __shfl_sync(FULL, base, leader);
      if (inst == -1) {
        const unsigned long long my = base + (__popc(need & ((1u << pair0) - 1u)) >> 1);
        inst = (long long)my < n_lim ? (long long)my : -2;
        if (inst >= 0) {
          const double* o = consts + inst;
#pragma unroll
          for (int k = 0; k < JH; ++k) {
            const int r = p * JH + k;
#pragma unroll
            for (int s = 0; s < J; ++s) {
              const int hi = r >= s ? r : s, lo = r >= s ? s : r;
              si[k][s] = o[(hi * (hi + 1) / 2 + lo) * n_inst];
            }
#pragma unroll
            for (int rr = 0; rr < R; ++rr) qcol[rr][k] = o[(K::NS + rr * J + r) * n_inst];
          }
#pragma unroll
          for (int i = 0; i < RH; ++i) {
            const int r = 2 * i + p;
            const bool ok = r < R;
#pragma unroll
            for (int j = 0; j < J; ++j) qrow[i][j] = ok ? o[(K::NS + r * J + j) * n_inst] : 0.0;
#pragma unroll
            for (int l = 0; l < CPR; ++l) bb[i][l] = ok ? o[(K::NS + K::NQ + r + l * M) * n_inst] : 1e300;
          }
        }
#pragma unroll
        for (int k = 0; k < JH; ++k) { lam[k] = 0.0; zl[k] = 0.0; yl[k] = 0.0; }
#pragma unroll
        for (int i = 0; i < RH; ++i)
#pragma unroll
          for (int l = 0; l < CPR; ++l) { del[i][l] = 0.0; zc[i][l] = 0.0; yc[i][l] = 0.0; }
        ze = 0.0;
        ye = 0.0;
        it = 0;
        pend = false;
      }
    }
    if (__all_sync(FULL, inst == -2)) break;

    // ---- a batch of iterations; every lane runs the body (the shuffles need the whole
    // warp), lanes without an instance compute on stale state and write nothing.
    // Software-pipelined: iteration k+1's update is formed (into n_*) while iteration k's
    // termination test runs on the current state -- two independent dependency chains the
    // scheduler interleaves; when the test stops the instance, the current state (iteration
    // k) is written and the speculative update is dropped, so iterates, iteration counts and
    // outputs are k_qp_admm's exactly.
#pragma unroll 1
    for (int kb = 0; kb < qp.batch; ++kb) {
      if (__all_sync(FULL, inst < 0)) break;
      const bool live = inst >= 0;
      // ===== update chain: the next iterate from the current state
      double rdel[RH][CPR], fT[RH];
#pragma unroll
      for (int i = 0; i < RH; ++i) {
        double tC[CPR];
#pragma unroll
        for (int l = 0; l < CPR; ++l) {
          const double wc = __dsub_rn(zc[i][l], yc[i][l]);
          rdel[i][l] = __fma_rn(sig, del[i][l], -wc);
          tC[l] = __fma_rn(kp, rdel[i][l], wc);
        }
        fT[i] = CANON ? __dsub_rn(tC[0], tC[1]) : tC[0];
      }
      const double we = __fma_rn(req, ze, -ye);
      double fTa[R];
#pragma unroll
      for (int i = 0; i < RH; ++i) {
        const double oth = XCH(fT[i]);
        if (2 * i < R) fTa[2 * i] = p == 0 ? fT[i] : oth;
        if (2 * i + 1 < R) fTa[2 * i + 1] = p == 0 ? oth : fT[i];
      }
      double rv[JH];
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        const double wl = __dsub_rn(zl[k], yl[k]);
        double acc = __fma_rn(sig, lam[k], __dadd_rn(wl, we));
#pragma unroll
        for (int r = 0; r < R; ++r) acc = __fma_rn(qcol[r][k], fTa[r], acc);
        rv[k] = acc;
      }
      double rva[J];
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        const double oth = XCH(rv[k]);
        rva[k] = p == 0 ? rv[k] : oth;
        rva[JH + k] = p == 0 ? oth : rv[k];
      }
      double a[JH];
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < J; ++s) acc = __fma_rn(si[k][s], rva[s], acc);
        a[k] = acc;
      }
      double aa[J];
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        const double oth = XCH(a[k]);
        aa[k] = p == 0 ? a[k] : oth;
        aa[JH + k] = p == 0 ? oth : a[k];
      }
      bool n_su = true, n_cu = true;
      double n_lam[JH], n_zl[JH], n_yl[JH], n_dyl[JH];
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        const double zr = RELAX(a[k], zl[k]);
        const double zn = clip_nonneg(__dadd_rn(zr, yl[k]));
        const double yn = __dadd_rn(yl[k], __dsub_rn(zr, zn));
        n_dyl[k] = __dsub_rn(yn, yl[k]);
        n_su &= not_pos(n_dyl[k]);
        n_lam[k] = RELAX(a[k], lam[k]);
        n_zl[k] = zn;
        n_yl[k] = yn;
        n_cu &= fabs(__dsub_rn(n_lam[k], zn)) <= eps;
      }
      double sa = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) sa += aa[j];
      double n_del[RH][CPR], n_zc[RH][CPR], n_yc[RH][CPR], n_dyc[RH][CPR];
#pragma unroll
      for (int i = 0; i < RH; ++i) {
        double qa = 0.0;
#pragma unroll
        for (int j = 0; j < J; ++j) qa = __fma_rn(qrow[i][j], aa[j], qa);
#pragma unroll
        for (int l = 0; l < CPR; ++l) {
          const double q = l == 0 ? qa : -qa;
          const double d = __fma_rn(rdel[i][l], ikdd, kp * q);
          const double zr = RELAX(__dsub_rn(q, d), zc[i][l]);
          const double zn = clip_upper(__dadd_rn(zr, yc[i][l]), bb[i][l]);
          const double yn = __dadd_rn(yc[i][l], __dsub_rn(zr, zn));
          n_dyc[i][l] = __dsub_rn(yn, yc[i][l]);
          n_su &= not_neg(n_dyc[i][l]);
          n_del[i][l] = RELAX(d, del[i][l]);
          n_zc[i][l] = zn;
          n_yc[i][l] = yn;
        }
      }
      double n_ye, n_dye;
      {
        const double zr = RELAX(sa, ze);
        n_ye = __dadd_rn(ye, __dmul_rn(req, __dsub_rn(zr, 1.0)));
        n_dye = __dsub_rn(n_ye, ye);
      }

      // ===== termination test of the current state (iteration `it`; none before the first)
      bool conv = cu;
      double la[J];
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        const double oth = XCH(lam[k]);
        la[k] = p == 0 ? lam[k] : oth;
        la[JH + k] = p == 0 ? oth : lam[k];
      }
      double sl = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) sl = __dadd_rn(sl, la[j]);
      conv &= fabs(__dsub_rn(sl, 1.0)) <= eps;
      double fY[RH];
#pragma unroll
      for (int i = 0; i < RH; ++i) {
        double ql = 0.0;
#pragma unroll
        for (int j = 0; j < J; ++j) ql = __fma_rn(qrow[i][j], la[j], ql);
#pragma unroll
        for (int l = 0; l < CPR; ++l) {
          const double ax = __dsub_rn(l == 0 ? ql : -ql, del[i][l]);
          conv &= fabs(__dsub_rn(ax, zc[i][l])) <= eps;
          conv &= fabs(__fma_rn(2.0, del[i][l], -yc[i][l])) <= eps;
        }
        fY[i] = CANON ? __dsub_rn(yc[i][0], yc[i][1]) : yc[i][0];
      }
      double fYa[R];
#pragma unroll
      for (int i = 0; i < RH; ++i) {
        const double oth = XCH(fY[i]);
        if (2 * i < R) fYa[2 * i] = p == 0 ? fY[i] : oth;
        if (2 * i + 1 < R) fYa[2 * i + 1] = p == 0 ? oth : fY[i];
      }
#pragma unroll
      for (int k = 0; k < JH; ++k) {
        double acc = __dadd_rn(yl[k], ye);
#pragma unroll
        for (int r = 0; r < R; ++r) acc = __fma_rn(qcol[r][k], fYa[r], acc);
        conv &= fabs(acc) <= eps;
      }
      // combine the pair's partial tests
      const unsigned bc = __ballot_sync(FULL, conv), bs = __ballot_sync(FULL, su);
      conv = pend && ((bc >> pair0) & 3u) == 3u;
      const bool sign_ok = ((bs >> pair0) & 3u) == 3u;

      int status = conv ? BZG_SOLVED : -1;
      const bool cert = live && pend && !conv && sign_ok;
      if (__any_sync(FULL, cert)) {
        // primal-infeasibility certificate (k_qp_admm's test, qpsolver.py:193-209), formed on
        // every lane of the warp and applied where `cert` holds
        double pr[RH][CPR];
#pragma unroll
        for (int i = 0; i < RH; ++i)
#pragma unroll
          for (int l = 0; l < CPR; ++l) pr[i][l] = __dmul_rn(bb[i][l], dyc[i][l]);
        double supp = 0.0;  // sum over c in 0..C-1 in order
#pragma unroll
        for (int l = 0; l < CPR; ++l)
#pragma unroll
          for (int i = 0; i < RH; ++i) {
            const double oth = XCH(pr[i][l]);
            // stored row 2i holds constraint rows 2i + l*M, 2i+1 holds 2i+1 + l*M
            if (2 * i < R) supp = __dadd_rn(supp, p == 0 ? pr[i][l] : oth);
            if (2 * i + 1 < R) supp = __dadd_rn(supp, p == 0 ? oth : pr[i][l]);
          }
        supp = __dadd_rn(supp, dye);
        double dmax = fabs(dye);
#pragma unroll
        for (int k = 0; k < JH; ++k) dmax = max_nn(dmax, fabs(dyl[k]));
#pragma unroll
        for (int i = 0; i < RH; ++i)
#pragma unroll
          for (int l = 0; l < CPR; ++l) dmax = max_nn(dmax, fabs(dyc[i][l]));
        dmax = max_nn(dmax, XCH(dmax));
        const double lim = qp.eps_pinf * dmax;
        bool small = true;
        double fD[RH];
#pragma unroll
        for (int i = 0; i < RH; ++i) {
#pragma unroll
          for (int l = 0; l < CPR; ++l) small &= fabs(dyc[i][l]) <= lim;
          fD[i] = CANON ? __dsub_rn(dyc[i][0], dyc[i][1]) : dyc[i][0];
        }
        double fDa[R];
#pragma unroll
        for (int i = 0; i < RH; ++i) {
          const double oth = XCH(fD[i]);
          if (2 * i < R) fDa[2 * i] = p == 0 ? fD[i] : oth;
          if (2 * i + 1 < R) fDa[2 * i + 1] = p == 0 ? oth : fD[i];
        }
#pragma unroll
        for (int k = 0; k < JH; ++k) {
          double acc = __dadd_rn(dyl[k], dye);
#pragma unroll
          for (int r = 0; r < R; ++r) acc = __fma_rn(qcol[r][k], fDa[r], acc);
          small &= fabs(acc) <= lim;
        }
        const unsigned bsm = __ballot_sync(FULL, small);
        small = ((bsm >> pair0) & 3u) == 3u;
        if (cert && supp < 0.0 && dmax > 1e-13 && supp <= -lim && small) status = BZG_INFEASIBLE;
      }
      if (pend && status < 0 && it >= qp.max_iter) status = BZG_MAX_ITER;
      if (live && status >= 0) {
        double* xo = x_out + inst * NV;
        double* zo = zy_out + inst * 2 * MC;
        if (p == 0) {
          st_out[inst] = (int8_t)status;
          it_out[inst] = it;
          zo[MC - 1] = ze;
          zo[2 * MC - 1] = ye;
        }
#pragma unroll
        for (int k = 0; k < JH; ++k) {
          const int j = p * JH + k;
          xo[j] = lam[k];
          zo[C + j] = zl[k];
          zo[MC + C + j] = yl[k];
        }
#pragma unroll
        for (int i = 0; i < RH; ++i) {
          const int r = 2 * i + p;
          if (r < R)
#pragma unroll
            for (int l = 0; l < CPR; ++l) {
              const int c = r + l * M;
              xo[J + c] = del[i][l];
              zo[c] = zc[i][l];
              zo[MC + c] = yc[i][l];
            }
        }
        inst = -1;
      } else {  // commit the next iterate
        it += live ? 1 : 0;
        pend = true;
        cu = n_cu;
        su = n_su;
#pragma unroll
        for (int k = 0; k < JH; ++k) {
          lam[k] = n_lam[k];
          zl[k] = n_zl[k];
          yl[k] = n_yl[k];
          dyl[k] = n_dyl[k];
        }
#pragma unroll
        for (int i = 0; i < RH; ++i)
#pragma unroll
          for (int l = 0; l < CPR; ++l) {
            del[i][l] = n_del[i][l];
            zc[i][l] = n_zc[i][l];
            yc[i][l] = n_yc[i][l];
            dyc[i][l] = n_dyc[i][l];
          }
        ze = 1.0;
        ye = n_ye;
        dye = n_dye;
      }
    }
  }
#undef RELAX
#undef XCH
}

}  // namespace
}  // namespace bzg
