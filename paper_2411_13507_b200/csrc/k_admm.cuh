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
// qpsolver.py:164-231 operation by operation; only the linear solve and the fused
// relaxation (RELAX) differ from the reference by rounding.
//
// Scheduling: persistent lanes.  Each lane owns one instance; between batches of
// kAdmmBatch iterations, lanes whose instance terminated fetch the next one with one
// warp-aggregated atomic, so the 500-iteration MAX_ITER instances do not idle the warp.
// The hot loop only decides termination (compare-only tests); the residual maxima the
// polish needs are recomputed from the stored (x, z, y) by k_qp_select.
#pragma once

namespace bzg {
namespace {

// Relaxation alpha*xt + (1-alpha)*x as one FMA over the rounded second product.  The
// reference rounds both products and the sum; the fused form differs by at most an ulp, the
// order of the linear-solve difference, and saves 21 FP64 instructions per iteration (4% of
// k_qp_admm).  Golden QP verdicts, statuses and counters are unchanged (tests/test_gpu_parity.py).
#define RELAX(a, b) __fma_rn(al, (a), __dmul_rn(oma, (b)))

constexpr int kAdmmBatch = 16;  // default of QpParams::batch (BZG_ADMM_BATCH overrides; 4..32 within 2%)

template <int G, int M, int C>
__device__ __forceinline__ void admm_setup(double (&Q)[C][2 * G], double (&Si)[G * (2 * G + 1)], double rho,
                                           double req, double sig, double ikdd) {
  constexpr int J = 2 * G;
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

// Comparisons and clips as one DSETP (+ selects): fmin/fmax carry NaN handling that costs
// ~6 instructions each, and 64-bit integer tests cost ~5; no operand here is NaN.
__device__ __forceinline__ bool not_pos(double v) { return !(v > 0.0); }
__device__ __forceinline__ bool not_neg(double v) { return !(v < 0.0); }
// max(t, 0): clip to [0, +inf) (the sign of a zero result is immaterial downstream)
__device__ __forceinline__ double clip_nonneg(double t) { return t < 0.0 ? 0.0 : t; }
// min(v, u): clip to (-inf, u]
__device__ __forceinline__ double clip_upper(double v, double u) { return v <= u ? v : u; }
// max of two non-negative values
__device__ __forceinline__ double max_nn(double a, double b) { return a > b ? a : b; }

// Constraint-matrix products of the cut QP.  Q = A_O P (C x J).  For a canonical box
// (A_O = [I; -I], Box.to_polytope order) Q = [P; -P] exactly, so only the M rows of P are
// kept and every product is formed once per output dimension.
template <int G, int M, int C, bool CANON>
struct QOps {
  static constexpr int J = 2 * G, R = CANON ? M : C;
  double q[R][J];
  __device__ __forceinline__ void load(const double (&Q)[C][J]) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < J; ++j) q[r][j] = Q[r][j];
  }
  // out_c = Q_c . v   (FMA chain over j)
  __device__ __forceinline__ void mul(const double (&v)[J], double (&out)[C]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) acc = __fma_rn(q[r][j], v[j], acc);
      out[r] = acc;
      if (CANON) out[r + M] = -acc;
    }
  }
  // f = w folded onto the stored rows: w_r - w_{r+M} (canonical box) or w itself
  __device__ __forceinline__ void fold(const double (&w)[C], double (&f)[R]) const {
#pragma unroll
    for (int r = 0; r < R; ++r) f[r] = CANON ? __dsub_rn(w[r], w[r + M]) : w[r];
  }
  // returns acc + sum_c Q_cj w_c, with f = fold(w)
  __device__ __forceinline__ double tmulf(int j, const double (&f)[R], double acc) const {
#pragma unroll
    for (int r = 0; r < R; ++r) acc = __fma_rn(q[r][j], f[r], acc);
    return acc;
  }
  __device__ __forceinline__ double tmul(int j, const double (&w)[C], double acc) const {
    double f[R];
    fold(w, f);
    return tmulf(j, f, acc);
  }
};

// Per-instance constants of the iteration, prepared by k_qp_setup: the packed S^-1 (J(J+1)/2),
// the stored rows of Q (R x J) and b (C), as consecutive doubles per instance.
template <int G, int M, int C, bool CANON>
struct QpConsts {
  static constexpr int J = 2 * G, R = CANON ? M : C, NS = J * (J + 1) / 2, NQ = R * J, N = NS + NQ + C;
};

// One thread per instance: control points, Q = A_O P, and the Schur-complement inverse.
// Hoisted out of k_qp_admm, where the persistent lanes refill one instance at a time and
// the few refilling lanes would run this ~800-instruction setup while the rest of the
// warp idles (ncu: 23 of 32 lanes active).  Same arithmetic, so the iterates are unchanged.
template <int G, int M, int C, bool CANON>
__global__ void __launch_bounds__(128) k_qp_setup(QpParams qp, DParams dp, const double* __restrict__ Vx,
                                                  const int* __restrict__ src, const int* __restrict__ dst,
                                                  const ObsRec<M, obs_cap<C>()>* __restrict__ obs,
                                                  const unsigned long long* __restrict__ pend, long long n_inst,
                                                  const unsigned long long* __restrict__ d_n,
                                                  double* __restrict__ consts) {
  BZG_PDL_ENTRY();
  using K = QpConsts<G, M, C, CANON>;
  const long long n = dev_count(n_inst, d_n);
  const double rho = qp.rho, req = qp.rho_eq, sig = qp.sigma;
  const double kdd = 2.0 + sig + rho, ikdd = 1.0 / kdd;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    double Qf[C][2 * G], b[C], Si[K::NS];
    load_instance<G, M, C>(dp, Vx, src, dst, obs, pend[t], Qf, b);
    admm_setup<G, M, C>(Qf, Si, rho, req, sig, ikdd);
    // field-major: field k of instance t at consts[k * n_inst + t] (coalesced); n_inst is the
    // capacity of the work list, the stride every reader uses
    double* o = consts + t;
#pragma unroll
    for (int k = 0; k < K::NS; ++k) o[k * n_inst] = Si[k];
#pragma unroll
    for (int r = 0; r < K::R; ++r)
#pragma unroll
      for (int j = 0; j < K::J; ++j) o[(K::NS + r * K::J + j) * n_inst] = Qf[r][j];
#pragma unroll
    for (int c = 0; c < C; ++c) o[(K::NS + K::NQ + c) * n_inst] = b[c];
  }
}

// Tail compaction.  One instance per lane keeps the FP64 pipe busy while the work list lasts,
// but once it is drained the warps thin out: each warp instruction costs the pipe the same two
// cycles however few lanes are live (ncu on cfg2: 12.6 of 32 lanes per instruction), so the
// last, longest chains crawl behind their sparse neighbours.  A pass with dump_below > 0 parks
// the live iterates of a thinned warp (x / zy slots of the instance, iteration count in
// it_out) and queues the instance; the next launch resumes the queue densely packed, 32 per
// warp, from exactly that state, so every iterate is unchanged (bitwise).  The last pass
// has dump_below = 0 and runs everything it holds to termination.
struct AdmmPass {
  const int* rq_in;                // resume pass: instances to continue; nullptr: 0 .. n_inst-1
  const unsigned long long* rq_in_n;
  int* rq_out;                     // parked instances of this pass (n_inst capacity)
  unsigned long long* rq_out_n;
  int dump_below;                  // 0: never park
  int park_after;                  // > 0: park every instance still running after this many
                                   // iterations (longest-last schedule: the next pass runs the
                                   // long ones together); its lane takes new work
};

// REL: eps_rel != 0 (termination tolerances depend on the iterate, qpsolver.py:181-186)
// UNIT: rho == 1 (CutConfig default) -- the multiplications by rho and 1/rho are exact and skipped
// CANON: every obstacle is a canonical box (see QOps)
template <int G, int M, int C, bool REL, bool UNIT, bool CANON>
__global__ void __launch_bounds__(128, 3) k_qp_admm(QpParams qp, const double* __restrict__ consts, long long n_inst,
                                                 unsigned long long* __restrict__ next, int8_t* __restrict__ st_out,
                                                 int* __restrict__ it_out, double* __restrict__ x_out,
                                                 double* __restrict__ zy_out, AdmmPass pass,
                                                 const unsigned long long* __restrict__ d_n) {
  BZG_PDL_ENTRY();
  constexpr int J = 2 * G, NV = J + C, MC = C + J + 1;
  const int lane = threadIdx.x & 31;
  const double rho = UNIT ? 1.0 : qp.rho, req = qp.rho_eq, ri = UNIT ? 1.0 : 1.0 / qp.rho;
  const double sig = qp.sigma, al = qp.alpha, oma = qp.one_m_alpha, eps = qp.eps_abs;
  const double kdd = 2.0 + sig + rho, ikdd = 1.0 / kdd, kp = rho * ikdd;

  long long inst = -1;  // -1 needs work, -2 exhausted
  int it = 0;
  QOps<G, M, C, CANON> Q;
  double Si[J * (J + 1) / 2], b[C];
  double lam[J], del[C], zc[C], zl[J], ze, yc[C], yl[J], ye;
#define SI(r, s) Si[(r) >= (s) ? (r) * ((r) + 1) / 2 + (s) : (s) * ((s) + 1) / 2 + (r)]
#define RHO_MUL(v) (UNIT ? (v) : __dmul_rn(rho, (v)))
#define RI_MUL(v) (UNIT ? (v) : __dmul_rn(ri, (v)))

  const long long n_src = pass.rq_in ? (long long)*pass.rq_in_n : dev_count(n_inst, d_n);
  while (true) {
    // ---- tail compaction (see AdmmPass): once the work source is drained, a warp left with
    // fewer than pass.dump_below live lanes parks their iterates in their own x / zy slots,
    // queues them for the next, densely packed pass and retires
    if (pass.dump_below > 0) {
      const unsigned live = __ballot_sync(0xffffffffu, inst >= 0);
      if (live && __popc(live) < pass.dump_below && __any_sync(0xffffffffu, inst == -2)) {
        if (inst >= 0) {
          double* xo = x_out + inst * NV;
          double* zo = zy_out + inst * 2 * MC;
#pragma unroll
          for (int j = 0; j < J; ++j) { xo[j] = lam[j]; zo[C + j] = zl[j]; zo[MC + C + j] = yl[j]; }
#pragma unroll
          for (int c = 0; c < C; ++c) { xo[J + c] = del[c]; zo[c] = zc[c]; zo[MC + c] = yc[c]; }
          zo[MC - 1] = ze;
          zo[2 * MC - 1] = ye;
          it_out[inst] = it;
        }
        // queue the live lanes (warp-aggregated append; the whole warp is here)
        const int leader = __ffs(live) - 1;
        unsigned long long qb = 0;
        if (lane == leader) qb = atomicAdd(pass.rq_out_n, (unsigned long long)__popc(live));
        qb = __shfl_sync(0xffffffffu, qb, leader);
        if (inst >= 0) pass.rq_out[qb + __popc(live & ((1u << lane) - 1u))] = (int)inst;
        inst = -2;
      }
    }
    if (pass.park_after > 0) {
      const bool park = inst >= 0 && it >= pass.park_after;
      const unsigned pk = __ballot_sync(0xffffffffu, park);
      if (pk) {
        if (park) {
          double* xo = x_out + inst * NV;
          double* zo = zy_out + inst * 2 * MC;
#pragma unroll
          for (int j = 0; j < J; ++j) { xo[j] = lam[j]; zo[C + j] = zl[j]; zo[MC + C + j] = yl[j]; }
#pragma unroll
          for (int c = 0; c < C; ++c) { xo[J + c] = del[c]; zo[c] = zc[c]; zo[MC + c] = yc[c]; }
          zo[MC - 1] = ze;
          zo[2 * MC - 1] = ye;
          it_out[inst] = it;
        }
        const int leader = __ffs(pk) - 1;
        unsigned long long qb = 0;
        if (lane == leader) qb = atomicAdd(pass.rq_out_n, (unsigned long long)__popc(pk));
        qb = __shfl_sync(0xffffffffu, qb, leader);
        if (park) {
          pass.rq_out[qb + __popc(pk & ((1u << lane) - 1u))] = (int)inst;
          inst = -1;  // this lane takes new work
        }
      }
    }
    // ---- refill lanes whose instance terminated (one atomic per warp)
    const unsigned need = __ballot_sync(0xffffffffu, inst == -1);
    if (need) {
      unsigned long long base = 0;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base = atomicAdd(next, (unsigned long long)__popc(need));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (inst == -1) {
        const unsigned long long my = base + __popc(need & ((1u << lane) - 1u));
        inst = (long long)my < n_src ? (pass.rq_in ? (long long)pass.rq_in[my] : (long long)my) : -2;
        if (inst >= 0) {  // constants from k_qp_setup
          using K = QpConsts<G, M, C, CANON>;
          const double* o = consts + inst;
#pragma unroll
          for (int k = 0; k < K::NS; ++k) Si[k] = o[k * n_inst];
#pragma unroll
          for (int r = 0; r < K::R; ++r)
#pragma unroll
            for (int j = 0; j < J; ++j) Q.q[r][j] = o[(K::NS + r * J + j) * n_inst];
#pragma unroll
          for (int c = 0; c < C; ++c) b[c] = o[(K::NS + K::NQ + c) * n_inst];
        }
        if (inst >= 0 && pass.rq_in) {  // resume a parked instance exactly where it stopped
          const double* xo = x_out + inst * NV;
          const double* zo = zy_out + inst * 2 * MC;
#pragma unroll
          for (int j = 0; j < J; ++j) { lam[j] = xo[j]; zl[j] = zo[C + j]; yl[j] = zo[MC + C + j]; }
#pragma unroll
          for (int c = 0; c < C; ++c) { del[c] = xo[J + c]; zc[c] = zo[c]; yc[c] = zo[MC + c]; }
          ze = zo[MC - 1];
          ye = zo[2 * MC - 1];
          it = it_out[inst];
        } else {
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

    // ---- a batch of iterations (qpsolver.py:164-211)
#pragma unroll 1
    for (int k = 0; k < qp.batch; ++k) {
      if (inst < 0) break;
      ++it;
      double rdel[C], tC[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double wc = UNIT ? __dsub_rn(zc[c], yc[c]) : __fma_rn(rho, zc[c], -yc[c]);  // (R z - y)_c
        rdel[c] = __fma_rn(sig, del[c], -wc);                                            // sigma delta - w_c
        tC[c] = __fma_rn(kp, rdel[c], wc);
      }
      const double we = __fma_rn(req, ze, -ye);
      double rv[J], fT[QOps<G, M, C, CANON>::R];
      Q.fold(tC, fT);
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const double wl = UNIT ? __dsub_rn(zl[j], yl[j]) : __fma_rn(rho, zl[j], -yl[j]);
        rv[j] = Q.tmulf(j, fT, __fma_rn(sig, lam[j], __dadd_rn(wl, we)));
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
      bool conv = true;     // every |(A x - z)_i| <= eps_p and |(P x + A'y)_j| <= eps_d
      double dyc[C], dyl[J];
      double sa = 0.0;
      double maxAx = 0.0, maxz = 1.0, maxPx = 0.0, maxATy = 0.0, rprim = 0.0, rdual = 0.0;  // REL only
#pragma unroll
      for (int j = 0; j < J; ++j) {
        sa += a[j];
        const double zr = RELAX(a[j], zl[j]);
        const double zn = clip_nonneg(__dadd_rn(zr, RI_MUL(yl[j])));
        const double yn = __dadd_rn(yl[j], RHO_MUL(__dsub_rn(zr, zn)));
        dyl[j] = __dsub_rn(yn, yl[j]);
        sign_ok &= not_pos(dyl[j]);
        lam[j] = RELAX(a[j], lam[j]);
        zl[j] = zn;
        yl[j] = yn;
        const double r = __dsub_rn(lam[j], zn);
        if (REL) {
          rprim = fmax(rprim, fabs(r)); maxAx = fmax(maxAx, fabs(lam[j])); maxz = fmax(maxz, fabs(zn));
        } else {
          conv &= fabs(r) <= eps;
        }
      }
      double qa[C];
      Q.mul(a, qa);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double d = __fma_rn(rdel[c], ikdd, kp * qa[c]);
        const double zr = RELAX(__dsub_rn(qa[c], d), zc[c]);
        const double zn = clip_upper(__dadd_rn(zr, RI_MUL(yc[c])), b[c]);
        const double yn = __dadd_rn(yc[c], RHO_MUL(__dsub_rn(zr, zn)));
        dyc[c] = __dsub_rn(yn, yc[c]);
        sign_ok &= not_neg(dyc[c]);
        del[c] = RELAX(d, del[c]);
        zc[c] = zn;
        yc[c] = yn;
      }
      double dye;
      {
        const double zr = RELAX(sa, ze);
        const double yn = __dadd_rn(ye, __dmul_rn(req, __dsub_rn(zr, 1.0)));  // z clipped to [1, 1]
        dye = __dsub_rn(yn, ye);
        ze = 1.0;
        ye = yn;
      }
      // termination test at the new iterate (qpsolver.py:176-188)
      double sl = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) sl = __dadd_rn(sl, lam[j]);
      {
        const double r = __dsub_rn(sl, 1.0);
        if (REL) { rprim = fmax(rprim, fabs(r)); maxAx = fmax(maxAx, fabs(sl)); }
        else conv &= fabs(r) <= eps;
      }
      // (forming these only when the cheaper tests passed was tried: the branch is taken by
      // some lane of most warps and the kernel got 2% slower)
      {
        double ql[C];
        Q.mul(lam, ql);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double ax = __dsub_rn(ql[c], del[c]);
          const double r = __dsub_rn(ax, zc[c]);
          if (REL) {
            rprim = fmax(rprim, fabs(r)); maxAx = fmax(maxAx, fabs(ax)); maxz = fmax(maxz, fabs(zc[c]));
          } else {
            conv &= fabs(r) <= eps;
          }
        }
        double fY[QOps<G, M, C, CANON>::R];
        Q.fold(yc, fY);
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const double acc = Q.tmulf(j, fY, __dadd_rn(yl[j], ye));
          if (REL) { rdual = fmax(rdual, fabs(acc)); maxATy = fmax(maxATy, fabs(acc)); }
          else conv &= fabs(acc) <= eps;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          // P x - ... = 2 delta_c - y_c; 2 delta_c is exact, so one FMA rounds like the subtraction
          const double r = __fma_rn(2.0, del[c], -yc[c]);
          if (REL) {
            rdual = fmax(rdual, fabs(r)); maxPx = fmax(maxPx, fabs(__dmul_rn(2.0, del[c])));
            maxATy = fmax(maxATy, fabs(yc[c]));
          } else {
            conv &= fabs(r) <= eps;
          }
        }
      }
      if (REL) conv = rprim <= eps + qp.eps_rel * fmax(maxAx, maxz) && rdual <= eps + qp.eps_rel * fmax(maxPx, maxATy);

      int status = conv ? BZG_SOLVED : -1;
      if (!conv && sign_ok) {
        // primal-infeasibility certificate (qpsolver.py:193-209): with every dy_i on a finite
        // bound, support = sum_c b_c dy_c + dy_eq.  The three conditions are tested cheapest
        // first (few lanes of a warp take this branch, so its length is paid warp-wide).
        // supp <= -eps_pinf * dmax with dmax > 1e-13 implies supp < 0: test that first
        double supp = 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) supp = __dadd_rn(supp, __dmul_rn(b[c], dyc[c]));
        supp = __dadd_rn(supp, dye);
        double dmax = 0.0;
        if (supp < 0.0) {
          dmax = fabs(dye);
#pragma unroll
          for (int j = 0; j < J; ++j) dmax = max_nn(dmax, fabs(dyl[j]));
#pragma unroll
          for (int c = 0; c < C; ++c) dmax = max_nn(dmax, fabs(dyc[c]));
        }
        if (dmax > 1e-13) {
          const double lim = qp.eps_pinf * dmax;
          if (supp <= -lim) {  // then ||A'dy||_inf <= lim: delta columns, then lambda columns
            bool small = true;
#pragma unroll
            for (int c = 0; c < C; ++c) small &= fabs(dyc[c]) <= lim;
#pragma unroll
            for (int j = 0; j < J; ++j) small &= fabs(Q.tmul(j, dyc, __dadd_rn(dyl[j], dye))) <= lim;
            if (small) status = BZG_INFEASIBLE;
          }
        }
      }
      if (status < 0 && it >= qp.max_iter) status = BZG_MAX_ITER;
      if (status >= 0) {
        st_out[inst] = (int8_t)status;
        it_out[inst] = it;
        double* xo = x_out + inst * NV;
        double* zo = zy_out + inst * 2 * MC;
#pragma unroll
        for (int j = 0; j < J; ++j) { xo[j] = lam[j]; zo[C + j] = zl[j]; zo[MC + C + j] = yl[j]; }
#pragma unroll
        for (int c = 0; c < C; ++c) { xo[J + c] = del[c]; zo[c] = zc[c]; zo[MC + c] = yc[c]; }
        zo[MC - 1] = ze;
        zo[2 * MC - 1] = ye;
        inst = -1;
      }
    }
  }
#undef SI
#undef RELAX
#undef RHO_MUL
#undef RI_MUL
}

}  // namespace
}  // namespace bzg
