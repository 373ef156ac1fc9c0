// Cut-QP verdict selection and active-set polish (one thread per instance).  Included by k_cut.cu.
#pragma once

namespace bzg {
namespace {

// Verdict from the ADMM iterate and the polish work list.  The polish only changes x,
// never the status (qpsolver.py:301-303), and the verdict is SOLVED and ||delta|| > eps_cut
// (graph.py:329): MAX_ITER / INFEASIBLE instances are unsafe whatever x, and a SOLVED
// instance whose ADMM ||delta|| is at least `screen` cannot drop below eps_cut when
// polished (both iterates are 1e-7-feasible, the ADMM
// one is 1e-7-KKT with exact complementarity, so both norms are within ~1e-3 of the
// optimal ||delta*||).  screen <= 0 polishes every SOLVED instance, as the reference does.
//
// The residual maxima of the selected instances are formed by the polish (qp_residuals).
template <int G, int M, int C>
__global__ void k_qp_select(long long n_inst, const unsigned long long* __restrict__ d_n, int polish, double screen,
                            double eps_cut, const int8_t* __restrict__ st, const double* __restrict__ x,
                            double* __restrict__ delta_out, uint8_t* __restrict__ safe_out, int* __restrict__ list,
                            unsigned long long* __restrict__ n_list) {
  BZG_PDL_ENTRY();
  constexpr int J = 2 * G, NV = J + C;
  const long long n = dev_count(n_inst, d_n);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n; t0 += stride) {  // warp-uniform
    const long long t = t0 + threadIdx.x;
    bool need = false;
    if (t < n) {
      double s = 0.0;
#pragma unroll
      for (int c = J; c < NV; ++c) s = __fma_rn(x[t * NV + c], x[t * NV + c], s);
      const double dl = sqrt(s);
      const bool solved = st[t] == BZG_SOLVED;
      delta_out[t] = dl;
      safe_out[t] = (uint8_t)(solved && dl > eps_cut);
      // polish 1: SOLVED only (the verdict is all cut_graph uses); 2: also MAX_ITER, whose
      // polished x the reference returns from solve() (cut_qp's ||delta||)
      need = polish && (solved || (polish == 2 && st[t] == BZG_MAX_ITER)) && (screen <= 0.0 || dl < screen);
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
}

// rp = max |A x - z|, rd = max |P x + q + A'y| (qpsolver.py:179-180) at the terminal ADMM
// iterate (x, z, y): recorded with the snapshot in the reference (qpsolver.py:191), formed
// here by the polish for its own instances (dense lanes) instead of by k_qp_select, where only
// the polish candidates among each warp's 32 instances needed them.
template <int G, int M, int C>
__device__ __forceinline__ void qp_residuals(const double (&Q)[C][2 * G], const double* __restrict__ xv,
                                             const double* __restrict__ z, double& rp, double& rd) {
  constexpr int J = 2 * G, MC = C + J + 1;
  const double* y = z + MC;
  double sl = 0.0;
  rp = 0.0;
  rd = 0.0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    sl = __dadd_rn(sl, xv[j]);
    rp = fmax(rp, fabs(__dsub_rn(xv[j], z[C + j])));
    double acc = __dadd_rn(y[C + j], y[MC - 1]);
#pragma unroll
    for (int c = 0; c < C; ++c) acc = __fma_rn(Q[c][j], y[c], acc);
    rd = fmax(rd, fabs(acc));
  }
  rp = fmax(rp, fabs(__dsub_rn(sl, z[MC - 1])));
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) acc = __fma_rn(Q[c][j], xv[j], acc);
    rp = fmax(rp, fabs(__dsub_rn(__dsub_rn(acc, xv[J + c]), z[c])));
    rd = fmax(rd, fabs(__dsub_rn(__dmul_rn(2.0, xv[J + c]), y[c])));
  }
}

// Active-set polish (qpsolver.py:236-279), one THREAD per selected SOLVED instance.
//
// The reference solves the regularised reduced KKT system
//   K = [[P + d I, G'], [G, -d I]],  d = 1e-8,  G = active rows of A,  rhs = [-q; g]
// by LU with partial pivoting (np.linalg.solve) plus two refinement steps against K.
// Here K is solved by exact block elimination with well-conditioned pivots, then a small
// dense LU with partial pivoting:
//   * delta_c (pivot 2 + d): it appears only in obstacle row c of G (coefficient -1);
//   * each active lambda-bound row j (G row e_j) with lambda_j: the 2x2 pivot
//     [[d, 1], [1, -d]] (determinant -(1 + d^2));
//   * the remaining "core" unknowns (free lambda_j, nu of active obstacle rows, nu of the
//     sum row) form an (J + C + 1)-dim system with unused slots as identity rows.
// Residuals of the two refinement steps are taken against the full K, so the iterate
// converges to the same regularised solution as the reference; then the acceptance test
// max(rp', rd') < max(rp, rd).
constexpr int kPolishThreads = 64;

template <int G, int M, int C>
constexpr int polish_dim() { return 2 * G + C + 1; }  // core: J + C + 1

template <int G, int M, int C>
__global__ void __launch_bounds__(kPolishThreads) k_qp_polish(
    DParams dp, const double* __restrict__ Vx, const int* __restrict__ src, const int* __restrict__ dst,
    const ObsRec<M, obs_cap<C>()>* __restrict__ obs, const unsigned long long* __restrict__ pend, const int* __restrict__ list,
    long long n_list, double eps_cut, double* __restrict__ x_io, const double* __restrict__ zy,
    double* __restrict__ delta_out, uint8_t* __restrict__ safe_out, const int8_t* __restrict__ st) {
  BZG_PDL_ENTRY();
  constexpr int J = 2 * G, NV = J + C, MC = C + J + 1, NC = J + C + 1;
  constexpr int BS = kPolishThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Rm = reinterpret_cast<double*>(smem_raw) + threadIdx.x;  // core (r, c) at Rm[(r*NC+c)*BS]
  double* Ym = Rm + NC * NC * BS;                                   // work vector y[r] at Ym[r*BS]
  const long long li = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= n_list) return;
  const long long inst = list[li];
  auto R = [&](int r, int c) -> double& { return Rm[(r * NC + c) * BS]; };
  auto Y = [&](int r) -> double& { return Ym[r * BS]; };

  double x[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) x[t] = x_io[inst * NV + t];
  double Q[C][J], b[C];
  load_instance<G, M, C>(dp, Vx, src, dst, obs, pend[inst], Q, b);
  double rp, rd;
  qp_residuals<G, M, C>(Q, x_io + inst * NV, zy + inst * 2 * MC, rp, rd);
  // constraint slot i of A (graph.py:275-281): i < C obstacle row [Q_i, -e_i];
  // C <= i < C+J lambda bound [e_{i-C}, 0]; i = C+J the sum row [1..1, 0]
  auto Gl = [&](int i, int j) -> double {  // lambda part of row i (compile-time i, j)
    return i < C ? Q[i < C ? i : 0][j] : (i < C + J ? (i - C == j ? 1.0 : 0.0) : 1.0);
  };
  auto a_dot = [&](int i, const double (&v)[NV]) -> double {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const double g = Gl(i, j);
      if (g != 0.0) acc = __fma_rn(g, v[j], acc);
    }
    if (i < C) acc = __fma_rn(-1.0, v[J + (i < C ? i : 0)], acc);
    return acc;
  };
  auto lo_of = [&](int i) -> double { return i < C ? -INFINITY : (i < C + J ? 0.0 : 1.0); };
  auto hi_of = [&](int i) -> double { return i < C ? b[i < C ? i : 0] : (i < C + J ? INFINITY : 1.0); };
  // active set at z = A x (qpsolver.py:245-249)
  const double tol = fmax(1e-7, 10.0 * rp);
  unsigned long long act = 0, atlo = 0;  // MC = C + J + 1 rows: up to 41 with kObsRowsBig
#pragma unroll
  for (int i = 0; i < MC; ++i) {
    const double zi = a_dot(i, x);
    const bool l_ = __dsub_rn(zi, lo_of(i)) <= tol, u_ = __dsub_rn(hi_of(i), zi) <= tol;
    act |= (unsigned long long)(l_ || u_) << i;
    atlo |= (unsigned long long)l_ << i;
  }
  bool accept = false;
  double xp[NV];
  if (act) {
    const double reg = 1e-8, i2 = 1.0 / (2.0 + reg), e2 = reg / (1.0 + reg * reg), r2 = 1.0 / (1.0 + reg * reg);
    auto a_on = [&](int i) -> bool { return act >> i & 1ull; };
    // core slot of row/column r: r < J lambda_r (used iff lambda bound r inactive),
    // J <= r < J+C nu of obstacle row r-J, r = J+C nu of the sum row
    auto core_used = [&](int r) -> bool { return r < J ? !a_on(C + r) : (r < J + C ? a_on(r - J) : a_on(C + J)); };
    auto core_row = [&](int r) -> int { return r < J ? -1 : (r < J + C ? r - J : C + J); };  // constraint slot
    // ---- build the core matrix (compile-time indices keep Q in registers)
#pragma unroll
    for (int r = 0; r < NC; ++r)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        double v = 0.0;
        if (!core_used(r) || !core_used(c)) {
          v = (r == c) ? 1.0 : 0.0;
        } else if (r < J && c < J) {
          v = (r == c) ? reg : 0.0;
        } else if (r < J) {
          v = Gl(core_row(c), r);
        } else if (c < J) {
          v = Gl(core_row(r), c);
        } else {
          const int i = core_row(r), k = core_row(c);
          double s = 0.0;  // sum over eliminated lambda bounds j of G[i][j] G[k][j]
#pragma unroll
          for (int j = 0; j < J; ++j)
            if (a_on(C + j)) s = __fma_rn(Gl(i, j), Gl(k, j), s);
          v = -e2 * s;
          if (r == c) v = __dsub_rn(v, i < C ? reg + i2 : reg);
        }
        R(r, c) = v;
      }
    // ---- LU with partial pivoting (first max |.|, reciprocal scaling as dgetf2)
    unsigned char perm[NC];
#pragma unroll
    for (int r = 0; r < NC; ++r) perm[r] = (unsigned char)r;
    bool singular = false;
#pragma unroll 1
    for (int cc = 0; cc < NC; ++cc) {
      int piv = cc;
      double best = fabs(R(cc, cc));
#pragma unroll 1
      for (int r = cc + 1; r < NC; ++r) {
        const double v = fabs(R(r, cc));
        if (v > best) { best = v; piv = r; }
      }
      if (best == 0.0) { singular = true; break; }
      if (piv != cc) {
#pragma unroll 1
        for (int c = 0; c < NC; ++c) {
          const double t = R(cc, c);
          R(cc, c) = R(piv, c);
          R(piv, c) = t;
        }
        const unsigned char t = perm[cc];
        perm[cc] = perm[piv];
        perm[piv] = t;
      }
      const double rpv = 1.0 / R(cc, cc);
#pragma unroll 1
      for (int r = cc + 1; r < NC; ++r) {
        const double l = __dmul_rn(R(r, cc), rpv);
        R(r, cc) = l;
        if (l != 0.0) {
#pragma unroll 1
          for (int c = cc + 1; c < NC; ++c) R(r, c) = __fma_rn(-l, R(cc, c), R(r, c));
        }
      }
    }
    if (!singular) {
      // solve K w = (rx, rn) for w = (x (NV), nu (MC slots; 0 on inactive slots))
      auto solve = [&](const double (&rx)[NV], const double (&rn)[MC], double (&wx)[NV], double (&wn)[MC]) {
        double rr[MC];  // constraint rhs after eliminating delta
#pragma unroll
        for (int i = 0; i < MC; ++i) rr[i] = (i < C && a_on(i)) ? __fma_rn(rx[J + (i < C ? i : 0)], i2, rn[i]) : rn[i];
        double lamb[J];  // a_j + e2 (b_j - d a_j): the eliminated lambda_j without its nu coupling
#pragma unroll
        for (int j = 0; j < J; ++j) lamb[j] = __fma_rn(e2, __fma_rn(-reg, rr[C + j], rx[j]), rr[C + j]);
        double v[NC];
#pragma unroll
        for (int r = 0; r < NC; ++r) {
          double t = 0.0;
          if (core_used(r)) {
            if (r < J) {
              t = rx[r];
            } else {
              const int i = core_row(r);
              t = rr[i];
#pragma unroll
              for (int j = 0; j < J; ++j)
                if (a_on(C + j)) t = __fma_rn(-Gl(i, j), lamb[j], t);
            }
          }
          v[r] = t;
        }
#pragma unroll 1
        for (int r = 0; r < NC; ++r) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < NC; ++q) if (q == perm[r]) t = v[q];
#pragma unroll 1
          for (int c = 0; c < r; ++c) t = __fma_rn(-R(r, c), Y(c), t);
          Y(r) = t;
        }
#pragma unroll 1
        for (int r = NC - 1; r >= 0; --r) {
          double t = Y(r);
#pragma unroll 1
          for (int c = r + 1; c < NC; ++c) t = __fma_rn(-R(r, c), Y(c), t);
          Y(r) = t / R(r, r);
        }
        double core[NC];
#pragma unroll
        for (int r = 0; r < NC; ++r) core[r] = core_used(r) ? Y(r) : 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) wn[i] = 0.0;
#pragma unroll
        for (int r = J; r < NC; ++r) wn[core_row(r)] = core[r];
        // recover the eliminated lambda-bound pairs, then lambda_free, then delta
#pragma unroll
        for (int j = 0; j < J; ++j) {
          if (a_on(C + j)) {
            double t = __fma_rn(-reg, rr[C + j], rx[j]);
#pragma unroll
            for (int r = J; r < NC; ++r) t = __fma_rn(-Gl(core_row(r), j), core[r], t);
            wn[C + j] = __dmul_rn(t, r2);
            wx[j] = __fma_rn(reg, wn[C + j], rr[C + j]);
          } else {
            wx[j] = core[j];
          }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) wx[J + c] = __dmul_rn(__dadd_rn(rx[J + c], a_on(c) ? wn[c] : 0.0), i2);
      };
      // K w for the full system (rows: x then active constraint slots)
      auto kmul = [&](const double (&wx)[NV], const double (&wn)[MC], double (&ox)[NV], double (&on)[MC]) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          double acc = __dmul_rn(reg, wx[j]);
#pragma unroll
          for (int i = 0; i < MC; ++i)
            if (a_on(i)) acc = __fma_rn(Gl(i, j), wn[i], acc);
          ox[j] = acc;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) ox[J + c] = __fma_rn(2.0 + reg, wx[J + c], a_on(c) ? -wn[c] : 0.0);
#pragma unroll
        for (int i = 0; i < MC; ++i) on[i] = a_on(i) ? __fma_rn(-reg, wn[i], a_dot(i, wx)) : 0.0;
      };
      double bx[NV], bn[MC], wx[NV], wn[MC];
#pragma unroll
      for (int t = 0; t < NV; ++t) bx[t] = 0.0;  // -q = 0
#pragma unroll
      for (int i = 0; i < MC; ++i) bn[i] = a_on(i) ? ((atlo >> i & 1ull) ? lo_of(i) : hi_of(i)) : 0.0;
      solve(bx, bn, wx, wn);
#pragma unroll 1
      for (int rep = 0; rep < 2; ++rep) {
        double kx[NV], kn[MC], rx[NV], rn[MC], dx[NV], dn[MC];
        kmul(wx, wn, kx, kn);
#pragma unroll
        for (int t = 0; t < NV; ++t) rx[t] = __dsub_rn(bx[t], kx[t]);
#pragma unroll
        for (int i = 0; i < MC; ++i) rn[i] = __dsub_rn(bn[i], kn[i]);
        solve(rx, rn, dx, dn);
#pragma unroll
        for (int t = 0; t < NV; ++t) wx[t] = __dadd_rn(wx[t], dx[t]);
#pragma unroll
        for (int i = 0; i < MC; ++i) wn[i] = __dadd_rn(wn[i], dn[i]);
      }
      // acceptance (qpsolver.py:271-279)
      double upv = 0.0, lov = 0.0;
#pragma unroll
      for (int i = 0; i < MC; ++i) {
        const double zi = a_dot(i, wx);
        upv = fmax(upv, fmax(__dsub_rn(zi, hi_of(i)), 0.0));
        lov = fmax(lov, fmax(__dsub_rn(lo_of(i), zi), 0.0));
      }
      double rdt = 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j) {  // |P x + A' y| with y = nu on active slots
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) acc = __fma_rn(Gl(i, j), wn[i], acc);
        rdt = fmax(rdt, fabs(acc));
      }
#pragma unroll
      for (int c = 0; c < C; ++c) rdt = fmax(rdt, fabs(__fma_rn(-1.0, wn[c], __dmul_rn(2.0, wx[J + c]))));
      if (fmax(__dadd_rn(upv, lov), rdt) < fmax(rp, rd)) {
        accept = true;
#pragma unroll
        for (int t = 0; t < NV; ++t) xp[t] = wx[t];
      }
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double dc = accept ? xp[J + c] : x[J + c];
    s = __fma_rn(dc, dc, s);
  }
  const double dl = sqrt(s);
  delta_out[inst] = dl;
  safe_out[inst] = (uint8_t)(st[inst] == BZG_SOLVED && dl > eps_cut);
}

// Register-resident polish: the same regularised KKT system and two refinement steps, solved
// through a Schur complement on the multipliers of the active obstacle rows and the sum row
// (at most C + 1 unknowns) instead of a dense LU on the 11-slot core in shared memory.
//   delta_c = (rx_dc + nu_c) / (2 + d)                       (delta pivot, as above)
//   lambda_j = alpha_j - beta_j u_j,  u_j = sum_i g_i(j) nu_i  (g: Q rows, the sum row's ones)
//     free j:   alpha_j = rx_j / d,                       beta_j = 1 / d
//     bound j:  alpha_j = rn_j + e (rx_j - d rn_j),        beta_j = e = d / (1 + d^2)
//               (nu_j = (rx_j - d rn_j - u_j) / (1 + d^2), the 2x2 bound pivot)
//   S nu = t,   S_ik = sum_j beta_j g_i(j) g_k(j) + d_i [i = k],  t_i = sum_j g_i(j) alpha_j - rhs_i
// S is symmetric positive definite (beta, d_i > 0): Cholesky, no pivoting.  K has condition
// ~1/d either way, so this solve and the reference's LU reach the regularised solution to the
// same forward accuracy after the refinement steps (residuals against the full K, as above).
template <int G, int M, int C>
__device__ __forceinline__ void polish_one_reg(
    long long inst, const DParams& dp, const double* __restrict__ Vx, const int* __restrict__ src,
    const int* __restrict__ dst, const ObsRec<M, obs_cap<C>()>* __restrict__ obs, const unsigned long long* __restrict__ pend,
    double eps_cut, double* __restrict__ x_io, const double* __restrict__ zy, double* __restrict__ delta_out,
    uint8_t* __restrict__ safe_out, const int8_t* __restrict__ st) {
  constexpr int J = 2 * G, NV = J + C, MC = C + J + 1, NS = C + 1;
  double x[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) x[t] = x_io[inst * NV + t];
  double Q[C][J], b[C];
  load_instance<G, M, C>(dp, Vx, src, dst, obs, pend[inst], Q, b);
  double rp, rd;
  qp_residuals<G, M, C>(Q, x_io + inst * NV, zy + inst * 2 * MC, rp, rd);
  auto Gl = [&](int i, int j) -> double {  // lambda part of constraint row i (compile-time i, j)
    return i < C ? Q[i < C ? i : 0][j] : (i < C + J ? (i - C == j ? 1.0 : 0.0) : 1.0);
  };
  auto a_dot = [&](int i, const double (&v)[NV]) -> double {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const double g = Gl(i, j);
      if (g != 0.0) acc = __fma_rn(g, v[j], acc);
    }
    if (i < C) acc = __fma_rn(-1.0, v[J + (i < C ? i : 0)], acc);
    return acc;
  };
  auto lo_of = [&](int i) -> double { return i < C ? -INFINITY : (i < C + J ? 0.0 : 1.0); };
  auto hi_of = [&](int i) -> double { return i < C ? b[i < C ? i : 0] : (i < C + J ? INFINITY : 1.0); };
  const double tol = fmax(1e-7, 10.0 * rp);
  unsigned long long act = 0, atlo = 0;  // MC = C + J + 1 rows: up to 41 with kObsRowsBig
#pragma unroll
  for (int i = 0; i < MC; ++i) {
    const double zi = a_dot(i, x);
    const bool l_ = __dsub_rn(zi, lo_of(i)) <= tol, u_ = __dsub_rn(hi_of(i), zi) <= tol;
    act |= (unsigned long long)(l_ || u_) << i;
    atlo |= (unsigned long long)l_ << i;
  }
  bool accept = false;
  double xp[NV];
  if (act) {
    const double reg = 1e-8, i2 = 1.0 / (2.0 + reg), e2 = reg / (1.0 + reg * reg), r2 = 1.0 / (1.0 + reg * reg);
    const double ireg = 1.0 / reg;
    auto a_on = [&](int i) -> bool { return act >> i & 1ull; };
    auto bound = [&](int j) -> bool { return a_on(C + j); };
    auto used = [&](int s) -> bool { return s < C ? a_on(s) : a_on(C + J); };  // nu slot s: obstacle row / sum row
    auto gs = [&](int s, int j) -> double { return s < C ? Q[s < C ? s : 0][j] : 1.0; };
    // ---- S = sum_j beta_j g g' + diag(d), Cholesky (compile-time indices: registers only)
    double L[NS][NS];
#pragma unroll
    for (int i = 0; i < NS; ++i)
#pragma unroll
      for (int k = 0; k <= i; ++k) {
        double v;
        if (!used(i) || !used(k)) {
          v = i == k ? 1.0 : 0.0;
        } else {
          v = 0.0;
#pragma unroll
          for (int j = 0; j < J; ++j) v = __fma_rn(__dmul_rn(bound(j) ? e2 : ireg, gs(i, j)), gs(k, j), v);
          if (i == k) v = __dadd_rn(v, i < C ? i2 + reg : reg);
        }
        L[i][k] = v;
      }
    double Ld[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) {
#pragma unroll
      for (int k = 0; k < i; ++k) {
        double t = L[i][k];
#pragma unroll
        for (int q = 0; q < k; ++q) t = __fma_rn(-L[i][q], L[k][q], t);
        L[i][k] = t * Ld[k];
      }
      double dd = L[i][i];
#pragma unroll
      for (int q = 0; q < i; ++q) dd = __fma_rn(-L[i][q], L[i][q], dd);
      L[i][i] = sqrt(dd);
      Ld[i] = 1.0 / L[i][i];
    }
    auto solve = [&](const double (&rx)[NV], const double (&rn)[MC], double (&wx)[NV], double (&wn)[MC]) {
      double alpha[J];
#pragma unroll
      for (int j = 0; j < J; ++j)
        alpha[j] = bound(j) ? __fma_rn(e2, __fma_rn(-reg, rn[C + j], rx[j]), rn[C + j]) : __dmul_rn(rx[j], ireg);
      double t[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        double acc = 0.0;
        if (used(s)) {
          const double rhs = s < C ? __fma_rn(rx[J + (s < C ? s : 0)], i2, rn[s < C ? s : 0]) : rn[C + J];
#pragma unroll
          for (int j = 0; j < J; ++j) acc = __fma_rn(gs(s, j), alpha[j], acc);
          acc = __dsub_rn(acc, rhs);
        }
        t[s] = acc;
      }
#pragma unroll
      for (int i = 0; i < NS; ++i) {  // L y = t
        double v = t[i];
#pragma unroll
        for (int k = 0; k < i; ++k) v = __fma_rn(-L[i][k], t[k], v);
        t[i] = v * Ld[i];
      }
#pragma unroll
      for (int i = NS - 1; i >= 0; --i) {  // L' nu = y
        double v = t[i];
#pragma unroll
        for (int k = i + 1; k < NS; ++k) v = __fma_rn(-L[k][i], t[k], v);
        t[i] = v * Ld[i];
      }
#pragma unroll
      for (int i = 0; i < MC; ++i) wn[i] = 0.0;
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (used(s)) wn[s < C ? s : C + J] = t[s];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        double u = 0.0;
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (used(s)) u = __fma_rn(gs(s, j), t[s], u);
        if (bound(j)) {
          wn[C + j] = __dmul_rn(__dsub_rn(__fma_rn(-reg, rn[C + j], rx[j]), u), r2);
          wx[j] = __fma_rn(reg, wn[C + j], rn[C + j]);
        } else {
          wx[j] = __fma_rn(-ireg, u, alpha[j]);
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) wx[J + c] = __dmul_rn(__dadd_rn(rx[J + c], a_on(c) ? wn[c] : 0.0), i2);
    };
    auto kmul = [&](const double (&wx)[NV], const double (&wn)[MC], double (&ox)[NV], double (&on)[MC]) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        double acc = __dmul_rn(reg, wx[j]);
#pragma unroll
        for (int i = 0; i < MC; ++i)
          if (a_on(i)) acc = __fma_rn(Gl(i, j), wn[i], acc);
        ox[j] = acc;
      }
#pragma unroll
      for (int c = 0; c < C; ++c) ox[J + c] = __fma_rn(2.0 + reg, wx[J + c], a_on(c) ? -wn[c] : 0.0);
#pragma unroll
      for (int i = 0; i < MC; ++i) on[i] = a_on(i) ? __fma_rn(-reg, wn[i], a_dot(i, wx)) : 0.0;
    };
    double bx[NV], bn[MC], wx[NV], wn[MC];
#pragma unroll
    for (int t = 0; t < NV; ++t) bx[t] = 0.0;  // -q = 0
#pragma unroll
    for (int i = 0; i < MC; ++i) bn[i] = a_on(i) ? ((atlo >> i & 1ull) ? lo_of(i) : hi_of(i)) : 0.0;
    solve(bx, bn, wx, wn);
#pragma unroll 1
    for (int rep = 0; rep < 2; ++rep) {
      double kx[NV], kn[MC], rx[NV], rn[MC], dx[NV], dn[MC];
      kmul(wx, wn, kx, kn);
#pragma unroll
      for (int t = 0; t < NV; ++t) rx[t] = __dsub_rn(bx[t], kx[t]);
#pragma unroll
      for (int i = 0; i < MC; ++i) rn[i] = __dsub_rn(bn[i], kn[i]);
      solve(rx, rn, dx, dn);
#pragma unroll
      for (int t = 0; t < NV; ++t) wx[t] = __dadd_rn(wx[t], dx[t]);
#pragma unroll
      for (int i = 0; i < MC; ++i) wn[i] = __dadd_rn(wn[i], dn[i]);
    }
    // acceptance (qpsolver.py:271-279)
    double upv = 0.0, lov = 0.0;
#pragma unroll
    for (int i = 0; i < MC; ++i) {
      const double zi = a_dot(i, wx);
      upv = fmax(upv, fmax(__dsub_rn(zi, hi_of(i)), 0.0));
      lov = fmax(lov, fmax(__dsub_rn(lo_of(i), zi), 0.0));
    }
    double rdt = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {  // |P x + A' y| with y = nu on active slots
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < MC; ++i) acc = __fma_rn(Gl(i, j), wn[i], acc);
      rdt = fmax(rdt, fabs(acc));
    }
#pragma unroll
    for (int c = 0; c < C; ++c) rdt = fmax(rdt, fabs(__fma_rn(-1.0, wn[c], __dmul_rn(2.0, wx[J + c]))));
    if (fmax(__dadd_rn(upv, lov), rdt) < fmax(rp, rd)) {
      accept = true;
#pragma unroll
      for (int t = 0; t < NV; ++t) xp[t] = wx[t];
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const double dc = accept ? xp[J + c] : x[J + c];
    s = __fma_rn(dc, dc, s);
  }
  const double dl = sqrt(s);
  delta_out[inst] = dl;
  safe_out[inst] = (uint8_t)(st[inst] == BZG_SOLVED && dl > eps_cut);
}

// Grid-stride over the work list, its length read on the device (no host round trip between
// k_qp_select and the polish).
template <int G, int M, int C>
__global__ void __launch_bounds__(128) k_qp_polish_reg(
    DParams dp, const double* __restrict__ Vx, const int* __restrict__ src, const int* __restrict__ dst,
    const ObsRec<M, obs_cap<C>()>* __restrict__ obs, const unsigned long long* __restrict__ pend, const int* __restrict__ list,
    const unsigned long long* __restrict__ n_list, double eps_cut, double* __restrict__ x_io,
    const double* __restrict__ zy, double* __restrict__ delta_out, uint8_t* __restrict__ safe_out,
    const int8_t* __restrict__ st) {
  BZG_PDL_ENTRY();
  const long long n = (long long)*n_list;
  for (long long li = (long long)blockIdx.x * blockDim.x + threadIdx.x; li < n; li += (long long)gridDim.x * blockDim.x)
    polish_one_reg<G, M, C>(list[li], dp, Vx, src, dst, obs, pend, eps_cut, x_io, zy, delta_out, safe_out, st);
}

}  // namespace
}  // namespace bzg
