// Cut-QP verdict selection and active-set polish (one warp per instance).  Included by k_cut.cu.
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
// For the selected instances the residual maxima rp = max|A x - z|, rd = max|P x + A'y|
// (qpsolver.py:179-180) are recomputed here from the stored terminal (x, z, y), exactly as
// the reference records them with the snapshot (qpsolver.py:191).
template <int G, int M>
__global__ void k_qp_select(DParams dp, const double* __restrict__ Vx, const int* __restrict__ src,
                            const int* __restrict__ dst, const ObsRec<M>* __restrict__ obs,
                            const unsigned long long* __restrict__ pend, long long n_inst, int polish,
                            double screen, double eps_cut, const int8_t* __restrict__ st,
                            const double* __restrict__ x, const double* __restrict__ zy,
                            double* __restrict__ res_out, double* __restrict__ delta_out,
                            uint8_t* __restrict__ safe_out, int* __restrict__ list,
                            unsigned long long* __restrict__ n_list) {
  constexpr int J = 2 * G, C = 2 * M, NV = J + C, MC = C + J + 1;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  bool need = false;
  if (t < n_inst) {
    double s = 0.0;
#pragma unroll
    for (int c = J; c < NV; ++c) s = __fma_rn(x[t * NV + c], x[t * NV + c], s);
    const double dl = sqrt(s);
    const bool solved = st[t] == BZG_SOLVED;
    delta_out[t] = dl;
    safe_out[t] = (uint8_t)(solved && dl > eps_cut);
    need = polish && solved && (screen <= 0.0 || dl < screen);
    if (need) {
      double Q[C][J], b[C];
      load_instance<G, M>(dp, Vx, src, dst, obs, pend[t], Q, b);
      const double* xv = x + t * NV;
      const double* z = zy + t * 2 * MC;
      const double* y = z + MC;
      double rp = 0.0, rd = 0.0, sl = 0.0;
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
      res_out[t * 2] = rp;
      res_out[t * 2 + 1] = rd;
    }
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

// Active-set polish (qpsolver.py:236-279), one THREAD per selected SOLVED instance.
//
// The reference solves the regularised reduced KKT system
//   K = [[P + d I, G'], [G, -d I]],  d = 1e-8,  G = active rows of A,  rhs = [-q; g]
// by LU with partial pivoting (np.linalg.solve) plus two refinement steps against K.
// The delta block of P + d I is (2 + d) I and each delta_c appears only in obstacle row
// c of G (coefficient -1), so delta is eliminated exactly with the well-conditioned pivot
// 2 + d; the remaining (lambda, nu) system
//   R = [[d I_J, G_l'], [G_l, -diag(d + [obstacle row] / (2 + d))]]
// (inactive constraint slots as decoupled identity rows) is factored by LU with partial
// pivoting in this thread's slice of shared memory.  Residuals of the refinement steps
// are taken against the full K, so the iterate converges to the same regularised solution
// as the reference; then the acceptance test max(rp', rd') < max(rp, rd).
constexpr int kPolishThreads = 64;

template <int G, int M>
constexpr int polish_dim() { return 2 * G + (2 * M + 2 * G + 1); }  // J + MC

template <int G, int M>
__global__ void __launch_bounds__(kPolishThreads) k_qp_polish(
    DParams dp, const double* __restrict__ Vx, const int* __restrict__ src, const int* __restrict__ dst,
    const ObsRec<M>* __restrict__ obs, const unsigned long long* __restrict__ pend, const int* __restrict__ list,
    long long n_list, double eps_cut, double* __restrict__ x_io, const double* __restrict__ res,
    double* __restrict__ delta_out, uint8_t* __restrict__ safe_out) {
  constexpr int J = 2 * G, C = 2 * M, NV = J + C, MC = C + J + 1, NR = J + MC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Rm = reinterpret_cast<double*>(smem_raw) + threadIdx.x;  // element (r, c) at Rm[(r*NR+c)*BS]
  double* Ym = Rm + NR * NR * kPolishThreads;                      // y[r] at Ym[r*BS]
  constexpr int BS = kPolishThreads;
  const long long li = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= n_list) return;
  const long long inst = list[li];
  auto R = [&](int r, int c) -> double& { return Rm[(r * NR + c) * BS]; };

  double x[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) x[t] = x_io[inst * NV + t];
  const double rp = res[inst * 2], rd = res[inst * 2 + 1];
  double Q[C][J], b[C];
  load_instance<G, M>(dp, Vx, src, dst, obs, pend[inst], Q, b);
  // constraint rows of A (graph.py:275-281): i < C: [Q_i, -e_i]; C <= i < C+J: [e_{i-C}, 0];
  // i = C+J: [1..1, 0]
  auto a_dot = [&](int i, const double (&v)[NV]) -> double {  // A_i . v, FMA chain over columns
    double acc = 0.0;
    if (i < C) {
#pragma unroll
      for (int j = 0; j < J; ++j) acc = __fma_rn(Q[i][j], v[j], acc);
#pragma unroll
      for (int c = 0; c < C; ++c) if (c == i) acc = __fma_rn(-1.0, v[J + c], acc);
    } else if (i < C + J) {
#pragma unroll
      for (int j = 0; j < J; ++j) if (j == i - C) acc = __fma_rn(1.0, v[j], acc);
    } else {
#pragma unroll
      for (int j = 0; j < J; ++j) acc = __fma_rn(1.0, v[j], acc);
    }
    return acc;
  };
  auto lo_of = [&](int i) -> double { return i < C ? -INFINITY : (i < C + J ? 0.0 : 1.0); };
  auto hi_of = [&](int i) -> double {
    double v = i < C + J ? INFINITY : 1.0;
#pragma unroll
    for (int c = 0; c < C; ++c) if (c == i) v = b[c];
    return v;
  };
  // active set at z = A x (qpsolver.py:245-249)
  const double tol = fmax(1e-7, 10.0 * rp);
  unsigned act = 0, atlo = 0;
#pragma unroll
  for (int i = 0; i < MC; ++i) {
    const double zi = a_dot(i, x);
    const bool l_ = __dsub_rn(zi, lo_of(i)) <= tol, u_ = __dsub_rn(hi_of(i), zi) <= tol;
    act |= (unsigned)(l_ || u_) << i;
    atlo |= (unsigned)l_ << i;
  }
  bool accept = false;
  double xp[NV];
  if (act) {
    const double reg = 1e-8, i2 = 1.0 / (2.0 + reg);
    // ---- build R (compile-time indices keep Q in registers) and factor it
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        double v = 0.0;
        if (r < J && c < J) {
          v = r == c ? reg : 0.0;
        } else if (r < J) {  // G_l' : column c-J is constraint slot i, row r is lambda_r
          const int i = c - J;
          if (act >> i & 1u) v = i < C ? Q[i < C ? i : 0][r] : (i < C + J ? (i - C == r ? 1.0 : 0.0) : 1.0);
        } else {
          const int i = r - J;
          if (!(act >> i & 1u)) v = (c == r) ? 1.0 : 0.0;
          else if (c < J) v = i < C ? Q[i < C ? i : 0][c < J ? c : 0] : (i < C + J ? (i - C == c ? 1.0 : 0.0) : 1.0);
          else if (c == r) v = -(reg + (i < C ? i2 : 0.0));
        }
        R(r, c) = v;
      }
    unsigned char perm[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) perm[r] = (unsigned char)r;
    bool singular = false;
#pragma unroll 1
    for (int cc = 0; cc < NR; ++cc) {
      int piv = cc;
      double best = fabs(R(cc, cc));
#pragma unroll 1
      for (int r = cc + 1; r < NR; ++r) {
        const double v = fabs(R(r, cc));
        if (v > best) { best = v; piv = r; }
      }
      if (best == 0.0) { singular = true; break; }
      if (piv != cc) {
#pragma unroll 1
        for (int c = 0; c < NR; ++c) {
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
      for (int r = cc + 1; r < NR; ++r) {
        const double l = __dmul_rn(R(r, cc), rpv);
        R(r, cc) = l;
        if (l != 0.0) {
#pragma unroll 1
          for (int c = cc + 1; c < NR; ++c) R(r, c) = __fma_rn(-l, R(cc, c), R(r, c));
        }
      }
    }
    if (!singular) {
      // solve K w = r for the full unknown w = (x (NV), nu (MC slots)); r given as (rx, rn)
      auto solve = [&](const double (&rx)[NV], const double (&rn)[MC], double (&wx)[NV], double (&wn)[MC]) {
        double v[NR];  // reduced rhs in original row order: lambda rows, then constraint slots
#pragma unroll
        for (int j = 0; j < J; ++j) v[j] = rx[j];
#pragma unroll
        for (int i = 0; i < MC; ++i) {
          double t = rn[i];
          if (i < C && (act >> i & 1u)) t = __fma_rn(rx[J + i], i2, t);  // + r_delta_c / (2 + d)
          v[J + i] = (act >> i & 1u) ? t : 0.0;
        }
        auto y = [&](int r) -> double& { return Ym[r * BS]; };
#pragma unroll 1
        for (int r = 0; r < NR; ++r) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < NR; ++q) if (q == perm[r]) t = v[q];
#pragma unroll 1
          for (int c = 0; c < r; ++c) t = __fma_rn(-R(r, c), y(c), t);
          y(r) = t;
        }
#pragma unroll 1
        for (int r = NR - 1; r >= 0; --r) {
          double t = y(r);
#pragma unroll 1
          for (int c = r + 1; c < NR; ++c) t = __fma_rn(-R(r, c), y(c), t);
          y(r) = t / R(r, r);
        }
#pragma unroll
        for (int j = 0; j < J; ++j) wx[j] = y(j);
#pragma unroll
        for (int i = 0; i < MC; ++i) wn[i] = (act >> i & 1u) ? y(J + i) : 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) wx[J + c] = __dmul_rn(__dadd_rn(rx[J + c], wn[c]), i2);
      };
      // K w for the full system (rows: x then active constraint slots)
      auto kmul = [&](const double (&wx)[NV], const double (&wn)[MC], double (&ox)[NV], double (&on)[MC]) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          double acc = __dmul_rn(reg, wx[j]);
#pragma unroll
          for (int i = 0; i < MC; ++i) {
            if (!(act >> i & 1u)) continue;
            const double g = i < C ? Q[i][j] : (i < C + J ? (i - C == j ? 1.0 : 0.0) : 1.0);
            acc = __fma_rn(g, wn[i], acc);
          }
          ox[j] = acc;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) ox[J + c] = __fma_rn(2.0 + reg, wx[J + c], (act >> c & 1u) ? -wn[c] : 0.0);
#pragma unroll
        for (int i = 0; i < MC; ++i) on[i] = (act >> i & 1u) ? __fma_rn(-reg, wn[i], a_dot(i, wx)) : 0.0;
      };
      double bx[NV], bn[MC], wx[NV], wn[MC];
#pragma unroll
      for (int t = 0; t < NV; ++t) bx[t] = 0.0;  // -q = 0
#pragma unroll
      for (int i = 0; i < MC; ++i) bn[i] = (act >> i & 1u) ? ((atlo >> i & 1u) ? lo_of(i) : hi_of(i)) : 0.0;
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
      for (int t = 0; t < NV; ++t) {  // |P x + A' y|_t with y = nu on active rows
        double acc = t >= J ? __dmul_rn(2.0, wx[t]) : 0.0;
#pragma unroll
        for (int i = 0; i < MC; ++i) {
          double a;
          if (i < C) a = t < J ? Q[i][t] : (t - J == i ? -1.0 : 0.0);
          else if (i < C + J) a = (t == i - C) ? 1.0 : 0.0;
          else a = t < J ? 1.0 : 0.0;
          acc = __fma_rn(a, wn[i], acc);
        }
        rdt = fmax(rdt, fabs(acc));
      }
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
  safe_out[inst] = (uint8_t)(dl > eps_cut);
}

}  // namespace
}  // namespace bzg
