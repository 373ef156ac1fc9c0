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
