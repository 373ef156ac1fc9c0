// Obstacle cut on device: box heuristic screen over every (edge, obstacle) pair,
// batched Cut-QP (dense ADMM + active-set polish) for the indeterminate pairs,
// and CutMask aggregation (alive, first-kill provenance, counters).
//
// Replaces reference graph.py:224-265 (_heuristic_batch, box branch),
// graph.py:268-299 (_cut_qp_problem / cut_qp), graph.py:302-350 (cut_graph) and the
// dense ADMM of qpsolver.py:129-304 it calls.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#include "bzg_internal.cuh"
#include "bzg_math.cuh"
#include "k_cut_types.cuh"

namespace bzg {

namespace {


// Branch 1 of _heuristic_batch (graph.py:236-239): einsum("cm,emj->ecj"), sequential from 0.
template <int G, int M>
__device__ __forceinline__ bool any_inside_einsum(const double (&P)[M][2 * G], const ObsRec<M>& o) {
  const int R = (int)o.rows;
  bool hit = false;
#pragma unroll
  for (int j = 0; j < 2 * G; ++j) {
    bool in = true;
    for (int c = 0; c < R; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) acc = __dadd_rn(acc, __dmul_rn(o.A[c][k], P[k][j]));
      in = in && (acc <= o.b_eps[c]);
    }
    hit = hit || in;
  }
  return hit;
}

// NaN-free max / min as one DSETP and selects (fmax/fmin carry NaN handling, ~6 instructions).
// Equal to np.maximum / np.minimum / np.clip for non-NaN operands up to the sign of a zero
// result, which no later comparison or square can see.
__device__ __forceinline__ double dmax2(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin2(double a, double b) { return a < b ? a : b; }

// Exact certificate that box_code_canon returns 1 (safe), from the bounding box
// [mn, mx] of the control points.  (1) No control point is inside when, for some axis,
// every point is beyond b + eps on one side.  (2) The face the reference picks is active
// at the anchor's projection, and face +k can only be active if some point has
// P_k > hi_k - 1e-6 (|clip(v_k) - hi_k| <= 1e-7 otherwise fails; thin boxes excepted),
// likewise -k.  (3) If every possibly-active face is cleared by all points
// (fl(P_kj - b) > margin for all j  <=>  fl(min_j P_kj - b) > margin, monotone rounding),
// the clearance test passes whichever of them is chosen, so the code is 1.
//
// (4) A possibly-active face that is not cleared is harmless if it can never be chosen: when
// some face s is active for every possible anchor (all points on its outer side: mn_k >= hi_k
// puts clip(v_k) = hi_k exactly, residual 0) and cleared, and the largest separation face f
// can reach, fl(max P - b_f), is below the smallest face s can have, fl(min P - b_s), then s
// beats f at every anchor (argmax over active faces), so f is not chosen.  This certifies
// obstacles far along one axis even when the polygon straddles the plane of a face of
// another axis (large maps: a few percent of all pairs instead of most).
// The pass-1 fields of one obstacle, packed for shared memory (16 doubles at m = 2, read
// as broadcast LDS.128 by every lane).  Built on the host from the ObsRec (fill_cert):
//   be_hi = b_eps[k], nbe_lo = -b_eps[M+k]   (-P > b_eps  <=>  P < -b_eps, negation exact)
//   ahi = hi - 1e-6 (act_hi), or -inf for a thin axis (face +k then always possibly active)
//   alo = lo + 1e-6 (act_lo), or +inf for a thin axis
//   bh = b[k], bl = b[M+k], hi, lo = as_box bounds
// A non-canonical obstacle gets be_hi = +inf and nbe_lo = -inf: test (1) then never passes
// and the pair goes to pass 2 without a separate canon branch.
template <int M>
struct __align__(16) CertRec {
  double be_hi[M], nbe_lo[M], ahi[M], alo[M], bh[M], bl[M], hi[M], lo[M];
  int idx;  // obstacle index within its launch chunk (records are sorted by lo[0] per chunk)
};

template <int M>
__device__ __forceinline__ bool canon_safe_cert(const double (&mn)[M], const double (&mx)[M], const CertRec<M>& o,
                                                double margin) {
  bool noin = false, ok = true;  // (1)-(3): every possibly-active face cleared
  double L = -INFINITY;          // (4): best lower bound of the separation of a surely-active cleared face
  double ub_bad = -INFINITY;     //      largest upper bound of a possibly-active uncleared face
#pragma unroll
  for (int k = 0; k < M; ++k) {
    noin |= (mn[k] > o.be_hi[k]) | (mx[k] < o.nbe_lo[k]);
    // face +k: sep = fl(v_k - b_k) in [fl(mn_k - b_k), fl(mx_k - b_k)]
    const double lb_hi = __dsub_rn(mn[k], o.bh[k]);
    const bool pa_hi = mx[k] > o.ahi[k], clr_hi = lb_hi > margin;
    // face -k: sep = fl(-v_k - b_{M+k}) in [fl(-mx_k - b), fl(-mn_k - b)]
    const double lb_lo = __dsub_rn(-mx[k], o.bl[k]);
    const bool pa_lo = mn[k] < o.alo[k], clr_lo = lb_lo > margin;
    ok &= (!pa_hi | clr_hi) & (!pa_lo | clr_lo);
    if (clr_hi && mn[k] >= o.hi[k]) L = dmax2(L, lb_hi);
    if (clr_lo && mx[k] <= o.lo[k]) L = dmax2(L, lb_lo);
    if (pa_hi && !clr_hi) ub_bad = dmax2(ub_bad, __dsub_rn(mx[k], o.bh[k]));
    if (pa_lo && !clr_lo) ub_bad = dmax2(ub_bad, __dsub_rn(-mn[k], o.bl[k]));
  }
  // with (1): ok, or every uncleared possibly-active face loses to a surely-active cleared one
  // (no uncleared face leaves ub_bad = -inf < L only when L is finite; ok covers that case)
  return noin && (ok || ub_bad < L);
}

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
      const double t = __dadd_rn(dmax2(__dsub_rn(o.lo[k], P[k][j]), 0.0), dmax2(__dsub_rn(P[k][j], o.hi[k]), 0.0));
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
    pr[k] = dmin2(dmax2(vk, o.lo[k]), o.hi[k]);  // np.clip(v, lo, hi)
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

// Same codes for an obstacle whose rows are exactly [I; -I] (Box.to_polytope order,
// geometry.py:74-77, kept by inflate): every product with a +-1/0 coefficient is exact, so
// A.P_j reduces to +-P[k][j] and the arithmetic of box_code is reproduced bit for bit
// without the multiplications.
template <int G, int M>
__device__ __forceinline__ int box_code_canon(const double (&P)[M][2 * G], const ObsRec<M>& o, double margin) {
  constexpr int J = 2 * G;
  bool hit = false;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    bool in = true;
#pragma unroll
    for (int k = 0; k < M; ++k) in &= (P[k][j] <= o.b_eps[k]) & (-P[k][j] <= o.b_eps[M + k]);
    hit |= in;
  }
  if (hit) return 0;
  int anchor = 0;
  double best = 0.0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double d2 = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      // max(lo-P, 0) + max(P-hi, 0) == max(lo-P, P-hi, 0) exactly when lo <= hi (as_box)
      const double t = dmax2(dmax2(__dsub_rn(o.lo[k], P[k][j]), __dsub_rn(P[k][j], o.hi[k])), 0.0);
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
    pr[k] = dmin2(dmax2(vk, o.lo[k]), o.hi[k]);
  }
  int face = 0;
  double fbest = -INFINITY;
#pragma unroll
  for (int c = 0; c < 2 * M; ++c) {
    const int k = c < M ? c : c - M;
    const double sv = c < M ? v[k] : -v[k], sp = c < M ? pr[k] : -pr[k];
    const double sep = __dsub_rn(sv, o.b[c]);
    const double val = (fabs(__dsub_rn(sp, o.b[c])) <= 1e-7) ? sep : -INFINITY;
    if (c == 0 || val > fbest) { fbest = val; face = c; }
  }
  bool clear = true;
#pragma unroll
  for (int c = 0; c < 2 * M; ++c) {
    if (face == c) {
      const int k = c < M ? c : c - M;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const double hp = c < M ? P[k][j] : -P[k][j];
        clear = clear && (__dsub_rn(hp, o.b[c]) > margin);
      }
    }
  }
  return clear ? 1 : 2;
}

// One thread per edge, all obstacles of the chunk [o0, o1) in list order.
// Tracks the first heuristic kill, counts codes, and appends indeterminate pairs
// to the QP work list with warp-aggregated atomics.
// Pairs with a general (non-box) obstacle that pass branch 1 go to a second work list
// (gen_pend) for k_cut_general, so the projection QPs do not weigh on this kernel.
__device__ __forceinline__ void warp_append(bool want_me, unsigned long long item, unsigned long long* n,
                                            unsigned long long cap, unsigned long long* list) {
  const unsigned am = __activemask();
  const unsigned want = __ballot_sync(am, want_me);
  if (!want) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  const int leader = __ffs(want) - 1;
  if (lane == leader) base = atomicAdd(n, (unsigned long long)__popc(want));
  base = __shfl_sync(am, base, leader);
  if (want_me) {
    const unsigned long long slot = base + __popc(want & ((1u << lane) - 1u));
    if (slot < cap) list[slot] = item;
  }
}

constexpr int kHeurThreads = 256, kHeurWarps = kHeurThreads / 32;  // (128 x 5 blocks measured slower)

// ---- spatial pre-screen for canonical boxes (large maps): a uniform grid over the first two
// output axes holds, per cell and obstacle chunk, the mask of obstacles whose box grown by R
// meets the cell.  If an edge's control-polygon bounding box B has extent ext <= R - 0.01
// (max over axes of mx - mn), an obstacle whose grown box misses every cell B touches is more
// than R >= ext + 0.01 away from B along some axis, say below B on axis x: every point has
// P_x - hi_x > ext + 0.01, so no point is inside (1), face +x is active at every anchor and
// cleared, and every other face that could be active and is not cleared has separation at
// most ext + 1e-6 < mn_x - hi_x -- canon_safe_cert (4) holds: code 1 without evaluating it.
// Per-obstacle outcome bits of one cut (the re-cut cache, cut_graph_cached): bit e of row o
// of `kill` = (edge e, obstacle o) heuristic code 0; of `qsafe` / `qunsafe` = the pair's
// Cut-QP verdict.  kill == nullptr: not recorded.
struct CutBits {
  uint32_t* kill;
  uint32_t* qsafe;
  uint32_t* qunsafe;
  long long Wb;      // words per obstacle row: ceil(E / 32)
  long long stride;  // words from one obstacle's row to the next (Wb, or 3 Wb in a slot-major pool)
};
__device__ __forceinline__ void set_bit(uint32_t* rowbase, long long stride, int o, long long e) {
  atomicOr(rowbase + (size_t)o * stride + (e >> 5), 1u << (e & 31));
}

constexpr int kGridCells = 64;  // per axis
struct ObsGrid {
  double x0, y0, inv_cx, inv_cy, R;  // grid origin, 1 / cell size, growth radius
  unsigned long long ext_bits;       // max sampled edge extent (double bits)
  unsigned long long pop, bits;      // set mask bits / all mask bits: the grid is used when sparse
};

// Strided sample of edge control-polygon extents (at most 64 k edges), max into ext_bits.
template <int G, int M>
__global__ void k_obs_grid_extent(DParams dp, const double* __restrict__ Vx, long long E,
                                  const int* __restrict__ src, const int* __restrict__ dst, ObsGrid* __restrict__ gp,
                                  const long long* __restrict__ dE) {
  BZG_PDL_ENTRY();
  constexpr int N = G * M;
  if (dE) E = min(E, *dE);  // a captured plan's edge count (E = its capacity)
  const long long stride = E > 65536 ? E / 65536 : 1;
  const long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * stride;
  double ext = 0.0;
  if (e < E) {
    double xi[N], xj[N], P[M][2 * G];
    const long long a = src[e], b = dst[e];
#pragma unroll
    for (int k = 0; k < N; ++k) { xi[k] = Vx[a * N + k]; xj[k] = Vx[b * N + k]; }
    control_points<G, M>(xi, xj, dp.D, P);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double mn = P[k][0], mx = P[k][0];
#pragma unroll
      for (int j = 1; j < 2 * G; ++j) { mn = fmin(mn, P[k][j]); mx = fmax(mx, P[k][j]); }
      ext = fmax(ext, mx - mn);
    }
  }
  for (int d = 16; d > 0; d >>= 1) ext = fmax(ext, __shfl_down_sync(0xffffffffu, ext, d));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(&gp->ext_bits, (unsigned long long)__double_as_longlong(ext));
}

// masks[chunk][cell]: bit oi set when obstacle o0 + oi, grown by R, meets the cell.  The grid
// spans the obstacles' box bounds (lo0, lo1)-(hi0, hi1) (host) grown by R = 1.25 max sampled
// extent + 0.02 (edges above R - 0.01 test every obstacle); thread 0 publishes it in gpp.
template <int M>
__global__ void k_obs_grid_masks(const ObsRec<M>* __restrict__ obs, int n_obs, int chunk,
                                 const double* __restrict__ bnd, ObsGrid* __restrict__ gpp,
                                 unsigned long long* __restrict__ masks) {
  BZG_PDL_ENTRY();
  const double lo0 = bnd[0], lo1 = bnd[1], hi0 = bnd[2], hi1 = bnd[3];  // the obstacles' xy bounds
  const int cell = blockIdx.x * blockDim.x + threadIdx.x, ch = blockIdx.y;
  if (cell >= kGridCells * kGridCells) return;
  ObsGrid gp;
  gp.R = 1.25 * __longlong_as_double((long long)gpp->ext_bits) + 0.02;
  gp.x0 = lo0 - gp.R;
  gp.y0 = lo1 - gp.R;
  gp.inv_cx = kGridCells / fmax(hi0 - lo0 + 2 * gp.R, 1e-300);
  gp.inv_cy = kGridCells / fmax(hi1 - lo1 + 2 * gp.R, 1e-300);
  if (cell == 0 && ch == 0) {
    gpp->R = gp.R;
    gpp->x0 = gp.x0;
    gpp->y0 = gp.y0;
    gpp->inv_cx = gp.inv_cx;
    gpp->inv_cy = gp.inv_cy;
    gpp->bits = (unsigned long long)kGridCells * kGridCells * n_obs;
  }
  const int cx = cell % kGridCells, cy = cell / kGridCells;
  const double x0 = gp.x0 + cx / gp.inv_cx, x1 = gp.x0 + (cx + 1) / gp.inv_cx;
  const double y0 = gp.y0 + cy / gp.inv_cy, y1 = gp.y0 + (cy + 1) / gp.inv_cy;
  unsigned long long m = 0;
  const int o0 = ch * chunk, o1 = min(n_obs, o0 + chunk);
  for (int o = o0; o < o1; ++o) {
    const ObsRec<M>& r = obs[o];
    const bool meet = r.canon == 0.0 ||  // the argument above covers canonical boxes only
                      (r.lo[0] - gp.R <= x1 && r.hi[0] + gp.R >= x0 && r.lo[1] - gp.R <= y1 && r.hi[1] + gp.R >= y0);
    m |= (unsigned long long)meet << (o - o0);
  }
  masks[(size_t)ch * kGridCells * kGridCells + cell] = m;
  unsigned long long p = __popcll(m);
  for (int d = 16; d > 0; d >>= 1) p += __shfl_down_sync(0xffffffffu, p, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(&gpp->pop, p);
}
constexpr int kHeurRound = 8;  // pass-2 pairs per edge per round

// dynamic shared memory of k_cut_heuristic: obstacles, per-warp control points, pair lists, kills
template <int G, int M>
size_t heur_smem(int nob) {
  return (sizeof(ObsRec<M>) + sizeof(CertRec<M>) + 2 * sizeof(double)) * nob +
         (size_t)kHeurWarps * 32 * (M * 2 * G) * sizeof(double) +
         (size_t)kHeurWarps * 32 * kHeurRound * sizeof(uint16_t) + (size_t)kHeurWarps * 32 * sizeof(int);
}

template <int G, int M>
__global__ void __launch_bounds__(kHeurThreads, 3) k_cut_heuristic(DParams dp, const double* __restrict__ Vx, long long E, const int* __restrict__ src,
                                const int* __restrict__ dst, const ObsRec<M>* __restrict__ obs,
                                const CertRec<M>* __restrict__ certs, int o0, int o1, const double* __restrict__ wmaxp,
                                double margin, int* __restrict__ first_kill, unsigned long long* __restrict__ counters,
                                unsigned long long* __restrict__ n_pend, unsigned long long cap,
                                unsigned long long* __restrict__ pend, unsigned long long* __restrict__ n_gen,
                                unsigned long long gen_cap, unsigned long long* __restrict__ gen_pend,
                                const ObsGrid* __restrict__ grid, const unsigned long long* __restrict__ gmask,
                                CutBits bits, const long long* __restrict__ dE) {
  BZG_PDL_ENTRY();
  constexpr int N = G * M;
  if (dE) E = min(E, *dE);  // a captured plan's edge count (E = its capacity)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const double wmax = *wmaxp;  // the chunk's x-window width (-1: no window), from the staged obstacles
  const bool use_grid = grid != nullptr;  // the host passes the grid only when it is sparse
  const int nob = o1 - o0;
  // shared memory: [CertRec x nob][sorted lo[0] x nob][pos x nob][ObsRec x nob][per-warp pass-2 staging]
  CertRec<M>* s_cert = reinterpret_cast<CertRec<M>*>(smem_raw);
  double* s_lo = reinterpret_cast<double*>(smem_raw + sizeof(CertRec<M>) * nob);
  int* s_pos = reinterpret_cast<int*>(s_lo + nob);  // original chunk index -> sorted position
  ObsRec<M>* s_obs = reinterpret_cast<ObsRec<M>*>(smem_raw + (sizeof(CertRec<M>) + 2 * sizeof(double)) * nob);
  // with the grid, each edge touches a few obstacles: pass 2 reads their full records through
  // L1 instead of staging every record into every block's shared memory
  if (!use_grid) {
    const double* srcp = reinterpret_cast<const double*>(obs + o0);
    double* dstp = reinterpret_cast<double*>(s_obs);
    const int nd = nob * (int)(sizeof(ObsRec<M>) / sizeof(double));
    for (int t = threadIdx.x; t < nd; t += blockDim.x) dstp[t] = srcp[t];
  }
  // pass-1 records, always staged (compact): the hot loop reads them with broadcast LDS
  {
    const double* srcp = reinterpret_cast<const double*>(certs + o0);
    double* dstp = reinterpret_cast<double*>(s_cert);
    const int nd = nob * (int)(sizeof(CertRec<M>) / sizeof(double));
    for (int t = threadIdx.x; t < nd; t += blockDim.x) dstp[t] = srcp[t];
    for (int t = threadIdx.x; t < nob; t += blockDim.x) {
      s_lo[t] = certs[o0 + t].lo[0];
      s_pos[certs[o0 + t].idx] = t;
    }
  }
  __shared__ unsigned long long s_cnt[3];
  __shared__ int s_done;
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) s_done = 0;
  __syncthreads();
  unsigned c0 = 0, c1 = 0, c2 = 0;
  // persistent blocks: the records above are staged once per block, which then walks 256-edge
  // tiles (one block per tile restaged ~30 KB of records for every 256 edges)
  const long long n_tiles = (E + kHeurThreads - 1) / kHeurThreads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const long long e = tile * kHeurThreads + threadIdx.x;
    const bool valid = e < E;
    double P[M][2 * G] = {};
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
    // pass-2 staging: each lane's control points in shared memory for the lanes that take its
    // pairs.  Stored before pass 1 so P is dead during pass 1 and the bounding box (mn, mx)
    // stays in registers there (with P live the compiler rebuilt mn / mx from P for every
    // obstacle of the window: ~60 compare / select instructions per pass-1 test).
    constexpr int NP = M * 2 * G;
    unsigned char* base = smem_raw + (sizeof(ObsRec<M>) + sizeof(CertRec<M>) + 2 * sizeof(double)) * nob;
    double* s_P = reinterpret_cast<double*>(base) + (size_t)warp * 32 * NP;
    base += (size_t)kHeurWarps * 32 * NP * sizeof(double);
    uint16_t* s_it = reinterpret_cast<uint16_t*>(base) + warp * 32 * kHeurRound;
    base += (size_t)kHeurWarps * 32 * kHeurRound * sizeof(uint16_t);
    int* s_kill = reinterpret_cast<int*>(base) + warp * 32;
  #pragma unroll
    for (int k = 0; k < M; ++k)
  #pragma unroll
      for (int j = 0; j < 2 * G; ++j) s_P[lane * NP + k * 2 * G + j] = P[k][j];
    // pass 1 (coherent across the warp): certify code 1 from the control-polygon bounding box
    unsigned long long hard = 0;
    if (valid) {
      double mn[M], mx[M];
  #pragma unroll
      for (int k = 0; k < M; ++k) {
        mn[k] = P[k][0];
        mx[k] = P[k][0];
  #pragma unroll
        for (int j = 1; j < 2 * G; ++j) { mn[k] = dmin2(mn[k], P[k][j]); mx[k] = dmax2(mx[k], P[k][j]); }
      }
      const unsigned long long all = nob >= 64 ? ~0ull : ((1ull << nob) - 1ull);
      unsigned long long cand = all;
      // spatial pre-screen (ObsGrid): far obstacles are code 1; used when the grown obstacles
      // leave most cells empty (large maps; small maps skip it)
      if (M >= 2 && use_grid) {
        const ObsGrid gp = *grid;
        double ext = 0.0;
  #pragma unroll
        for (int k = 0; k < M; ++k) ext = dmax2(ext, __dsub_rn(mx[k], mn[k]));
        if (__dadd_rn(ext, 0.01) <= gp.R) {
          auto cell = [](double v, double o, double s) -> int {  // one cell of slack for rounding
            const double c = floor((v - o) * s);
            return (int)fmin(fmax(c, -1.0), (double)kGridCells);
          };
          const int cx0 = max(cell(mn[0], gp.x0, gp.inv_cx) - 1, 0), cx1 = min(cell(mx[0], gp.x0, gp.inv_cx) + 1, kGridCells - 1);
          const int cy0 = max(cell(mn[1], gp.y0, gp.inv_cy) - 1, 0), cy1 = min(cell(mx[1], gp.y0, gp.inv_cy) + 1, kGridCells - 1);
          unsigned long long m = 0;
          for (int cy = cy0; cy <= cy1; ++cy)
            for (int cx = cx0; cx <= cx1; ++cx) m |= gmask[cy * kGridCells + cx];
          cand &= m;
        }
      }
      if (cand == all) {
        // x-window over the lo[0]-sorted records: a canonical box farther than T = ext + 0.02
        // from the bounding box along x is certified code 1 by the ObsGrid argument above
        // (separation > ext + 0.01 along one axis; the 0.01 slack absorbs the rounding of T and
        // of the window bounds).  Boxes with lo_x > mx_x + T lie right of it, boxes with
        // lo_x < mn_x - T - wmax have hi_x <= lo_x + wmax < mn_x - T and lie left of it.
        int i0 = 0, i1 = nob;
        // y-band: inside the x-window, a box farther than T along y is certified the same way
        double yl = -INFINITY, yh = INFINITY;
        if (wmax >= 0.0) {
          double ext = 0.0;
  #pragma unroll
          for (int k = 0; k < M; ++k) ext = dmax2(ext, __dsub_rn(mx[k], mn[k]));
          const double T = ext + 0.02, wl = mn[0] - T - wmax, wh = mx[0] + T;
          if (M >= 2) {
            yl = mn[M >= 2 ? 1 : 0] - T;  // hi_y < yl: below the band
            yh = mx[M >= 2 ? 1 : 0] + T;  // lo_y > yh: above it
          }
          int lo = 0, hi = nob;  // first sorted lo >= wl
          while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_lo[mid] < wl) lo = mid + 1; else hi = mid; }
          i0 = lo;
          hi = nob;  // first sorted lo > wh
          while (lo < hi) { const int mid = (lo + hi) >> 1; if (s_lo[mid] <= wh) lo = mid + 1; else hi = mid; }
          i1 = lo;
          c1 += nob - (i1 - i0);
        }
        for (int i = i0; i < i1; ++i) {
          const CertRec<M>& o = s_cert[i];
          if ((M >= 2 && (o.hi[M >= 2 ? 1 : 0] < yl || o.lo[M >= 2 ? 1 : 0] > yh)) ||
              canon_safe_cert<M>(mn, mx, o, margin))
            ++c1;
          else
            hard |= 1ull << o.idx;
        }
      } else {
        c1 += __popcll(all & ~cand);
        for (unsigned long long rest = cand; rest; rest &= rest - 1ull) {
          const int oi = __ffsll((long long)rest) - 1;
          if (canon_safe_cert<M>(mn, mx, s_cert[s_pos[oi]], margin)) ++c1;
          else hard |= 1ull << oi;
        }
      }
    }
    // pass 2 (warp-cooperative): the uncertified (edge, obstacle) pairs of the warp's 32 edges
    // are dealt out to all 32 lanes, a round of at most kHeurRound pairs per edge at a time, so
    // lanes whose edge has few hard obstacles do not idle while others work through theirs.
    // Each lane's control points are staged in shared memory for the lanes that take its pairs.
    s_kill[lane] = kill;
    const long long e0 = e - lane;
    __syncwarp();
    while (__any_sync(0xffffffffu, hard != 0)) {
      const int cnt = min(__popcll(hard), kHeurRound);
      int off = cnt;  // inclusive warp scan of cnt
  #pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += t;
      }
      const int total = __shfl_sync(0xffffffffu, off, 31);
      off -= cnt;
      if (lane == 0) atomicAdd(counters + 8, (unsigned long long)total);
      for (int q = 0; q < cnt; ++q) {
        const int oi = __ffsll((long long)hard) - 1;
        hard &= hard - 1;
        s_it[off + q] = (uint16_t)((lane << 8) | oi);
      }
      __syncwarp();
      for (int b0 = 0; b0 < total; b0 += 32) {
        int code = -1;
        unsigned long long item = 0;
        if (b0 + lane < total) {
          const int it = s_it[b0 + lane], owner = it >> 8, oi = it & 255;
          double Pq[M][2 * G];
  #pragma unroll
          for (int k = 0; k < M; ++k)
  #pragma unroll
            for (int j = 0; j < 2 * G; ++j) Pq[k][j] = s_P[owner * NP + k * 2 * G + j];
          auto eval = [&](const ObsRec<M>& o) -> int {
            if (o.is_box == 0.0)  // 3: decided by k_cut_general (all of it when the rows exceed the record)
              return (o.rows <= (double)kObsRows && any_inside_einsum<G, M>(Pq, o)) ? 0 : 3;
            return o.canon != 0.0 ? box_code_canon<G, M>(Pq, o, margin) : box_code<G, M>(Pq, o, margin);
          };
          // two call sites so each reads its records with the address space known (LDS / LDG)
          code = use_grid ? eval(obs[o0 + oi]) : eval(s_obs[oi]);
          c0 += code == 0;
          c1 += code == 1;
          c2 += code == 2;
          if (code == 0) {
            atomicMin(s_kill + owner, o0 + oi);
            if (bits.kill) set_bit(bits.kill, bits.stride, o0 + oi, e0 + owner);
          }
          item = ((unsigned long long)(e0 + owner) << 20) | (unsigned long long)(o0 + oi);
        }
        warp_append(code == 2, item, n_pend, cap, pend);
        warp_append(code == 3, item, n_gen, gen_cap, gen_pend);
      }
      __syncwarp();
    }
    if (valid) first_kill[e] = s_kill[lane];
    __syncwarp();  // the warp's staging slices are rewritten by the next tile
  }
  // counters without a block barrier (warps finish pass 2 at different times): warp sums into
  // shared memory, and the block's last warp to finish adds them to the global counters
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    c0 += __shfl_down_sync(0xffffffffu, c0, d);
    c1 += __shfl_down_sync(0xffffffffu, c1, d);
    c2 += __shfl_down_sync(0xffffffffu, c2, d);
  }
  if (lane == 0) {
    atomicAdd(s_cnt + 0, (unsigned long long)c0);
    atomicAdd(s_cnt + 1, (unsigned long long)c1);
    atomicAdd(s_cnt + 2, (unsigned long long)c2);
    __threadfence_block();
    if (atomicAdd(&s_done, 1) == kHeurWarps - 1) {
      __threadfence_block();
      atomicAdd(counters + 0, atomicAdd(s_cnt + 0, 0ull));
      atomicAdd(counters + 1, atomicAdd(s_cnt + 1, 0ull));
      atomicAdd(counters + 2, atomicAdd(s_cnt + 2, 0ull));
    }
  }
}

}  // namespace
}  // namespace bzg

#include "k_general.cuh"

namespace bzg {
namespace {

constexpr double kEpsGeo = 1e-9;  // geometry.EPS_GEO (geometry.py:14), closest_point's default eps

// cut_heuristic past branch 1 (graph.py:242-247 -> 202-221) for the general-obstacle pairs,
// one thread per pair.  Same bookkeeping as k_cut_heuristic: first kill by atomicMin, codes
// counted, indeterminate pairs appended to the QP work list.  counters[7] flags an
// obstacle whose projection QP certified it empty (the reference raises ValueError).
template <int G, int M, int RC>
__global__ void k_cut_general(DParams dp, const double* __restrict__ Vx, const int* __restrict__ src,
                              const int* __restrict__ dst, const ObsRec<M, RC>* __restrict__ obs,
                              const unsigned long long* __restrict__ gen, long long n_cap,
                              const unsigned long long* __restrict__ d_n, double margin,
                              int* __restrict__ first_kill, unsigned long long* __restrict__ counters,
                              unsigned long long* __restrict__ n_pend, unsigned long long cap,
                              unsigned long long* __restrict__ pend, int8_t* __restrict__ code_out, CutBits bits) {
  BZG_PDL_ENTRY();
  constexpr int N = G * M;
  // n = min(*d_n, n_cap): the pair count of the screen, known on the device only
  const long long n = d_n ? ((long long)*d_n < n_cap ? (long long)*d_n : n_cap) : n_cap;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n; t0 += stride) {  // warp-uniform
    const long long t = t0 + threadIdx.x;
    int code = -2;
    unsigned long long item = 0;
    if (t < n) {
      item = gen[t];
      const long long e = (long long)(item >> 20);
      const int oi = (int)(item & 0xFFFFF);
      double xi[N], xj[N], P[M][2 * G];
      const long long a = src[e], c = dst[e];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        xi[k] = Vx[a * N + k];
        xj[k] = Vx[c * N + k];
      }
      control_points<G, M>(xi, xj, dp.D, P);
      code = general_code<G, M, RC>(P, obs[oi], margin, kEpsGeo);
      if (code == 0) {
        atomicMin(first_kill + e, oi);
        if (bits.kill) set_bit(bits.kill, bits.stride, oi, e);
      }
      if (code >= 0) atomicAdd(counters + code, 1ull);
      if (code == -1) atomicOr(counters + 7, 1ull);
      if (code_out) code_out[t] = (int8_t)code;
    }
    warp_append(code == 2, item, n_pend, cap, pend);
  }
}

// ------------------------------------------------------------------ aggregation
__global__ void k_qp_verdicts(const unsigned long long* __restrict__ pend, long long n_cap,
                              const unsigned long long* __restrict__ d_n, const uint8_t* __restrict__ safe,
                              int* __restrict__ qp_kill, uint8_t* __restrict__ qp_saved,
                              unsigned long long* __restrict__ counters, CutBits bits) {
  BZG_PDL_ENTRY();
  const long long n = (long long)*d_n < n_cap ? (long long)*d_n : n_cap;
  unsigned long long s = 0, u = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const unsigned long long pk = pend[t];
    const long long e = (long long)(pk >> 20);
    const int o = (int)(pk & 0xFFFFF);
    if (safe[t]) {
      qp_saved[e] = 1;
      ++s;
      if (bits.kill) set_bit(bits.qsafe, bits.stride, o, e);
    } else {
      atomicMin(qp_kill + e, o);
      ++u;
      if (bits.kill) set_bit(bits.qunsafe, bits.stride, o, e);
    }
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long ts = BR(tmp).Sum(s);
  __syncthreads();
  unsigned long long tu = BR(tmp).Sum(u);
  if (threadIdx.x == 0) {
    if (ts) atomicAdd(counters + 3, ts);
    if (tu) atomicAdd(counters + 4, tu);
  }
}

// alive / provenance from the first killing obstacle (graph.py:316-340)
__global__ void k_mask_finalize(long long E, int n_obs, const int* __restrict__ first_kill,
                                const int* __restrict__ qp_kill, const uint8_t* __restrict__ qp_saved,
                                uint8_t* __restrict__ alive, uint8_t* __restrict__ prov) {
  BZG_PDL_ENTRY();
  // four edges per thread: 16-byte loads of both kill arrays, 4-byte flag loads and stores
  const long long e0 = 4 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  if (e0 >= E) return;
  auto one = [&](int kh, int kq, uint8_t saved, uint8_t& a, uint8_t& p) {
    const bool dead = kh < n_obs || kq < n_obs;
    a = dead ? 0 : 1;
    if (dead) p = kh < kq ? BZG_HEURISTIC_UNSAFE : BZG_QP_UNSAFE;
    else p = saved ? BZG_QP_SAFE : BZG_HEURISTIC_SAFE;
  };
  if (e0 + 4 <= E) {
    const int4 kh = *reinterpret_cast<const int4*>(first_kill + e0);
    const int4 kq = *reinterpret_cast<const int4*>(qp_kill + e0);
    const uint32_t sv = *reinterpret_cast<const uint32_t*>(qp_saved + e0);
    uint8_t a[4], p[4];
    one(kh.x, kq.x, (uint8_t)(sv & 0xFF), a[0], p[0]);
    one(kh.y, kq.y, (uint8_t)((sv >> 8) & 0xFF), a[1], p[1]);
    one(kh.z, kq.z, (uint8_t)((sv >> 16) & 0xFF), a[2], p[2]);
    one(kh.w, kq.w, (uint8_t)(sv >> 24), a[3], p[3]);
    *reinterpret_cast<uint32_t*>(alive + e0) = a[0] | (a[1] << 8) | (a[2] << 16) | ((uint32_t)a[3] << 24);
    *reinterpret_cast<uint32_t*>(prov + e0) = p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24);
  } else {
    for (long long e = e0; e < E; ++e) one(first_kill[e], qp_kill[e], qp_saved[e], alive[e], prov[e]);
  }
}

__global__ void k_unpack_pend(const unsigned long long* __restrict__ pend, long long n, long long* __restrict__ e,
                              int* __restrict__ o) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  e[t] = (long long)(pend[t] >> 20);
  o[t] = (int)(pend[t] & 0xFFFFF);
}

__global__ void k_fill_int(int* p, long long n, int v) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < n) p[t] = v;
}

// The cut's per-edge state in one pass: kill = qkill = v (no obstacle yet), saved = 0; four
// edges per thread (16-byte stores to both int arrays, one 4-byte store of flags).
__global__ void k_cut_init(int* __restrict__ kill, int* __restrict__ qkill, uint8_t* __restrict__ saved, long long n,
                           int v) {
  BZG_PDL_ENTRY();
  const long long e = 4 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  if (e + 4 <= n) {
    const int4 q = make_int4(v, v, v, v);
    *reinterpret_cast<int4*>(kill + e) = q;
    *reinterpret_cast<int4*>(qkill + e) = q;
    *reinterpret_cast<uint32_t*>(saved + e) = 0u;
  } else {
    for (long long k = e; k < n; ++k) {
      kill[k] = v;
      qkill[k] = v;
      saved[k] = 0;
    }
  }
}

// ||delta|| above which the ADMM verdict is final (see k_qp_select); BZG_POLISH_SCREEN=0
// polishes every SOLVED instance exactly like the reference.
double polish_screen() {
  const char* s = std::getenv("BZG_POLISH_SCREEN");
  return s ? std::atof(s) : 1e-2;
}


template <typename F>
void dispatch_cut(int G, int M, F&& f) {
#define BZG_GM(g, m) \
  if (G == g && M == m) { f(std::integral_constant<int, g>{}, std::integral_constant<int, m>{}); return; }
  BZG_GM(1, 1) BZG_GM(1, 2) BZG_GM(1, 3) BZG_GM(2, 1) BZG_GM(2, 2) BZG_GM(2, 3)
  BZG_GM(3, 1) BZG_GM(3, 2) BZG_GM(3, 3) BZG_GM(4, 1) BZG_GM(4, 2) BZG_GM(4, 3)
#undef BZG_GM
  throw Error(BZG_EUNSUPPORTED, "device cut supports gamma in 1..4 and m in 1..3");
}

// Device records of the obstacle list; rows normalised by the caller (geometry.py:135-137).
// RC = row capacity of the record (an obstacle with more rows keeps only `rows`, see ObsRec).
template <int M, int RC = kObsRows>
std::vector<ObsRec<M, RC>> fill_obs(int n_obs, const int32_t* row_off, const double* A, const double* b,
                                    const uint8_t* is_box, const double* box_lo, const double* box_hi, double eps_geo) {
  std::vector<ObsRec<M, RC>> h(std::max(n_obs, 1));
  for (int o = 0; o < n_obs; ++o) {
    ObsRec<M, RC>& r = h[o];
    const int rows = row_off[o + 1] - row_off[o];
    r.rows = rows;
    r.is_box = is_box[o] ? 1.0 : 0.0;
    const int kept = rows <= RC ? rows : 0;  // an over-capacity obstacle: rows only
    for (int q = 0; q < RC; ++q) {
      const int row = row_off[o] + q;
      double s = 0.0;
      for (int k = 0; k < M; ++k) {
        r.A[q][k] = q < kept ? A[(size_t)row * M + k] : 0.0;
        const double sq = r.A[q][k] * r.A[q][k];
        s = k == 0 ? sq : s + sq;  // np.linalg.norm(axis=1): left fold of the squares
      }
      r.norm2[q] = q < kept ? std::sqrt(s) : 1.0;
      r.b[q] = q < kept ? b[row] : 1e300;
      r.b_eps[q] = q < kept ? b[row] + eps_geo : 1e300;  // O.b + eps_geo (graph.py:234)
    }
    for (int k = 0; k < M; ++k) {
      r.lo[k] = box_lo[(size_t)o * M + k];
      r.hi[k] = box_hi[(size_t)o * M + k];
    }
    bool canon = is_box[o] != 0;
    for (int q = 0; q < 2 * M && q < RC; ++q)
      for (int k = 0; k < M; ++k) canon = canon && r.A[q][k] == (k == (q % M) ? (q < M ? 1.0 : -1.0) : 0.0);
    r.canon = canon ? 1.0 : 0.0;
    for (int k = 0; k < M; ++k) {
      r.act_hi[k] = r.hi[k] - 1e-6;
      r.act_lo[k] = r.lo[k] + 1e-6;
      r.thin[k] = (r.hi[k] - r.lo[k] > 1e-6) ? 0.0 : 1.0;
    }
  }
  return h;
}

// Pass-1 records, sorted by lo[0] within each launch chunk, and per chunk the widest box
// along axis 0 (the x-window of k_cut_heuristic), or -1 when the chunk has a non-canonical
// obstacle (every such pair must reach pass 2, so no obstacle may be skipped).
template <int M>
std::vector<CertRec<M>> fill_cert(const std::vector<ObsRec<M>>& h, int n_obs, int chunk, std::vector<double>& wmax) {
  std::vector<CertRec<M>> out(h.size());
  std::vector<CertRec<M>> flat(h.size());
  for (size_t o = 0; o < h.size(); ++o) {
    const ObsRec<M>& r = h[o];
    CertRec<M>& q = flat[o];
    const bool canon = r.canon != 0.0;
    for (int k = 0; k < M; ++k) {
      q.be_hi[k] = canon ? r.b_eps[k] : INFINITY;
      q.nbe_lo[k] = canon ? -r.b_eps[M + k] : -INFINITY;
      q.ahi[k] = r.thin[k] != 0.0 ? -INFINITY : r.act_hi[k];
      q.alo[k] = r.thin[k] != 0.0 ? INFINITY : r.act_lo[k];
      q.bh[k] = r.b[k];
      q.bl[k] = r.b[M + k];
      q.hi[k] = r.hi[k];
      q.lo[k] = r.lo[k];
    }
  }
  wmax.clear();
  for (int o0 = 0; o0 < std::max(n_obs, 1); o0 += chunk) {
    const int o1 = std::min(std::max(n_obs, 1), o0 + chunk);
    std::vector<int> ord(o1 - o0);
    for (int i = 0; i < o1 - o0; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return flat[o0 + a].lo[0] < flat[o0 + b].lo[0]; });
    double w = 0.0;
    bool all_canon = n_obs > 0;
    for (int i = 0; i < o1 - o0; ++i) {
      out[o0 + i] = flat[o0 + ord[i]];
      out[o0 + i].idx = ord[i];
      if (o0 + ord[i] < n_obs) {
        all_canon = all_canon && h[o0 + ord[i]].canon != 0.0;
        w = std::max(w, flat[o0 + ord[i]].hi[0] - flat[o0 + ord[i]].lo[0]);
      }
    }
    wmax.push_back(all_canon && std::isfinite(w) ? w : -1.0);
  }
  return out;
}

// Validates the obstacle list; returns the padded row count of a Cut-QP launch
// (2m when every obstacle fits, else kObsRows, else kObsRowsBig).
int check_obstacles(int n_obs, const int32_t* row_off, const uint8_t* is_box, int m) {
  int max_rows = 2 * m;
  for (int o = 0; o < n_obs; ++o) {
    const int rows = row_off[o + 1] - row_off[o];
    BZG_REQUIRE(rows >= 1 && rows <= kObsRowsBig, BZG_EUNSUPPORTED,
                "obstacle " + std::to_string(o) + " has " + std::to_string(rows) + " rows; the device cut takes 1.." +
                    std::to_string(kObsRowsBig));
    BZG_REQUIRE(!is_box[o] || rows == 2 * m, BZG_EINVAL, "box obstacle must have 2m rows");
    max_rows = std::max(max_rows, rows);
  }
  return max_rows <= 2 * m ? 2 * m : (max_rows <= kObsRows ? kObsRows : kObsRowsBig);
}

template <int M, typename F>
void dispatch_rows(int qp_rows, F&& f) {
  if (qp_rows <= 2 * M) f(std::integral_constant<int, 2 * M>{});
  else if (qp_rows <= kObsRows) {
    if constexpr (2 * M < kObsRows) f(std::integral_constant<int, kObsRows>{});
  } else {
    f(std::integral_constant<int, kObsRowsBig>{});
  }
}

}  // namespace

namespace {

// ---- a cut in three steps: host preparation (cut_prepare: obstacle records, pass-1
// certificates, per-chunk x-windows and the xy bounds, staged in ONE blob uploaded with one
// copy), the launches (cut_enqueue: no host round trip, every buffer from c->ws or the mask,
// so a replanner can capture it), and the host finish after the stream synchronised.
struct CutPrep {
  std::vector<unsigned char> blob;
  int n_obs = 0, qp_rows = 0, chunk = 1, n_chunks = 1;
  bool big = false, canon_all = true, any_general = false, grid_cand = false;
  double blo[2] = {INFINITY, INFINITY}, bhi[2] = {-INFINITY, -INFINITY};
  size_t off_rec = 0, off_wmax = 0, off_bnd = 0, off_big = 0;
  // everything a captured launch sequence depends on besides the blob's contents
  bool same_shape(const CutPrep& o) const {
    return blob.size() == o.blob.size() && n_obs == o.n_obs && qp_rows == o.qp_rows && chunk == o.chunk &&
           n_chunks == o.n_chunks && big == o.big && canon_all == o.canon_all && any_general == o.any_general &&
           grid_cand == o.grid_cand;
  }
};

inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

template <int Mc>
void cut_prepare_t(const Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
                   const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
                   int qp_rows, CutPrep& p) {
  using Rec = ObsRec<Mc>;
  const std::vector<Rec> h = fill_obs<Mc>(n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg->eps_geo);
  // obstacles per launch: fits shared memory and the 64-bit per-edge "hard" mask
  p.chunk = std::min(64, std::max(1, (int)(96 * 1024 / sizeof(Rec))));
  std::vector<double> wmax;
  const std::vector<CertRec<Mc>> hc = fill_cert<Mc>(h, n_obs, p.chunk, wmax);
  if (std::getenv("BZG_NO_OBS_WINDOW"))  // read per call (tests toggle it): test every obstacle
    for (double& w : wmax) w = -1.0;
  p.n_obs = n_obs;
  p.qp_rows = qp_rows;
  p.n_chunks = (int)wmax.size();
  p.big = qp_rows > kObsRows;
  p.canon_all = true;
  p.any_general = false;
  for (int o = 0; o < n_obs; ++o) {
    p.canon_all = p.canon_all && h[o].canon != 0.0;
    p.any_general = p.any_general || h[o].is_box == 0.0;
    for (int k = 0; k < 2 && k < Mc; ++k) {
      p.blo[k] = std::min(p.blo[k], h[o].lo[k]);
      p.bhi[k] = std::max(p.bhi[k], h[o].hi[k]);
    }
  }
  p.grid_cand = Mc >= 2 && n_obs >= 8 && g->E > 0 && std::getenv("BZG_NO_OBS_GRID") == nullptr;  // per call
  // [CertRec x n][ObsRec x n][wmax x chunks][xy bounds][ObsRec<M, kObsRowsBig> x n when big]
  const size_t cert_bytes = sizeof(CertRec<Mc>) * hc.size();  // CertRec is 16-byte aligned and sized
  p.off_rec = align16(cert_bytes);
  p.off_wmax = align16(p.off_rec + sizeof(Rec) * h.size());
  p.off_bnd = align16(p.off_wmax + sizeof(double) * wmax.size());
  p.off_big = align16(p.off_bnd + 4 * sizeof(double));
  std::vector<ObsRec<Mc, kObsRowsBig>> hbig;
  if (p.big) hbig = fill_obs<Mc, kObsRowsBig>(n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg->eps_geo);
  p.blob.assign(p.off_big + sizeof(ObsRec<Mc, kObsRowsBig>) * hbig.size(), 0);
  std::memcpy(p.blob.data(), hc.data(), cert_bytes);
  std::memcpy(p.blob.data() + p.off_rec, h.data(), sizeof(Rec) * h.size());
  std::memcpy(p.blob.data() + p.off_wmax, wmax.data(), sizeof(double) * wmax.size());
  const double bnd[4] = {p.blo[0], Mc >= 2 ? p.blo[1] : 0.0, p.bhi[0], Mc >= 2 ? p.bhi[1] : 0.0};
  std::memcpy(p.blob.data() + p.off_bnd, bnd, sizeof(bnd));
  if (p.big) std::memcpy(p.blob.data() + p.off_big, hbig.data(), sizeof(ObsRec<Mc, kObsRowsBig>) * hbig.size());
}

// Work-list capacities and the obstacle-grid mode of one cut_enqueue: grid 0 = no grid,
// 1 = build it (k_obs_grid_extent / k_obs_grid_masks) and use it, 2 = use the one built
// earlier on this stream.
struct CutCaps {
  unsigned long long cap = 0, gen_cap = 1;
  long long qcap = 0;
  int grid = 0;
};

template <int Gc, int Mc>
void grid_build(Ctx* c, Graph* g, const CutPrep& p, const unsigned char* d_blob) {
  const long long E = g->E;
  DParams dp{};
  for (size_t k = 0; k < g->D.size(); ++k) dp.D[k] = g->D[k];
  DevBuf &d_grid = c->ws[WS_OBSGRIDHDR], &d_gmask = c->ws[WS_OBSGRID];
  d_grid.alloc(sizeof(ObsGrid), c->stream);
  BZG_CHECK_CUDA(cudaMemsetAsync(d_grid.ptr, 0, sizeof(ObsGrid), c->stream));
  d_gmask.alloc((size_t)p.n_chunks * kGridCells * kGridCells * sizeof(unsigned long long), c->stream);
  launch(c, "k_obs_grid_extent", k_obs_grid_extent<Gc, Mc>, dim3(div_up(std::min(E, 65536ll), 256)), dim3(256), 0, dp,
         g->vertices.as<double>(), E, g->src.as<int>(), g->dst.as<int>(), d_grid.as<ObsGrid>(), (const long long*)g->dE);
  launch(c, "k_obs_grid_masks", k_obs_grid_masks<Mc>, dim3(kGridCells * kGridCells / 256, (unsigned)p.n_chunks),
         dim3(256), 0, reinterpret_cast<const ObsRec<Mc>*>(d_blob + p.off_rec), p.n_obs, p.chunk,
         reinterpret_cast<const double*>(d_blob + p.off_bnd), d_grid.as<ObsGrid>(),
         d_gmask.as<unsigned long long>());
}

// The cut's launches: reset, (grid), screen per obstacle chunk, general pairs, Cut-QP stage,
// verdicts, mask, and the counters' read-back into h_cnt (8 words: codes 0/1/2, QP safe /
// unsafe, QP work-list length, general-list length, empty-polytope flag).  Also resets the
// mask's cached search keys (its alive set changes).  No host synchronisation.
template <int Gc, int Mc>
void cut_enqueue(Ctx* c, Graph* g, const CutPrep& p, const unsigned char* d_blob, const bzg_cut_config* cfg, Mask* mk,
                 CutBits cbits, const CutCaps& cc, unsigned long long* h_cnt) {
  const long long E = g->E;
  const int n_obs = p.n_obs;
  DParams dp{};
  for (size_t k = 0; k < g->D.size(); ++k) dp.D[k] = g->D[k];
  const CertRec<Mc>* d_cert = reinterpret_cast<const CertRec<Mc>*>(d_blob);
  const ObsRec<Mc>* d_recs = reinterpret_cast<const ObsRec<Mc>*>(d_blob + p.off_rec);
  const double* d_wmax = reinterpret_cast<const double*>(d_blob + p.off_wmax);
  const void* d_qp_obs = p.big ? (const void*)(d_blob + p.off_big) : (const void*)d_recs;
  DevBuf &d_kill = c->ws[WS_KILL], &d_qkill = c->ws[WS_QKILL], &d_saved = c->ws[WS_SAVED], &d_cnt = c->ws[WS_CUTCNT];
  DevBuf &d_pend = c->ws[WS_PEND], &d_gen = c->ws[WS_GEN];
  d_kill.alloc(std::max(E, 1ll) * sizeof(int), c->stream);
  d_qkill.alloc(std::max(E, 1ll) * sizeof(int), c->stream);
  d_saved.alloc(std::max(E, 1ll), c->stream);
  d_cnt.alloc(16 * sizeof(unsigned long long), c->stream);  // [8]: pass-2 pairs (diagnostic)
  d_pend.alloc(cc.cap * sizeof(unsigned long long), c->stream);
  d_gen.alloc(cc.gen_cap * sizeof(unsigned long long), c->stream);
  unsigned long long* dcnt = d_cnt.as<unsigned long long>();
  BZG_CHECK_CUDA(cudaMemsetAsync(d_cnt.ptr, 0, 16 * sizeof(unsigned long long), c->stream));
  launch(c, "k_cut_init", k_cut_init, dim3(div_up(div_up(E, 4), 256)), dim3(256), 0, d_kill.as<int>(),
         d_qkill.as<int>(), d_saved.as<uint8_t>(), E, n_obs);
  if (cbits.kill && n_obs > 0)  // the recorded outcome rows (n_obs rows of Wb words, stride apart)
    for (uint32_t* rows : {cbits.kill, cbits.qsafe, cbits.qunsafe})
      BZG_CHECK_CUDA(cudaMemset2DAsync(rows, cbits.stride * sizeof(uint32_t), 0, cbits.Wb * sizeof(uint32_t), n_obs,
                                       c->stream));
  for (DevBuf* key : {&mk->tree_key, &mk->reach_key})  // the mask's alive set changes: no cached tree
    if (key->ptr) BZG_CHECK_CUDA(cudaMemsetAsync(key->ptr, 0xFF, sizeof(long long), c->stream));
  if (cc.grid == 1) grid_build<Gc, Mc>(c, g, p, d_blob);
  const bool use_grid = cc.grid != 0;
  DevBuf &d_grid = c->ws[WS_OBSGRIDHDR], &d_gmask = c->ws[WS_OBSGRID];

  // ---- heuristic screen (obstacle chunks sized to shared memory)
  for (int o0 = 0; o0 < n_obs; o0 += p.chunk) {
    const int o1 = std::min(n_obs, o0 + p.chunk);
    const size_t smem = heur_smem<Gc, Mc>(o1 - o0);
    auto kern = k_cut_heuristic<Gc, Mc>;
    ensure_dyn_smem((const void*)kern, smem);
    const unsigned long long* gm =
        use_grid ? d_gmask.as<unsigned long long>() + (size_t)(o0 / p.chunk) * kGridCells * kGridCells : nullptr;
    const long long hblocks = std::min<long long>(div_up(E, kHeurThreads), (long long)c->num_sms * 3);
    launch(c, "k_cut_heuristic", kern, dim3((unsigned)hblocks), dim3(kHeurThreads), smem, dp, g->vertices.as<double>(),
           E, g->src.as<int>(), g->dst.as<int>(), d_recs, d_cert, o0, o1, d_wmax + o0 / p.chunk, cfg->heur_margin,
           d_kill.as<int>(), dcnt, dcnt + 5, cc.cap, d_pend.as<unsigned long long>(), dcnt + 6, cc.gen_cap,
           d_gen.as<unsigned long long>(), use_grid ? d_grid.as<ObsGrid>() : (const ObsGrid*)nullptr, gm, cbits,
           (const long long*)g->dE);
  }
  if (p.any_general) {
    // general obstacles: cut_heuristic past branch 1 over the device-side list, appending
    // to the same QP work list
    const long long gblocks = std::min<long long>(div_up((long long)cc.gen_cap, 64), c->num_sms * 16ll);
    if (p.big)
      launch(c, "k_cut_general", k_cut_general<Gc, Mc, kObsRowsBig>, dim3((unsigned)gblocks), dim3(64), 0, dp,
             g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(),
             reinterpret_cast<const ObsRec<Mc, kObsRowsBig>*>(d_blob + p.off_big), d_gen.as<unsigned long long>(),
             (long long)cc.gen_cap, (const unsigned long long*)(dcnt + 6), cfg->heur_margin, d_kill.as<int>(), dcnt,
             dcnt + 5, cc.cap, d_pend.as<unsigned long long>(), (int8_t*)nullptr, cbits);
    else
      launch(c, "k_cut_general", k_cut_general<Gc, Mc, kObsRows>, dim3((unsigned)gblocks), dim3(64), 0, dp,
             g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(), d_recs, d_gen.as<unsigned long long>(),
             (long long)cc.gen_cap, (const unsigned long long*)(dcnt + 6), cfg->heur_margin, d_kill.as<int>(), dcnt,
             dcnt + 5, cc.cap, d_pend.as<unsigned long long>(), (int8_t*)nullptr, cbits);
  }
  c->trace("cut: heuristic");

  // ---- Cut-QP over the device-side work list (its length stays on the device, dcnt[5]); the
  // per-instance buffers have capacity qcap, checked after the read-back
  DevBuf &d_safe = c->ws[WS_QSAFE], &d_qst = c->ws[WS_QSTATUS], &d_qit = c->ws[WS_QITERS], &d_qdl = c->ws[WS_QDELTA];
  if (E > 0 && n_obs > 0) {
    const long long qcap = cc.qcap;
    d_safe.alloc(qcap, c->stream);
    d_qst.alloc(qcap, c->stream);
    d_qit.alloc(qcap * sizeof(int), c->stream);
    d_qdl.alloc(qcap * sizeof(double), c->stream);
    dispatch_rows<Mc>(p.qp_rows, [&](auto C_) {
      constexpr int Cc = decltype(C_)::value;
      QpJob job{g, {}, d_qp_obs, p.canon_all, d_pend.as<unsigned long long>(), qcap, dcnt + 5, cfg,
                cfg->qp_polish ? 1 : 0, polish_screen(), mk, &d_safe, d_qst.as<int8_t>(), d_qit.as<int>(),
                d_qdl.as<double>()};
      for (int k = 0; k < 64; ++k) job.D[k] = dp.D[k];
      qp_solve(c, Gc, Mc, Cc, job);
    });
    c->trace("cut: qp");
    launch(c, "k_qp_verdicts", k_qp_verdicts, dim3((unsigned)std::min<long long>(div_up(qcap, 256), c->num_sms * 8ll)),
           dim3(256), 0, d_pend.as<unsigned long long>(), qcap, (const unsigned long long*)(dcnt + 5),
           d_safe.as<uint8_t>(), d_qkill.as<int>(), d_saved.as<uint8_t>(), dcnt, cbits);
  }
  launch(c, "k_mask_finalize", k_mask_finalize, dim3(div_up(div_up(E, 4), 256)), dim3(256), 0, E, n_obs,
         d_kill.as<int>(), d_qkill.as<int>(), d_saved.as<uint8_t>(), mk->alive.as<uint8_t>(), mk->prov.as<uint8_t>());
  BZG_CHECK_CUDA(cudaMemcpyAsync(h_cnt, d_cnt.ptr, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
}

// the mask fields a cut sets on the host before its launches
void mask_begin(Ctx* c, Graph* g, Mask* mk, int n_obs) {
  const long long E = g->E;
  mk->g = g;
  mk->ctx = c;
  mk->E = E;
  mk->n_obs = n_obs;
  mk->alive.alloc(std::max(E, 1ll), c->stream);
  mk->prov.alloc(std::max(E, 1ll), c->stream);
  for (int i = 0; i < 6; ++i) mk->counters[i] = 0;
  mk->counters[0] = E * (long long)n_obs;
  mk->reach_vg = -1;
  mk->n_qp = 0;
}

// counters of a finished cut from its read-back
void mask_counters(Mask* mk, const unsigned long long* hcnt) {
  for (int i = 0; i < 5; ++i) mk->counters[1 + i] = (long long)hcnt[i];
}

// first cut on this context: half the screen's list capacity; afterwards the last count + 25%
CutCaps default_caps(Ctx* c, const Graph* g, const CutPrep& p) {
  CutCaps cc;
  cc.cap = (unsigned long long)std::max<long long>(1 << 20, g->E * (long long)p.n_obs / 32);
  cc.gen_cap = p.any_general ? cc.cap : 1;
  cc.qcap = c->qp_hint > 0 ? std::min<long long>((long long)cc.cap, c->qp_hint + c->qp_hint / 4 + 1024)
                           : (long long)cc.cap / 2;
  return cc;
}

// The grid decision: the grid pays only when the grown obstacles leave most cells empty (large
// maps); a dense grid costs more per edge than it saves.  That is known after building it (the
// fill count needs a host round trip), so the decision is kept per context for the same obstacle
// count and bounds: repeated cuts of one map decide once.  Returns the CutCaps grid mode.
template <int Gc, int Mc>
int grid_decide(Ctx* c, Graph* g, const CutPrep& p, const unsigned char* d_blob) {
  if (!p.grid_cand) return 0;
  const bool known = c->grid_nobs == p.n_obs && c->grid_key[0] == p.blo[0] && c->grid_key[1] == p.blo[1] &&
                     c->grid_key[2] == p.bhi[0] && c->grid_key[3] == p.bhi[1];
  if (known) return c->grid_sparse ? 1 : 0;
  grid_build<Gc, Mc>(c, g, p, d_blob);
  ObsGrid* hg = static_cast<ObsGrid*>(c->host_scratch(sizeof(ObsGrid) + 8 * sizeof(unsigned long long)));
  BZG_CHECK_CUDA(cudaMemcpyAsync(hg, c->ws[WS_OBSGRIDHDR].ptr, sizeof(ObsGrid), cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  // sparse: under 15% of (cell, obstacle) bits set (cfg3's 5 x 5 map is denser and runs faster
  // without the lookups; cfg5's large maps are far sparser)
  const bool sparse = hg->pop * 20 < hg->bits * 3;
  if (c->trace_on)
    std::fprintf(stderr, "[bzg cut] obstacle grid fill %.3f, R %.3f -> %s\n", (double)hg->pop / (double)hg->bits,
                 hg->R, sparse ? "used" : "not used");
  c->grid_nobs = p.n_obs;
  c->grid_key[0] = p.blo[0];
  c->grid_key[1] = p.blo[1];
  c->grid_key[2] = p.bhi[0];
  c->grid_key[3] = p.bhi[1];
  c->grid_sparse = sparse;
  return sparse ? 2 : 0;  // built above
}

// One stream of launches and ONE host synchronisation: the screen's pending count stays on the
// device and every QP kernel reads it there; the per-instance buffers are sized by a capacity
// (the previous cut's count with headroom).  The read-back at the end checks the capacities; an
// overflow (rare: a first cut much larger than the hint) reruns the cut with exact sizes.
void cut_graph_impl(Ctx* c, Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
                    const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
                    Mask* mk, CutBits cbits) {
  const long long E = g->E;
  const int m = g->m;
  BZG_REQUIRE(n_obs >= 0 && n_obs < (1 << 20), BZG_EINVAL, "obstacle count out of range");
  BZG_REQUIRE(E < (1ll << 43), BZG_EUNSUPPORTED, "edge count too large for the QP work list");
  const int qp_rows = check_obstacles(n_obs, row_off, is_box, m);
  mask_begin(c, g, mk, n_obs);
  dispatch_cut(g->gamma, m, [&](auto G_, auto M_) {
    constexpr int Gc = decltype(G_)::value, Mc = decltype(M_)::value;
    CutPrep p;
    cut_prepare_t<Mc>(g, n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg, qp_rows, p);
    DevBuf& d_blob = c->ws[WS_CUTOBS];
    d_blob.alloc(p.blob.size(), c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_blob.ptr, p.blob.data(), p.blob.size(), cudaMemcpyHostToDevice, c->stream));
    const unsigned char* db = d_blob.as<unsigned char>();
    CutCaps cc = default_caps(c, g, p);
    cc.grid = grid_decide<Gc, Mc>(c, g, p, db);
    unsigned long long* hcnt = static_cast<unsigned long long*>(c->host_scratch(8 * sizeof(unsigned long long)));
    for (int attempt = 0;; ++attempt) {
      BZG_REQUIRE(attempt < 4, BZG_ECUDA, "cut work lists kept overflowing");
      cut_enqueue<Gc, Mc>(c, g, p, db, cfg, mk, cbits, cc, hcnt);
      BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
      BZG_REQUIRE(hcnt[7] == 0, BZG_EINVAL, "cannot project onto an empty polytope (geometry.py:226-229)");
      const unsigned long long n_pend = hcnt[5], n_gen = hcnt[6];
      if (n_pend <= cc.cap && n_gen <= cc.gen_cap && (long long)n_pend <= cc.qcap) break;
      // a work list overflowed: grow it and rerun the cut from a clean state
      if (n_pend > cc.cap) cc.cap = n_pend + 1024;
      if (n_gen > cc.gen_cap) cc.gen_cap = n_gen + 1024;
      cc.qcap = std::max<long long>(cc.qcap, (long long)n_pend);
      if (cc.grid == 1) cc.grid = 2;  // built by the first attempt
    }
    const long long n_inst = (long long)hcnt[5];
    c->qp_hint = n_inst;
    c->cut_last_pend = hcnt[5];
    c->cut_last_gen = hcnt[6];
    if (c->trace_on) {
      unsigned long long h8 = 0;
      BZG_CHECK_CUDA(cudaMemcpy(&h8, c->ws[WS_CUTCNT].as<unsigned long long>() + 8, sizeof(h8), cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[bzg cut] pairs %lld, exact codes (pass 2) %llu, code0 %llu code1 %llu code2 %llu\n",
                   E * (long long)n_obs, h8, hcnt[0], hcnt[1], hcnt[2]);
    }
    mask_counters(mk, hcnt);
    // per-QP records of the mask, exact size, filled asynchronously after the read-back
    mk->n_qp = n_inst;
    if (n_inst > 0) {
      mk->qp_status.alloc(n_inst, c->stream);
      mk->qp_iters.alloc(n_inst * sizeof(int), c->stream);
      mk->qp_delta.alloc(n_inst * sizeof(double), c->stream);
      mk->qp_edge.alloc(n_inst * sizeof(long long), c->stream);
      mk->qp_obs.alloc(n_inst * sizeof(int), c->stream);
      BZG_CHECK_CUDA(cudaMemcpyAsync(mk->qp_status.ptr, c->ws[WS_QSTATUS].ptr, n_inst, cudaMemcpyDeviceToDevice,
                                     c->stream));
      BZG_CHECK_CUDA(cudaMemcpyAsync(mk->qp_iters.ptr, c->ws[WS_QITERS].ptr, n_inst * sizeof(int),
                                     cudaMemcpyDeviceToDevice, c->stream));
      BZG_CHECK_CUDA(cudaMemcpyAsync(mk->qp_delta.ptr, c->ws[WS_QDELTA].ptr, n_inst * sizeof(double),
                                     cudaMemcpyDeviceToDevice, c->stream));
      launch(c, "k_unpack_pend", k_unpack_pend, dim3(div_up(n_inst, 256)), dim3(256), 0,
             c->ws[WS_PEND].as<unsigned long long>(), n_inst, mk->qp_edge.as<long long>(), mk->qp_obs.as<int>());
    }
  });
}

// alive / provenance of 32 edges (one bit word) from the obstacles' outcome rows in list order:
// the first event of an edge -- a heuristic kill or a QP-unsafe verdict, never both for one
// obstacle -- decides its provenance (as k_mask_finalize's kh < kq, graph.py:316-340), any
// QP-safe verdict marks a surviving edge QP_SAFE.  One thread per word, so every row word is
// read once for 32 edges (a thread per edge re-read it 32 times in a 3 x n_obs dependent loop).
__global__ void k_cut_combine(long long E, int n_obs, const uint32_t* __restrict__ pool, long long Wb,
                              const int* __restrict__ slots, uint8_t* __restrict__ alive, uint8_t* __restrict__ prov) {
  BZG_PDL_ENTRY();
  const long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (w >= Wb) return;
  uint32_t hk = 0, qk = 0, first_h = 0, saved = 0;
  for (int o = 0; o < n_obs; ++o) {
    const uint32_t* base = pool + (size_t)__ldg(slots + o) * 3 * Wb;
    const uint32_t kill = base[w], qsafe = base[Wb + w], qun = base[2 * Wb + w];
    first_h |= kill & ~(hk | qk);
    hk |= kill;
    qk |= qun;
    saved |= qsafe;
  }
  const uint32_t dead = hk | qk;
  const long long e0 = w * 32;
  const int nb = (int)min(32ll, E - e0);
  auto alive_of = [&](int k) -> uint32_t { return ((dead >> k) & 1u) ? 0u : 1u; };
  auto prov_of = [&](int k) -> uint32_t {
    const uint32_t bit = 1u << k;
    return (dead & bit) ? ((first_h & bit) ? BZG_HEURISTIC_UNSAFE : BZG_QP_UNSAFE)
                        : ((saved & bit) ? BZG_QP_SAFE : BZG_HEURISTIC_SAFE);
  };
  if (nb == 32) {  // 32 bytes each, as two 16-byte stores (the arrays are 256-byte aligned)
    uint32_t a[8], p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = alive_of(4 * j) | alive_of(4 * j + 1) << 8 | alive_of(4 * j + 2) << 16 | alive_of(4 * j + 3) << 24;
      p[j] = prov_of(4 * j) | prov_of(4 * j + 1) << 8 | prov_of(4 * j + 2) << 16 | prov_of(4 * j + 3) << 24;
    }
    uint4* ap = reinterpret_cast<uint4*>(alive + e0);
    uint4* pp = reinterpret_cast<uint4*>(prov + e0);
    ap[0] = make_uint4(a[0], a[1], a[2], a[3]);
    ap[1] = make_uint4(a[4], a[5], a[6], a[7]);
    pp[0] = make_uint4(p[0], p[1], p[2], p[3]);
    pp[1] = make_uint4(p[4], p[5], p[6], p[7]);
  } else {
    for (int k = 0; k < nb; ++k) {
      alive[e0 + k] = (uint8_t)alive_of(k);
      prov[e0 + k] = (uint8_t)prov_of(k);
    }
  }
}

// popcounts of n_rows bit rows of Wb words into out[row]
__global__ void k_row_popcount(const uint32_t* __restrict__ rows, long long Wb, unsigned long long* __restrict__ out) {
  BZG_PDL_ENTRY();
  const uint32_t* r = rows + (size_t)blockIdx.x * Wb;
  unsigned long long s = 0;
  for (long long w = threadIdx.x; w < Wb; w += blockDim.x) s += __popc(r[w]);
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned long long t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) out[blockIdx.x] = t;
}

__global__ void k_remap_int(int* __restrict__ v, long long n, const int* __restrict__ map) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t < n) v[t] = map[v[t]];
}

// The re-cut cache (CutCache, bzg_graph_set_cut_cache): obstacles already cut on this graph --
// same rows, bounds and configuration, bit for bit -- contribute their stored outcome rows;
// the others (moved obstacles in a replanning loop, sim.py:324-330) are cut now, as a sub-list,
// recording their rows.  k_cut_combine then rebuilds alive / provenance in list order and the
// counters are sums of per-obstacle popcounts, so the mask equals a full cut's.  The QP
// records (qp_records) cover the QPs solved by this call.  Returns false when the list does
// not fit the cache (the caller cuts without it).
bool cut_graph_cached(Ctx* c, Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
                      const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
                      Mask* mk) {
  CutCache& cc = g->cut_cache;
  const long long E = g->E;
  const int m = g->m;
  const long long Wb = (E + 31) / 32;
  if (n_obs > cc.max_slots || E <= 0) return false;
  check_obstacles(n_obs, row_off, is_box, m);
  if (cc.Wb != Wb || (int)cc.key_of.size() != cc.max_slots) {
    cc.clear();
    cc.Wb = Wb;
    cc.key_of.assign(cc.max_slots, std::string());
    cc.stamp.assign(cc.max_slots, 0);
    cc.cnt.assign((size_t)cc.max_slots * 3, 0);
    cc.pool.alloc((size_t)cc.max_slots * 3 * Wb * sizeof(uint32_t), c->stream);
  }
  // keys: the obstacle's normalised rows, bounds, box flag and the whole cut configuration
  std::vector<std::string> keys(n_obs);
  for (int o = 0; o < n_obs; ++o) {
    const int r0 = row_off[o], r1 = row_off[o + 1];
    std::string k;
    k.append(reinterpret_cast<const char*>(cfg), sizeof(*cfg));
    k.append(reinterpret_cast<const char*>(A + (size_t)r0 * m), (size_t)(r1 - r0) * m * sizeof(double));
    k.append(reinterpret_cast<const char*>(b + r0), (size_t)(r1 - r0) * sizeof(double));
    k.push_back((char)is_box[o]);
    k.append(reinterpret_cast<const char*>(box_lo + (size_t)o * m), m * sizeof(double));
    k.append(reinterpret_cast<const char*>(box_hi + (size_t)o * m), m * sizeof(double));
    keys[o] = std::move(k);
  }
  ++cc.clock;
  std::unordered_map<std::string, int> in_list;
  for (int o = 0; o < n_obs; ++o) in_list.emplace(keys[o], o);
  // misses: distinct keys not cached, in first-occurrence order
  std::vector<int> miss;
  {
    std::unordered_map<std::string, int> seen;
    for (int o = 0; o < n_obs; ++o) {
      auto it = cc.slot_of.find(keys[o]);
      if (it != cc.slot_of.end()) { cc.stamp[it->second] = cc.clock; continue; }
      if (seen.emplace(keys[o], o).second) miss.push_back(o);
    }
  }
  // slots for the misses: free slots first, then least recently used ones not in this list
  // (enough exist: the list's own slots are at most n_obs - misses of the max_slots >= n_obs)
  {
    int avail = 0;
    for (int sl = 0; sl < cc.max_slots; ++sl)
      avail += cc.key_of[sl].empty() || (cc.stamp[sl] != cc.clock && !in_list.count(cc.key_of[sl]));
    if (avail < (int)miss.size()) return false;
  }
  std::vector<int> new_slot(miss.size());
  for (size_t i = 0; i < miss.size(); ++i) {
    int best = -1;
    for (int sl = 0; sl < cc.max_slots; ++sl) {
      const bool empty = cc.key_of[sl].empty();
      if (!empty && (cc.stamp[sl] == cc.clock || in_list.count(cc.key_of[sl]))) continue;  // in use now
      if (best < 0) { best = sl; continue; }
      const bool best_empty = cc.key_of[best].empty();
      if ((empty && !best_empty) || (empty == best_empty && cc.stamp[sl] < cc.stamp[best])) best = sl;
    }
    if (best < 0) return false;  // cannot happen while n_obs <= max_slots
    if (!cc.key_of[best].empty()) cc.slot_of.erase(cc.key_of[best]);
    cc.key_of[best] = keys[miss[i]];
    cc.slot_of[keys[miss[i]]] = best;
    cc.stamp[best] = cc.clock;
    new_slot[i] = best;
  }
  mask_begin(c, g, mk, n_obs);
  for (DevBuf* key : {&mk->tree_key, &mk->reach_key})  // the mask's alive set changes: no cached tree
    if (key->ptr) BZG_CHECK_CUDA(cudaMemsetAsync(key->ptr, 0xFF, sizeof(long long), c->stream));
  const int nm = (int)miss.size();
  if (nm > 0) {
    // the misses as a sub-list, cut with their outcome rows recorded
    std::vector<int32_t> sro(nm + 1, 0);
    std::vector<double> sA, sb, slo, shi;
    std::vector<uint8_t> sbox(nm);
    for (int i = 0; i < nm; ++i) {
      const int o = miss[i], r0 = row_off[o], r1 = row_off[o + 1];
      sro[i + 1] = sro[i] + (r1 - r0);
      sA.insert(sA.end(), A + (size_t)r0 * m, A + (size_t)r1 * m);
      sb.insert(sb.end(), b + r0, b + r1);
      sbox[i] = is_box[o];
      slo.insert(slo.end(), box_lo + (size_t)o * m, box_lo + (size_t)(o + 1) * m);
      shi.insert(shi.end(), box_hi + (size_t)o * m, box_hi + (size_t)(o + 1) * m);
    }
    DevBuf& tmp = c->ws[WS_CUTBITS];
    tmp.alloc((size_t)3 * nm * Wb * sizeof(uint32_t), c->stream);
    BZG_CHECK_CUDA(cudaMemsetAsync(tmp.ptr, 0, (size_t)3 * nm * Wb * sizeof(uint32_t), c->stream));
    uint32_t* tk = tmp.as<uint32_t>();
    CutBits bits{tk, tk + (size_t)nm * Wb, tk + (size_t)2 * nm * Wb, Wb, Wb};
    try {
      cut_graph_impl(c, g, nm, sro.data(), sA.data(), sb.data(), sbox.data(), slo.data(), shi.data(), cfg, mk, bits);
    } catch (...) {  // the new slots hold no outcome rows: forget them
      for (int i = 0; i < nm; ++i) {
        cc.slot_of.erase(cc.key_of[new_slot[i]]);
        cc.key_of[new_slot[i]].clear();
      }
      throw;
    }
    // per-obstacle popcounts, the rows into their slots
    c->arena->reset();
    TmpBuf d_pc(c);
    d_pc.alloc((size_t)3 * nm * sizeof(unsigned long long), c->stream);
    launch(c, "k_row_popcount", k_row_popcount, dim3(3 * nm), dim3(256), 0, (const uint32_t*)tk, Wb,
           d_pc.as<unsigned long long>());
    for (int i = 0; i < nm; ++i)
      for (int r = 0; r < 3; ++r)
        BZG_CHECK_CUDA(cudaMemcpyAsync(cc.pool.as<uint32_t>() + ((size_t)new_slot[i] * 3 + r) * Wb,
                                       tk + ((size_t)r * nm + i) * Wb, Wb * sizeof(uint32_t),
                                       cudaMemcpyDeviceToDevice, c->stream));
    std::vector<unsigned long long> hpc(3 * nm);
    BZG_CHECK_CUDA(cudaMemcpyAsync(hpc.data(), d_pc.ptr, hpc.size() * sizeof(unsigned long long),
                                   cudaMemcpyDeviceToHost, c->stream));
    // QP records: sub-list obstacle index -> its first position in the full list
    if (mk->n_qp > 0) {
      TmpBuf d_map(c);
      d_map.alloc(nm * sizeof(int), c->stream);
      BZG_CHECK_CUDA(cudaMemcpyAsync(d_map.ptr, miss.data(), nm * sizeof(int), cudaMemcpyHostToDevice, c->stream));
      launch(c, "k_remap_int", k_remap_int, dim3(div_up(mk->n_qp, 256)), dim3(256), 0, mk->qp_obs.as<int>(), mk->n_qp,
             (const int*)d_map.as<int>());
    }
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < nm; ++i)
      for (int r = 0; r < 3; ++r) cc.cnt[(size_t)new_slot[i] * 3 + r] = (long long)hpc[(size_t)r * nm + i];
  }
  // recombine the whole list from the slots
  std::vector<int> slots(n_obs);
  for (int o = 0; o < n_obs; ++o) slots[o] = cc.slot_of.at(keys[o]);
  DevBuf& d_slots = c->ws[WS_CUTSLOTS];
  d_slots.alloc(n_obs * sizeof(int), c->stream);
  BZG_CHECK_CUDA(cudaMemcpyAsync(d_slots.ptr, slots.data(), n_obs * sizeof(int), cudaMemcpyHostToDevice, c->stream));
  launch(c, "k_cut_combine", k_cut_combine, dim3(div_up(Wb, 256)), dim3(256), 0, E, n_obs,
         (const uint32_t*)cc.pool.as<uint32_t>(), Wb, (const int*)d_slots.as<int>(), mk->alive.as<uint8_t>(),
         mk->prov.as<uint8_t>());
  long long kill = 0, qs = 0, qu = 0;
  for (int o = 0; o < n_obs; ++o) {
    kill += cc.cnt[(size_t)slots[o] * 3 + 0];
    qs += cc.cnt[(size_t)slots[o] * 3 + 1];
    qu += cc.cnt[(size_t)slots[o] * 3 + 2];
  }
  mk->counters[0] = E * (long long)n_obs;
  mk->counters[1] = kill;
  mk->counters[3] = qs + qu;
  mk->counters[2] = mk->counters[0] - kill - (qs + qu);
  mk->counters[4] = qs;
  mk->counters[5] = qu;
  // the host sync that returns counters to the caller is the mask read-back (stream-ordered)
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  return true;
}

}  // namespace

}  // namespace bzg

#include "k_plans.cuh"

namespace bzg {

void cut_graph(Ctx* c, Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
               const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
               Mask* mk) {
  if (g->cut_cache.max_slots > 0 && n_obs > 0 &&
      cut_graph_cached(c, g, n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg, mk))
    return;
  cut_graph_impl(c, g, n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg, mk, CutBits{});
}

// The reference's scalar entry points on explicit control-point sets: cut_heuristic
// (graph.py:202-221, mode 0 -> code 0/1/2) and cut_qp (graph.py:285-299, mode 1 -> safe flag,
// ||delta||, solver status), set b against obstacle obs_index[b].  The sets become a
// pseudo-graph: vertex 2b holds control points 0..G-1 of set b, vertex 2b+1 points G..J-1,
// edge b = (2b, 2b+1) and D = I, so control_points() reproduces every set exactly (products
// with 1, FMAs with 0) and the graph kernels run unchanged.
void cut_points(Ctx* c, int m, int J, long long B, const double* points, const int32_t* obs_index, int n_obs,
                const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box, const double* box_lo,
                const double* box_hi, const bzg_cut_config* cfg, int mode, int8_t* code_out, double* delta_out,
                int8_t* status_out) {
  BZG_REQUIRE(mode == 0 || mode == 1, BZG_EINVAL, "mode must be 0 (cut_heuristic) or 1 (cut_qp)");
  BZG_REQUIRE(J >= 2 && J % 2 == 0, BZG_EUNSUPPORTED, "the device takes an even control-point count (p = 2*gamma - 1)");
  BZG_REQUIRE(B >= 0 && B < (1ll << 30), BZG_EINVAL, "set count out of range");
  BZG_REQUIRE(n_obs >= 1 && n_obs < (1 << 20), BZG_EINVAL, "obstacle count out of range");
  const int qp_rows = check_obstacles(n_obs, row_off, is_box, m);
  for (long long i = 0; i < B; ++i)
    BZG_REQUIRE(obs_index[i] >= 0 && obs_index[i] < n_obs, BZG_EINVAL, "obstacle index out of range");
  if (B == 0) return;
  const int G = J / 2;
  Graph g;
  g.ctx = c;
  g.m = m;
  g.gamma = G;
  g.p = J - 1;
  g.n = m * G;
  g.V = 2 * B;
  g.D.assign((size_t)J * J, 0.0);
  for (int j = 0; j < J; ++j) g.D[(size_t)j * J + j] = 1.0;
  std::vector<double> V((size_t)2 * B * m * G);
  std::vector<int32_t> src(B), dst(B);
  std::vector<unsigned long long> items(B);
  for (long long s = 0; s < B; ++s) {
    const double* P = points + (size_t)s * m * J;
    for (int q = 0; q < G; ++q)
      for (int k = 0; k < m; ++k) {
        V[(size_t)(2 * s) * m * G + q * m + k] = P[k * J + q];
        V[(size_t)(2 * s + 1) * m * G + q * m + k] = P[k * J + G + q];
      }
    src[s] = (int32_t)(2 * s);
    dst[s] = (int32_t)(2 * s + 1);
    items[s] = ((unsigned long long)s << 20) | (unsigned long long)obs_index[s];
  }
  const std::vector<double> cost(B, 0.0);
  g.vertices.alloc(V.size() * sizeof(double), c->stream);
  BZG_CHECK_CUDA(cudaMemcpyAsync(g.vertices.ptr, V.data(), V.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  set_edges(c, &g, B, src.data(), dst.data(), cost.data(), false);
  DParams dp{};
  for (size_t k = 0; k < g.D.size(); ++k) dp.D[k] = g.D[k];
  dispatch_cut(G, m, [&](auto G_, auto M_) {
    constexpr int Gc = decltype(G_)::value, Mc = decltype(M_)::value;
    using Rec = ObsRec<Mc>;
    const std::vector<Rec> h = fill_obs<Mc>(n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg->eps_geo);
    const bool big = qp_rows > kObsRows;
    const std::vector<ObsRec<Mc, kObsRowsBig>> hbig =
        big ? fill_obs<Mc, kObsRowsBig>(n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg->eps_geo)
            : std::vector<ObsRec<Mc, kObsRowsBig>>();
    DevBuf d_obs, d_items;
    const size_t obytes = big ? sizeof(ObsRec<Mc, kObsRowsBig>) * hbig.size() : sizeof(Rec) * h.size();
    d_obs.alloc(obytes, c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_obs.ptr, big ? (const void*)hbig.data() : (const void*)h.data(), obytes,
                                   cudaMemcpyHostToDevice, c->stream));
    d_items.alloc(B * sizeof(unsigned long long), c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_items.ptr, items.data(), B * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                                   c->stream));
    if (mode == 0) {
      DevBuf d_kill, d_cnt, d_pend, d_code;
      d_kill.alloc(B * sizeof(int), c->stream);
      d_cnt.alloc(8 * sizeof(unsigned long long), c->stream);
      d_pend.alloc(B * sizeof(unsigned long long), c->stream);
      d_code.alloc(B, c->stream);
      BZG_CHECK_CUDA(cudaMemsetAsync(d_cnt.ptr, 0, 8 * sizeof(unsigned long long), c->stream));
      launch(c, "k_fill_int", k_fill_int, dim3(div_up(B, 256)), dim3(256), 0, d_kill.as<int>(), B, n_obs);
      unsigned long long* dcnt = d_cnt.as<unsigned long long>();
      if (big)
        launch(c, "k_cut_general", k_cut_general<Gc, Mc, kObsRowsBig>, dim3(div_up(B, 64)), dim3(64), 0, dp,
               g.vertices.as<double>(), g.src.as<int>(), g.dst.as<int>(), (const ObsRec<Mc, kObsRowsBig>*)d_obs.ptr,
               d_items.as<unsigned long long>(), B, (const unsigned long long*)nullptr, cfg->heur_margin,
               d_kill.as<int>(), dcnt, dcnt + 5, (unsigned long long)B, d_pend.as<unsigned long long>(),
               d_code.as<int8_t>(), CutBits{});
      else
        launch(c, "k_cut_general", k_cut_general<Gc, Mc, kObsRows>, dim3(div_up(B, 64)), dim3(64), 0, dp,
               g.vertices.as<double>(), g.src.as<int>(), g.dst.as<int>(), d_obs.as<Rec>(),
               d_items.as<unsigned long long>(), B, (const unsigned long long*)nullptr, cfg->heur_margin,
               d_kill.as<int>(), dcnt, dcnt + 5, (unsigned long long)B, d_pend.as<unsigned long long>(),
               d_code.as<int8_t>(), CutBits{});
      unsigned long long* hcnt = static_cast<unsigned long long*>(c->host_scratch(8 * sizeof(unsigned long long)));
      BZG_CHECK_CUDA(cudaMemcpyAsync(hcnt, d_cnt.ptr, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
      BZG_CHECK_CUDA(cudaMemcpyAsync(code_out, d_code.ptr, B, cudaMemcpyDeviceToHost, c->stream));
      BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
      BZG_REQUIRE(hcnt[7] == 0, BZG_EINVAL, "cannot project onto an empty polytope (geometry.py:226-229)");
      return;
    }
    bool canon_all = true;
    for (int o = 0; o < n_obs; ++o) canon_all = canon_all && h[o].canon != 0.0;
    Mask mk;
    mk.g = &g;
    mk.ctx = c;
    mk.E = B;
    DevBuf &d_safe = c->ws[WS_QSAFE];
    dispatch_rows<Mc>(qp_rows, [&](auto C_) {
      mk.qp_status.alloc(B, c->stream);
      mk.qp_iters.alloc(B * sizeof(int), c->stream);
      mk.qp_delta.alloc(B * sizeof(double), c->stream);
      d_safe.alloc(B, c->stream);
      QpJob job{&g, {}, d_obs.ptr, canon_all, d_items.as<unsigned long long>(), B, nullptr, cfg, cfg->qp_polish ? 2 : 0,
                0.0, &mk, &d_safe, mk.qp_status.as<int8_t>(), mk.qp_iters.as<int>(), mk.qp_delta.as<double>()};
      for (int k = 0; k < 64; ++k) job.D[k] = dp.D[k];
      qp_solve(c, Gc, Mc, decltype(C_)::value, job);
    });
    if (code_out) BZG_CHECK_CUDA(cudaMemcpyAsync(code_out, d_safe.ptr, B, cudaMemcpyDeviceToHost, c->stream));
    if (delta_out)
      BZG_CHECK_CUDA(cudaMemcpyAsync(delta_out, mk.qp_delta.ptr, B * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (status_out) BZG_CHECK_CUDA(cudaMemcpyAsync(status_out, mk.qp_status.ptr, B, cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // namespace bzg
