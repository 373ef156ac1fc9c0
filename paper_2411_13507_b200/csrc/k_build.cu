// Graph build on device: PCG64 state sampling, oracle projections, all-pairs
// reachability test into a bit matrix, ordered CSR compaction and edge costs.
//
// Replaces reference graph.py:147-197 (build_graph).  Arithmetic order follows
// SURVEY.md §8(c) so vertices, edges, costs and control points are bitwise equal
// to the reference.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "bzg_internal.cuh"
#include "bzg_math.cuh"

namespace bzg {

namespace {

constexpr int kMaxN = 16;        // reduced state dimension n = m*gamma
constexpr int kMaxRows = 64;     // rows of the sampler's state polytope
constexpr int kMaxIntervals = 64;

struct SampleParams {
  double lo[kMaxN], range[kMaxN];
  double A[kMaxRows * kMaxN];
  double b_eps[kMaxRows];
  int n, rows;
};

// One thread per candidate row: jump the PCG64 stream to draw row*n, draw the n
// uniforms of that row (geometry.py:69-72 -> numpy random_uniform: lo + range*u,
// range = hi - lo) and test Xd membership (geometry.py:145-148).
// pcg_dev non-null: the four PCG64 words (state hi/lo, inc hi/lo) read from device memory (a
// captured plan's staging) instead of the by-value ones
__global__ void k_sample_candidates(SampleParams sp, unsigned long long st_hi, unsigned long long st_lo,
                                    unsigned long long inc_hi, unsigned long long inc_lo, long long row0,
                                    long long count, double* __restrict__ cand, int* __restrict__ flag,
                                    const unsigned long long* __restrict__ pcg_dev) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= count) return;
  if (pcg_dev) {
    st_hi = pcg_dev[0];
    st_lo = pcg_dev[1];
    inc_hi = pcg_dev[2];
    inc_lo = pcg_dev[3];
  }
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  u128 s = ((u128)st_hi << 64) | st_lo;
  s = pcg_advance(s, inc, (uint64_t)(row0 + t) * (uint64_t)sp.n);
  double x[kMaxN];
  for (int k = 0; k < sp.n; ++k) {
    const double u = pcg_next_double(s, inc);
    x[k] = __dadd_rn(sp.lo[k], __dmul_rn(sp.range[k], u));
    cand[t * sp.n + k] = x[k];
  }
  int ok = 1;
  for (int c = 0; c < sp.rows; ++c) ok &= fma_chain(x, sp.A + c * sp.n, sp.n) <= sp.b_eps[c];
  flag[t] = ok;
}

__global__ void k_sample_scatter(const double* __restrict__ cand, const int* __restrict__ flag,
                                 const int* __restrict__ pos, long long count, int n, long long need,
                                 double* __restrict__ out) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= count || !flag[t]) return;
  const long long p = pos[t];
  if (p >= need) return;
  for (int k = 0; k < n; ++k) out[p * n + k] = cand[t * n + k];
}

// ---------------------------------------------------------------- multi-region sampler
// All keep-in regions in one launch per round (regions.py sample_region_states): region r
// draws from its own PCG64 stream (default_rng([seed, r])) inside its own sampling box and
// accepts in its own state polytope rows [row_off[r], row_off[r+1]) -- build_graph's sampler
// (graph.py:147-157) per region.  Candidate t belongs to region r with
// cand_off[r] <= t < cand_off[r+1].
struct RegionSampleDev {
  const unsigned long long* pcg;  // R x 4: state_hi, state_lo, inc_hi, inc_lo
  const double* lo;               // R x n
  const double* range;            // R x n (hi - lo)
  const int* row_off;             // R + 1
  const double* A;                // rows x n
  const double* b_eps;            // rows
  const long long* cand_off;      // R + 1 (this round)
  const long long* row0;          // R: first stream row of this round
  int n, R;
};

__device__ __forceinline__ int region_of(const long long* off, int R, long long t) {
  int lo = 0, hi = R;  // largest r with off[r] <= t
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_sample_regions(RegionSampleDev rs, long long total, double* __restrict__ cand,
                                 int* __restrict__ flag) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= total) return;
  const int r = region_of(rs.cand_off, rs.R, t);
  const int n = rs.n;
  const unsigned long long* w = rs.pcg + 4 * r;
  const u128 inc = ((u128)w[2] << 64) | w[3];
  u128 s = ((u128)w[0] << 64) | w[1];
  s = pcg_advance(s, inc, (uint64_t)(rs.row0[r] + (t - rs.cand_off[r])) * (uint64_t)n);
  double x[kMaxN];
  for (int k = 0; k < n; ++k) {
    const double u = pcg_next_double(s, inc);
    x[k] = __dadd_rn(rs.lo[r * n + k], __dmul_rn(rs.range[r * n + k], u));
    cand[t * n + k] = x[k];
  }
  int ok = 1;
  for (int c = rs.row_off[r]; c < rs.row_off[r + 1]; ++c) ok &= fma_chain(x, rs.A + (size_t)c * n, n) <= rs.b_eps[c];
  flag[t] = ok;
}

// accepted candidate t of region r lands at dest[r] + (its rank among r's acceptances) if that
// rank is below need[r]; acc[r] = acceptances of r this round
__global__ void k_scatter_regions(const double* __restrict__ cand, const int* __restrict__ flag,
                                  const int* __restrict__ pos, const long long* __restrict__ cand_off, int R,
                                  long long total, int n, const long long* __restrict__ dest,
                                  const long long* __restrict__ need, double* __restrict__ out) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= total || !flag[t]) return;
  const int r = region_of(cand_off, R, t);
  const long long p = pos[t] - pos[cand_off[r]];
  if (p >= need[r]) return;
  for (int k = 0; k < n; ++k) out[(dest[r] + p) * n + k] = cand[t * n + k];
}

__global__ void k_region_acc(const int* __restrict__ pos, const long long* __restrict__ cand_off, int R,
                             long long* __restrict__ acc) {
  BZG_PDL_ENTRY();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) acc[r] = (long long)pos[cand_off[r + 1]] - (long long)pos[cand_off[r]];
}

// ---------------------------------------------------------------- projections
struct RowPlan {
  int n, K, n_src, n_dst;
  int row_iv[kMaxIntervals];   // F row of each interval (the "+" row of a negation pair)
  int row_src[kMaxIntervals];  // x1-only rows (F2 row == 0)
  int row_dst[kMaxIntervals];  // x2-only rows (F1 row == 0)
  double th_src[kMaxIntervals], th_dst[kMaxIntervals];
};

// ---------------------------------------------------------------- pair test
struct Bounds {
  double lo[kMaxIntervals], hi[kMaxIntervals];
};

constexpr int kPairThreads = 256;  // dst columns per block (8 warps x 32)

// Bit (i, j) of the pair matrix (graph.py:181-184): fl(a1[i,r] + a2[j,r]) <= G_r + eps for
// every row r, evaluated as intervals lo_q <= a1c[i,q] + a2[j,q] <= hi_q over the negation
// pairs plus the per-vertex one-sided predicates, diagonal cleared.
// ---------------------------------------------------------------- spatially tiled pair test
// Vertices are visited in Morton order of their position so that a warp's 32 destinations
// (a "group") and a block's 32 sources (a "tile") are close in state space.  Per interval q
// the group's [min, max] of a2 and the tile's [min, max] of a1 bound every pair sum; since
// fl(a + b) is monotone in each argument, fl(min1 + min2) > hi_q (or fl(max1 + max2) < lo_q)
// proves every pair of the block fails row q -- an exact cull.  Surviving (source, group)
// pairs are culled again with the source's own a1, and only then tested lane by lane.  Edge
// bits land in the original-index bit matrix (atomicOr), so the CSR order is unchanged.
constexpr int kTile = 32;

__global__ void k_morton(const double* __restrict__ Vx, long long V, int n, int m, double lo0, double lo1,
                         double lo2, double s0, double s1, double s2, unsigned* __restrict__ key, int* __restrict__ idx) {
  BZG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= V) return;
  const int bits = m == 1 ? 30 : (m == 2 ? 16 : 10);
  const unsigned cap = (1u << bits) - 1u;
  auto cell = [&](int k, double lo, double s) -> unsigned {
    const double t = (Vx[i * n + k] - lo) * s;
    return t <= 0.0 ? 0u : (t >= (double)cap ? cap : (unsigned)t);
  };
  unsigned c[3] = {cell(0, lo0, s0), m > 1 ? cell(1, lo1, s1) : 0u, m > 2 ? cell(2, lo2, s2) : 0u};
  unsigned code = 0;
  for (int b = bits - 1; b >= 0; --b)
    for (int k = 0; k < m; ++k) code = (code << 1) | ((c[k] >> b) & 1u);
  key[i] = code;
  idx[i] = (int)i;
}

// projections at sorted position s (vertex perm[s]); src_ok also requires the row block
// The oracle rows F (n_F x 2n, at most 96 x 12 doubles) are staged in shared memory first: read
// from global memory inside the per-row loops, every row was a dependent L2 round trip (~36 per
// vertex at gamma = 2), which made this kernel latency-bound at every size (18 us for 202
// vertices).  Same arithmetic (fma_chain over the same values).
__global__ void k_project_sorted(RowPlan rp, const double* __restrict__ F, int nF, const double* __restrict__ Vx,
                                 const int* __restrict__ perm, long long V, int Kpad, long long r0, long long r1,
                                 double* __restrict__ a1c, double* __restrict__ a2t, uint8_t* __restrict__ src_ok,
                                 uint8_t* __restrict__ dst_ok) {
  BZG_PDL_ENTRY();
  extern __shared__ double sF[];
  const int n = rp.n;
  for (int t = threadIdx.x; t < nF * 2 * n; t += blockDim.x) sF[t] = F[t];
  __syncthreads();
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= V) return;
  const long long i = perm[s];
  double v[kMaxN];
  for (int k = 0; k < n; ++k) v[k] = Vx[i * n + k];
  for (int q = 0; q < Kpad; ++q) {
    double x1 = 0.0, x2 = 0.0;
    if (q < rp.K) {
      const double* f = sF + (size_t)rp.row_iv[q] * 2 * n;
      x1 = fma_chain(v, f, n);
      x2 = fma_chain(v, f + n, n);
    }
    a1c[s * Kpad + q] = x1;
    a2t[(long long)q * V + s] = x2;
  }
  int ok = i >= r0 && i < r1;
  for (int q = 0; q < rp.n_src; ++q) ok &= fma_chain(v, sF + (size_t)rp.row_src[q] * 2 * n, n) <= rp.th_src[q];
  src_ok[s] = (uint8_t)ok;
  ok = 1;
  for (int q = 0; q < rp.n_dst; ++q) ok &= fma_chain(v, sF + (size_t)rp.row_dst[q] * 2 * n + n, n) <= rp.th_dst[q];
  dst_ok[s] = (uint8_t)ok;
}

// A row block's own sources, in the Morton order of the full sort: sorted positions whose
// vertex lies in [r0, r1) (flag + exclusive scan -> pos), then gathered so source tiles are
// dense in the block (a tile of the full order would hold ~32 / G of them).
__global__ void k_src_flags(const int* __restrict__ perm, long long V, long long r0, long long r1, int* __restrict__ flag) {
  BZG_PDL_ENTRY();
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s < V) flag[s] = (perm[s] >= r0 && perm[s] < r1) ? 1 : 0;
}

__global__ void k_src_gather(const int* __restrict__ perm, const int* __restrict__ flag, const int* __restrict__ pos,
                             long long V, int Kpad, const double* __restrict__ a1c, const uint8_t* __restrict__ src_ok,
                             const unsigned long long* __restrict__ smask, int RW, int* __restrict__ perm_src,
                             double* __restrict__ a1c_src, uint8_t* __restrict__ ok_src,
                             unsigned long long* __restrict__ smask_src) {
  BZG_PDL_ENTRY();
  const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= V || !flag[s]) return;
  const long long t = pos[s];
  perm_src[t] = perm[s];
  ok_src[t] = src_ok[s];
  for (int q = 0; q < Kpad; ++q) a1c_src[t * Kpad + q] = a1c[s * Kpad + q];
  for (int w = 0; w < RW; ++w) smask_src[t * RW + w] = smask[s * RW + w];
}

// [min, max] per (32-vertex group, interval) over the group's valid vertices
__global__ void k_group_bounds(const double* __restrict__ a, int transposed, long long V, int Kpad,
                               const uint8_t* __restrict__ ok, double* __restrict__ gmin, double* __restrict__ gmax) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long ng = (V + kTile - 1) / kTile;
  if (t >= ng * Kpad) return;
  const long long g = t / Kpad;
  const int q = (int)(t - g * Kpad);
  double mn = INFINITY, mx = -INFINITY;
  // loads issued unconditionally (independent, pipelined by the unroll); excluded rows select
  // the identities of fmin / fmax, so the bounds are exactly the conditional loop's
#pragma unroll 8
  for (int l = 0; l < kTile; ++l) {
    const long long s = g * kTile + l;
    const bool in = s < V;
    const long long sc = in ? s : 0;
    const bool use = in && ok[sc];
    const double v = transposed ? a[(long long)q * V + sc] : a[sc * Kpad + q];
    mn = fmin(mn, use ? v : INFINITY);
    mx = fmax(mx, use ? v : -INFINITY);
  }
  gmin[t] = mn;
  gmax[t] = mx;
}

// ---------------------------------------------------------------- keep-in regions
// Region r's added rows are one-sided, so region membership is a per-vertex bit: smask (as
// source, x1-only rows) and dmask (as destination, x2-only rows); an edge needs the base
// test and a common region, (S_i & D_j) != 0.
constexpr int kMaxRegionWords = 4;  // up to 256 regions

struct RegionRowsDev {
  const int* src_off;  // per region, rows [src_off[r], src_off[r+1]) of src_F / src_th
  const double* src_F; // (rows, n): F1 part of x1-only rows
  const double* src_th;
  const int* dst_off;
  const double* dst_F; // (rows, n): F2 part of x2-only rows
  const double* dst_th;
  int R, RW, n;
};

// G lanes per sorted vertex (G a power of two <= 32, sized by the host so V x G fills the GPU),
// each lane testing every G-th region of a 64-region mask word: regions whose (1e-6-grown)
// position box misses the vertex are skipped (membership implies P_0 = x1 resp. P_p = x2 lies
// in the region), the rest are tested row by row; the group ORs its bits by shuffles.  The
// group writes its vertex's mask words whole (no pre-zeroing) and folds them: a vertex in no
// region can neither start nor end an edge (src_ok / dst_ok cleared).  (One thread per vertex
// looping over all regions was latency-bound at 10 k vertices: 93 us at cfg5-10k's 200
// regions; one warp per vertex doubled the instructions at 100 k: 85 -> 195 us.)
__global__ void k_region_masks(RegionRowsDev rr, const double* __restrict__ Vx, const int* __restrict__ perm,
                               long long V, int m, const double* __restrict__ blo, const double* __restrict__ bhi,
                               unsigned long long* __restrict__ smask, unsigned long long* __restrict__ dmask,
                               uint8_t* __restrict__ src_ok, uint8_t* __restrict__ dst_ok, int G) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long s = t / G;
  const int sub = (int)(t % G);
  if (s >= V) return;  // uniform across the group
  const int lane = threadIdx.x & 31;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
  const long long i = perm[s];
  const int n = rr.n;
  double v[kMaxN];
  for (int k = 0; k < n; ++k) v[k] = Vx[i * n + k];
  bool any_s = false, any_d = false;
  for (int w = 0; w < rr.RW; ++w) {
    unsigned long long ms = 0, md = 0;
    for (int j = sub; j < 64; j += G) {
      const int r = w * 64 + j;
      if (r >= rr.R) break;
      bool inbox = true;
      if (blo)
        for (int k = 0; k < m; ++k) inbox &= (v[k] >= blo[r * m + k] - 1e-6) & (v[k] <= bhi[r * m + k] + 1e-6);
      if (!inbox) continue;
      int in_s = 1, in_d = 1;
      for (int q = rr.src_off[r]; q < rr.src_off[r + 1]; ++q)
        in_s &= fma_chain(v, rr.src_F + (size_t)q * n, n) <= rr.src_th[q];
      for (int q = rr.dst_off[r]; q < rr.dst_off[r + 1]; ++q)
        in_d &= fma_chain(v, rr.dst_F + (size_t)q * n, n) <= rr.dst_th[q];
      if (in_s) ms |= 1ull << j;
      if (in_d) md |= 1ull << j;
    }
    for (int off = G / 2; off > 0; off >>= 1) {
      ms |= __shfl_xor_sync(gmask, ms, off);
      md |= __shfl_xor_sync(gmask, md, off);
    }
    if (sub == 0) {
      smask[s * rr.RW + w] = ms;
      dmask[s * rr.RW + w] = md;
    }
    any_s |= ms != 0;
    any_d |= md != 0;
  }
  if (sub == 0) {
    if (!any_s) src_ok[s] = 0;
    if (!any_d) dst_ok[s] = 0;
  }
}

// OR of the masks over each 32-vertex group (tile / destination group cull); blockIdx.y = 1
// handles a second (mask, ok, out) triple in the same launch
__global__ void k_mask_or(const unsigned long long* __restrict__ mask, const uint8_t* __restrict__ ok, long long V,
                          int RW, unsigned long long* __restrict__ out, const unsigned long long* __restrict__ mask2,
                          const uint8_t* __restrict__ ok2, unsigned long long* __restrict__ out2) {
  BZG_PDL_ENTRY();
  if (blockIdx.y) {
    mask = mask2;
    ok = ok2;
    out = out2;
  }
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long ng = (V + kTile - 1) / kTile;
  if (t >= ng * RW) return;
  const long long g = t / RW;
  const int w = (int)(t - g * RW);
  unsigned long long acc = 0;
  for (int l = 0; l < kTile; ++l) {
    const long long s = g * kTile + l;
    if (s < V && ok[s]) acc |= mask[s * RW + w];
  }
  out[t] = acc;
}

struct RegionMasks {
  const unsigned long long *smask, *dmask, *tile_or, *group_or;
  int RW;
};

template <int K, bool REG>
__global__ void __launch_bounds__(kPairThreads, 3) k_pair_tiles(
    Bounds bd, const double* __restrict__ a1c, const double* __restrict__ a2t, const uint8_t* __restrict__ src_ok,
    const uint8_t* __restrict__ dst_ok, const int* __restrict__ perm, const double* __restrict__ tmin,
    const double* __restrict__ tmax, const double* __restrict__ gmin, const double* __restrict__ gmax, long long V,
    long long r0, long long W, uint32_t* __restrict__ bits, unsigned long long* __restrict__ rowcnt,
    RegionMasks rm, const int* __restrict__ perm_src, long long V_src) {
  BZG_PDL_ENTRY();
  __shared__ double s_a1[kTile][K];
  __shared__ uint8_t s_ok[kTile];
  __shared__ int s_orig[kTile];
  __shared__ unsigned long long s_sm[REG ? kTile : 1][kMaxRegionWords];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long tile = blockIdx.y;
  const long long i0 = tile * kTile;
  const int rows = (int)min((long long)kTile, V_src - i0);
  const long long g = (long long)blockIdx.x * (kPairThreads / 32) + warp;
  // ---- (tile, group) culls first: a block whose eight groups all fail skips the staging
  bool live = g * kTile < V;
  unsigned long long gor[kMaxRegionWords] = {0, 0, 0, 0}, dm[kMaxRegionWords] = {0, 0, 0, 0};
  if (REG && live) {
    bool share = false;
#pragma unroll
    for (int w = 0; w < kMaxRegionWords; ++w) {
      if (w < rm.RW) {
        gor[w] = rm.group_or[g * rm.RW + w];
        share |= (gor[w] & rm.tile_or[tile * rm.RW + w]) != 0;
      }
    }
    live = share;  // no region holds a source of the tile and a destination of the group
  }
  // interval bounds this lane watches in the cull tests: q = lane, lane + 32
  constexpr int QL = (K + 31) / 32;
  double gl[QL], gh[QL], lo_[QL], hi_[QL];
  bool cull = false;
#pragma unroll
  for (int u = 0; u < QL; ++u) {
    const int q = lane + 32 * u;
    const bool on = live && q < K;
    gl[u] = on ? gmin[g * K + q] : 0.0;
    gh[u] = on ? gmax[g * K + q] : 0.0;
    lo_[u] = q < K ? bd.lo[q] : -INFINITY;
    hi_[u] = q < K ? bd.hi[q] : INFINITY;
    if (on) cull |= (__dadd_rn(tmin[tile * K + q], gl[u]) > hi_[u]) | (__dadd_rn(tmax[tile * K + q], gh[u]) < lo_[u]);
  }
  live = live && !__any_sync(0xffffffffu, cull);  // else no pair of (tile, group) can pass
  if (!__syncthreads_or(live)) return;
  for (int e = tid; e < rows * K; e += kPairThreads) {
    const int ii = e / K, q = e - ii * K;
    s_a1[ii][q] = a1c[(i0 + ii) * K + q];
  }
  if (tid < rows) {
    s_ok[tid] = src_ok[i0 + tid];
    s_orig[tid] = perm_src[i0 + tid];
    if (REG)
      for (int w = 0; w < kMaxRegionWords; ++w) s_sm[tid][w] = w < rm.RW ? rm.smask[(i0 + tid) * rm.RW + w] : 0ull;
  }
  __syncthreads();
  if (!live) return;
  const long long j = g * kTile + lane;
  double a2[K];
  bool jok = j < V;
  int orig_j = 0;
  if (jok) {
#pragma unroll
    for (int q = 0; q < K; ++q) a2[q] = a2t[(long long)q * V + j];
    jok = dst_ok[j] != 0;
    orig_j = perm[j];
    if (REG) {
#pragma unroll
      for (int w = 0; w < kMaxRegionWords; ++w) dm[w] = w < rm.RW ? rm.dmask[j * rm.RW + w] : 0ull;
    }
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) a2[q] = 0.0;
  }
  for (int ii = 0; ii < rows; ++ii) {
    if (!s_ok[ii]) continue;
    bool jreg = true;
    if (REG) {
      bool share = false;
      jreg = false;
#pragma unroll
      for (int w = 0; w < kMaxRegionWords; ++w) {
        share |= (s_sm[ii][w] & gor[w]) != 0;
        jreg |= (s_sm[ii][w] & dm[w]) != 0;
      }
      if (!share) continue;  // uniform: the source shares no region with the group
    }
    bool c2 = false;
#pragma unroll
    for (int u = 0; u < QL; ++u) {
      const int q = lane + 32 * u;
      if (q < K) {
        const double a = s_a1[ii][q];
        c2 |= (__dadd_rn(a, gl[u]) > hi_[u]) | (__dadd_rn(a, gh[u]) < lo_[u]);
      }
    }
    if (__any_sync(0xffffffffu, c2)) continue;
    bool ok = jok && jreg && (s_orig[ii] != orig_j);  // by original index
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if ((q & 1) == 0 && q > 0) {
        if (!__any_sync(0xffffffffu, ok)) break;
      }
      const double s = __dadd_rn(s_a1[ii][q], a2[q]);
      ok = ok && (s <= bd.hi[q]) && (s >= bd.lo[q]);
    }
    const unsigned mk = __ballot_sync(0xffffffffu, ok);
    if (mk) {
      const long long row = (long long)s_orig[ii] - r0;
      if (ok) atomicOr(bits + row * W + (orig_j >> 5), 1u << (orig_j & 31));
      if (lane == 0) atomicAdd(rowcnt + row, (unsigned long long)__popc(mk));
    }
  }
}

// ---------------------------------------------------------------- compacted (tile, group) pairs
// The same exact culls as k_pair_tiles' prologue, one thread per (source tile, destination
// group), the survivors appended to a list.  A 2-D grid over every (tile, group) spends most
// of its blocks on pairs that cull (cfg5 at 100k nodes: 1.2 M blocks), so the tests below run
// over the list only.
__global__ void k_tile_group_cull(Bounds bd, const double* __restrict__ tmin, const double* __restrict__ tmax,
                                  const double* __restrict__ gmin, const double* __restrict__ gmax, long long ng,
                                  int K, RegionMasks rm, int reg, unsigned long long* __restrict__ list,
                                  unsigned long long* __restrict__ n_list) {
  BZG_PDL_ENTRY();
  const long long tile = blockIdx.y;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool live = g < ng;
  if (reg && live) {
    bool share = false;
    for (int w = 0; w < rm.RW; ++w) share |= (rm.group_or[g * rm.RW + w] & rm.tile_or[tile * rm.RW + w]) != 0;
    live = share;
  }
  if (live) {
    bool cull = false;
    for (int q = 0; q < K && !cull; ++q)
      cull = (__dadd_rn(tmin[tile * K + q], gmin[g * K + q]) > bd.hi[q]) |
             (__dadd_rn(tmax[tile * K + q], gmax[g * K + q]) < bd.lo[q]);
    live = !cull;
  }
  const unsigned want = __ballot_sync(0xffffffffu, live);
  if (!want) return;
  const int lane = threadIdx.x & 31, leader = __ffs(want) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(n_list, (unsigned long long)__popc(want));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (live) list[base + __popc(want & ((1u << lane) - 1u))] = ((unsigned long long)tile << 32) | (unsigned long long)g;
}

template <int K, bool REG>
size_t pair_list_smem() {
  constexpr int NW = kPairThreads / 32;
  return sizeof(double) * NW * kTile * K + (REG ? sizeof(unsigned long long) * NW * kTile * kMaxRegionWords : 0) +
         sizeof(int) * NW * kTile + NW * kTile;
}

// One warp per surviving (tile, group): the tile's 32 sources against the group's 32
// destinations, exactly k_pair_tiles' per-source cull and pair test, with the tile staged in
// the warp's own shared-memory slice.  Persistent grid over the device-side list length.
template <int K, bool REG>
__global__ void __launch_bounds__(kPairThreads, 3) k_pair_list(
    Bounds bd, const double* __restrict__ a1c, const double* __restrict__ a2t, const uint8_t* __restrict__ src_ok,
    const uint8_t* __restrict__ dst_ok, const int* __restrict__ perm, const double* __restrict__ gmin,
    const double* __restrict__ gmax, long long V, long long r0, long long W, uint32_t* __restrict__ bits,
    unsigned long long* __restrict__ rowcnt, RegionMasks rm, const unsigned long long* __restrict__ list,
    const unsigned long long* __restrict__ n_list, const int* __restrict__ perm_src, long long V_src) {
  BZG_PDL_ENTRY();
  constexpr int NW = kPairThreads / 32, QL = (K + 31) / 32;
  // dynamic shared memory (pair_list_smem): per warp a1 tile, region masks, original ids, flags
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto* s_a1_all = reinterpret_cast<double (*)[kTile][K]>(smem_raw);
  auto* s_sm_all = reinterpret_cast<unsigned long long (*)[kTile][kMaxRegionWords]>(smem_raw +
                                                                                    sizeof(double) * NW * kTile * K);
  int* s_orig_all = reinterpret_cast<int*>(smem_raw + sizeof(double) * NW * kTile * K +
                                           (REG ? sizeof(unsigned long long) * NW * kTile * kMaxRegionWords : 0));
  uint8_t* s_ok_all = reinterpret_cast<uint8_t*>(s_orig_all + NW * kTile);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double (*s_a1)[K] = s_a1_all[warp];
  uint8_t* s_ok = s_ok_all + warp * kTile;
  int* s_orig = s_orig_all + warp * kTile;
  const long long n = (long long)*n_list;
  for (long long e = (long long)blockIdx.x * NW + warp; e < n; e += (long long)gridDim.x * NW) {
    const unsigned long long it = list[e];
    const long long tile = (long long)(it >> 32), g = (long long)(it & 0xffffffffull);
    const long long i0 = tile * kTile;
    const int rows = (int)min((long long)kTile, V_src - i0);
    __syncwarp();
    for (int t = lane; t < rows * K; t += 32) {
      const int ii = t / K, q = t - ii * K;
      s_a1[ii][q] = a1c[(i0 + ii) * K + q];
    }
    if (lane < rows) {
      s_ok[lane] = src_ok[i0 + lane];
      s_orig[lane] = perm_src[i0 + lane];
      if (REG)
        for (int w = 0; w < kMaxRegionWords; ++w)
          s_sm_all[warp][lane][w] = w < rm.RW ? rm.smask[(i0 + lane) * rm.RW + w] : 0ull;
    }
    __syncwarp();
    unsigned long long gor[kMaxRegionWords] = {0, 0, 0, 0}, dm[kMaxRegionWords] = {0, 0, 0, 0};
    if (REG) {
#pragma unroll
      for (int w = 0; w < kMaxRegionWords; ++w) gor[w] = w < rm.RW ? rm.group_or[g * rm.RW + w] : 0ull;
    }
    double gl[QL], gh[QL], lo_[QL], hi_[QL];
#pragma unroll
    for (int u = 0; u < QL; ++u) {
      const int q = lane + 32 * u;
      const bool on = q < K;
      gl[u] = on ? gmin[g * K + q] : 0.0;
      gh[u] = on ? gmax[g * K + q] : 0.0;
      lo_[u] = on ? bd.lo[q] : -INFINITY;
      hi_[u] = on ? bd.hi[q] : INFINITY;
    }
    const long long j = g * kTile + lane;
    double a2[K];
    bool jok = j < V;
    int orig_j = 0;
    if (jok) {
#pragma unroll
      for (int q = 0; q < K; ++q) a2[q] = a2t[(long long)q * V + j];
      jok = dst_ok[j] != 0;
      orig_j = perm[j];
      if (REG) {
#pragma unroll
        for (int w = 0; w < kMaxRegionWords; ++w) dm[w] = w < rm.RW ? rm.dmask[j * rm.RW + w] : 0ull;
      }
    } else {
#pragma unroll
      for (int q = 0; q < K; ++q) a2[q] = 0.0;
    }
    for (int ii = 0; ii < rows; ++ii) {
      if (!s_ok[ii]) continue;
      bool jreg = true;
      if (REG) {
        bool share = false;
        jreg = false;
#pragma unroll
        for (int w = 0; w < kMaxRegionWords; ++w) {
          share |= (s_sm_all[warp][ii][w] & gor[w]) != 0;
          jreg |= (s_sm_all[warp][ii][w] & dm[w]) != 0;
        }
        if (!share) continue;  // uniform: the source shares no region with the group
      }
      bool c2 = false;
#pragma unroll
      for (int u = 0; u < QL; ++u) {
        const int q = lane + 32 * u;
        if (q < K) {
          const double a = s_a1[ii][q];
          c2 |= (__dadd_rn(a, gl[u]) > hi_[u]) | (__dadd_rn(a, gh[u]) < lo_[u]);
        }
      }
      if (__any_sync(0xffffffffu, c2)) continue;
      bool ok = jok && jreg && (s_orig[ii] != orig_j);  // by original index
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if ((q & 1) == 0 && q > 0) {
          if (!__any_sync(0xffffffffu, ok)) break;
        }
        const double s = __dadd_rn(s_a1[ii][q], a2[q]);
        ok = ok && (s <= bd.hi[q]) && (s >= bd.lo[q]);
      }
      const unsigned mk = __ballot_sync(0xffffffffu, ok);
      if (mk) {
        const long long row = (long long)s_orig[ii] - r0;
        if (ok) atomicOr(bits + row * W + (orig_j >> 5), 1u << (orig_j & 31));
        if (lane == 0) atomicAdd(rowcnt + row, (unsigned long long)__popc(mk));
      }
    }
  }
}

// ---------------------------------------------------------------- k_nearest prefilter
// graph.py:162-170: d2 = ((pos_i - pos_j)**2).sum(axis=2) -- squares, then a left fold over the
// m position coordinates, no FMA -- with an infinite diagonal, k = min(k_nearest, V-1), and
// edge i->j allowed iff j is among the k smallest of row i.  Non-negative doubles order like
// their bit patterns, so the k-th smallest key of a row is found by an MSB-first radix
// select (8-bit digits, warp-aggregated shared histograms).  Keys equal to it are kept
// lowest index first (argpartition's tie order is implementation-defined).  One block per
// source row masks the row's pair bits and recounts the row.
constexpr int kKnnThreads = 256;

__device__ __forceinline__ unsigned long long knn_key(const double* __restrict__ Vx, int n, int m,
                                                      const double (&pi)[3], long long j) {
  double s = 0.0;
  for (int k = 0; k < m; ++k) {
    const double d = __dsub_rn(pi[k], Vx[j * n + k]);
    const double sq = __dmul_rn(d, d);
    s = k == 0 ? sq : __dadd_rn(s, sq);
  }
  return (unsigned long long)__double_as_longlong(s);
}

__global__ void __launch_bounds__(kKnnThreads) k_knn_rows(const double* __restrict__ Vx, long long V, int n, int m,
                                                          long long k, long long r0, long long W,
                                                          uint32_t* __restrict__ bits,
                                                          unsigned long long* __restrict__ rowcnt) {
  BZG_PDL_ENTRY();
  typedef cub::BlockScan<unsigned long long, kKnnThreads> BS;
  typedef cub::BlockReduce<unsigned long long, kKnnThreads> BR;
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_krem, s_last;
  __shared__ union { typename BS::TempStorage scan; typename BR::TempStorage red; } tmp;
  const long long row = blockIdx.x, i = r0 + row;
  const int tid = threadIdx.x;
  uint32_t* wrow = bits + row * W;
  if (rowcnt[row] == 0) return;  // no pair edge to filter (uniform across the block)
  if (k == 0) {
    for (long long w = tid; w < W; w += kKnnThreads) wrow[w] = 0u;
    if (tid == 0) rowcnt[row] = 0;
    return;
  }
  double pi[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < m; ++q) pi[q] = Vx[i * n + q];
  unsigned long long prefix = 0;
  long long krem = k;  // rank (1-based) of the wanted key among keys matching prefix
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kKnnThreads) hist[b] = 0u;
    __syncthreads();
    const unsigned long long hi_mask = shift == 56 ? 0ull : (~0ull << (shift + 8));
    for (long long j0 = 0; j0 < V; j0 += kKnnThreads) {
      const long long j = j0 + tid;
      int digit = -1;
      if (j < V && j != i) {
        const unsigned long long key = knn_key(Vx, n, m, pi, j);
        if ((key & hi_mask) == prefix) digit = (int)((key >> shift) & 255ull);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, digit);
      if (digit >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[digit], (unsigned)__popc(peers));
    }
    __syncthreads();
    if (tid == 0) {
      long long cum = 0;
      for (int dgt = 0; dgt < 256; ++dgt) {
        if (cum + hist[dgt] >= krem) {
          s_prefix = prefix | ((unsigned long long)dgt << shift);
          s_krem = krem - cum;
          break;
        }
        cum += hist[dgt];
      }
    }
    __syncthreads();
    prefix = s_prefix;
    krem = s_krem;
  }
  // prefix = the k-th smallest key t; keep the first krem indices (ascending) whose key is t
  const unsigned long long t = prefix;
  const long long chunk = (V + kKnnThreads - 1) / kKnnThreads;
  const long long j0 = tid * chunk, j1 = j0 + chunk < V ? j0 + chunk : V;
  unsigned long long ties = 0;
  for (long long j = j0; j < j1; ++j) ties += (j != i && knn_key(Vx, n, m, pi, j) == t);
  unsigned long long before = 0;
  BS(tmp.scan).ExclusiveSum(ties, before);
  if ((long long)before < krem && (long long)(before + ties) >= krem) {
    long long need = krem - (long long)before;
    for (long long j = j0; j < j1; ++j)
      if (j != i && knn_key(Vx, n, m, pi, j) == t && --need == 0) { s_last = j; break; }
  }
  __syncthreads();
  const long long last = s_last;
  unsigned long long total = 0;
  for (long long w = tid; w < W; w += kKnnThreads) {
    uint32_t word = wrow[w];
    if (!word) continue;
    uint32_t allow = 0u;
    for (uint32_t rest = word; rest; rest &= rest - 1) {
      const int b = __ffs(rest) - 1;
      const long long j = w * 32 + b;
      const unsigned long long key = knn_key(Vx, n, m, pi, j);
      if (key < t || (key == t && j <= last)) allow |= 1u << b;
    }
    word &= allow;
    wrow[w] = word;
    total += __popc(word);
  }
  __syncthreads();
  const unsigned long long sum = BR(tmp.red).Sum(total);
  if (tid == 0) rowcnt[row] = sum;
}

// ---------------------------------------------------------------- compaction
struct DParams {
  double D[64];
};

// One warp per source row: ordered expansion of the row's bit words into
// (src, dst) in ascending dst (np.nonzero order, graph.py:187-190) and the edge cost
// (graph.py:192-197) computed from the two endpoint states.
constexpr int kExpandThreads = 256;

template <int G, int M>
__global__ void __launch_bounds__(kExpandThreads) k_expand(DParams dp, const double* __restrict__ Vx, long long r0,
                                                           long long r1, long long W,
                         const uint32_t* __restrict__ bits, const long long* __restrict__ rptr,
                         int* __restrict__ src, int* __restrict__ dst, double* __restrict__ cost, long long cap) {
  BZG_PDL_ENTRY();
  // The set bits of 32 words are first listed in ascending (word, bit) order in the warp's
  // shared slice, then the lanes take one edge each, so a word with many edges does not
  // serialise its lane while the others idle.  cap: the arrays' capacity (a captured plan's,
  // whose edge count is not known at launch; edges past it are dropped and the plan reruns).
  constexpr int N = G * M;
  __shared__ int s_j[kExpandThreads / 32][32 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long i = r0 + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (i >= r1) return;
  long long base = rptr[i - r0];
  const long long end = min(rptr[i - r0 + 1], cap);
  if (base >= end) return;
  double xi[N];
#pragma unroll
  for (int k = 0; k < N; ++k) xi[k] = Vx[i * N + k];
  const uint32_t* row = bits + (i - r0) * W;
  int* lst = s_j[warp];
  for (long long w0 = 0; w0 < W && base < end; w0 += 32) {
    if ((w0 & 127) == 0) {  // skip 128 empty words at a time (sparse rows of large graphs)
      uint32_t any = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const long long wq = w0 + 32 * q + lane;
        any |= wq < W ? row[wq] : 0u;
      }
      if (!__any_sync(0xffffffffu, any != 0)) {
        w0 += 96;
        continue;
      }
    }
    const long long w = w0 + lane;
    uint32_t word = w < W ? row[w] : 0u;
    const int c = __popc(word);
    const int incl = warp_incl_scan(c);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    for (int k = incl - c; word; ++k) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      lst[k] = (int)(w * 32 + b);
    }
    __syncwarp();
    for (int t = lane; t < total && base + t < end; t += 32) {
      const long long jv = lst[t];
      double xj[N];
#pragma unroll
      for (int k = 0; k < N; ++k) xj[k] = Vx[jv * N + k];
      double P[M][2 * G];
      control_points<G, M>(xi, xj, dp.D, P);
      src[base + t] = (int)i;
      dst[base + t] = (int)jv;
      cost[base + t] = polygon_length<G, M>(P);
    }
    __syncwarp();
    base += total;
  }
}

template <int G, int M>
__global__ void k_points(DParams dp, const double* __restrict__ Vx, long long E, const int* __restrict__ src,
                         const int* __restrict__ dst, double* __restrict__ out) {
  BZG_PDL_ENTRY();
  constexpr int N = G * M;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  double xi[N], xj[N];
  const long long a = src[e], b = dst[e];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    xi[k] = Vx[a * N + k];
    xj[k] = Vx[b * N + k];
  }
  double P[M][2 * G];
  control_points<G, M>(xi, xj, dp.D, P);
#pragma unroll
  for (int k = 0; k < M; ++k)
#pragma unroll
    for (int j = 0; j < 2 * G; ++j) out[e * M * 2 * G + k * 2 * G + j] = P[k][j];
}

// cap: the CSR arrays' capacity (a captured plan's; offsets past it are clipped so the search
// never reads beyond the arrays of a build whose edges overflowed -- the plan reruns it)
__global__ void k_row_ptr_global(const long long* __restrict__ local, long long V, long long r0, long long r1,
                                 long long* __restrict__ out, long long cap) {
  BZG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > V) return;
  const long long E = local[r1 - r0];
  const long long v = i <= r0 ? 0 : (i >= r1 ? E : local[i - r0]);
  out[i] = v < cap ? v : cap;
}

// row_ptr[i] = lower_bound(src, i) over a source-sorted edge list (gathered row blocks)
__global__ void k_row_ptr_from_src(const int* __restrict__ src, long long E, long long V, long long* __restrict__ out) {
  BZG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > V) return;
  long long lo = 0, hi = E;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (src[mid] < i) lo = mid + 1; else hi = mid;
  }
  out[i] = lo;
}

// check_edges (reachability.py:139-142): X1 F1' + X2 F2' <= G + eps, separable form.
__global__ void k_check_edges(const double* __restrict__ F, const double* __restrict__ thresh, int n, int nF,
                              long long k, const double* __restrict__ X1, const double* __restrict__ X2,
                              uint8_t* __restrict__ out) {
  BZG_PDL_ENTRY();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= k) return;
  int ok = 1;
  for (int r = 0; r < nF; ++r) {
    const double* f = F + (size_t)r * 2 * n;
    const double s = __dadd_rn(fma_chain(X1 + t * n, f, n), fma_chain(X2 + t * n, f + n, n));
    ok &= s <= thresh[r];
  }
  out[t] = (uint8_t)ok;
}

template <typename F>
void dispatch_gm(int G, int M, F&& f) {
#define BZG_GM(g, m) \
  if (G == g && M == m) { f(std::integral_constant<int, g>{}, std::integral_constant<int, m>{}); return; }
  BZG_GM(1, 1) BZG_GM(1, 2) BZG_GM(1, 3) BZG_GM(2, 1) BZG_GM(2, 2) BZG_GM(2, 3)
  BZG_GM(3, 1) BZG_GM(3, 2) BZG_GM(3, 3) BZG_GM(4, 1) BZG_GM(4, 2) BZG_GM(4, 3)
#undef BZG_GM
  throw Error(BZG_EUNSUPPORTED, "device path supports gamma in 1..4 and m in 1..3");
}

void exclusive_scan_ll(Ctx* c, const unsigned long long* in, long long* out, long long count) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, c->stream);
  c->ws[WS_SCRATCH].alloc(bytes, c->stream);
  ScopedLibLaunch l(c, "cub_scan_rows", 2);
  BZG_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(c->ws[WS_SCRATCH].ptr, bytes, in, out, count, c->stream));
}

void exclusive_scan_i(Ctx* c, const int* in, int* out, long long count) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, c->stream);
  c->ws[WS_SCRATCH].alloc(bytes, c->stream);
  ScopedLibLaunch l(c, "cub_scan_sample", 2);
  BZG_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(c->ws[WS_SCRATCH].ptr, bytes, in, out, count, c->stream));
}

}  // namespace

// ------------------------------------------------------------------ host side
void sample_states(Ctx* c, const bzg_build_desc* d, double* d_vertices, bool single_round,
                   const unsigned long long* pcg_dev) {
  const int n = d->m * d->gamma;
  BZG_REQUIRE(n <= kMaxN, BZG_EUNSUPPORTED, "state dimension too large for the device sampler");
  BZG_REQUIRE(d->xd_rows >= 1 && d->xd_rows <= kMaxRows, BZG_EUNSUPPORTED, "state polytope row count unsupported");
  SampleParams sp{};
  sp.n = n;
  sp.rows = d->xd_rows;
  for (int k = 0; k < n; ++k) {
    sp.lo[k] = d->sample_lo[k];
    sp.range[k] = d->sample_hi[k] - d->sample_lo[k];  // np.subtract(high, low)
  }
  for (int r = 0; r < d->xd_rows; ++r) {
    for (int k = 0; k < n; ++k) sp.A[r * n + k] = d->xd_A[r * n + k];
    sp.b_eps[r] = d->xd_b[r] + d->eps_geo;
  }
  long long need = d->N, row0 = 0, got = 0;
  // acceptance estimate: the last build's on this context (single_round: its one round is sized
  // from it and checked later, at build_pairs' read-back, instead of synchronising here)
  double est = single_round ? c->sample_est : 1.0;
  DevBuf &cand = c->ws[WS_CAND], &flag = c->ws[WS_FLAG], &pos = c->ws[WS_POS];
  int* h = static_cast<int*>(c->host_scratch(2 * sizeof(int)));
  for (int round = 0; need > 0; ++round) {
    BZG_REQUIRE(round < 10000, BZG_EINVAL, "sampler made no progress: state polytope misses the sampling box");
    long long count = (long long)std::ceil((double)need / std::max(est, 1e-3) * (single_round ? 1.10 : 1.05)) + 256;
    count = std::min<long long>(count, 1ll << 26);
    cand.alloc(count * n * sizeof(double), c->stream);
    flag.alloc((count + 1) * sizeof(int), c->stream);
    pos.alloc((count + 1) * sizeof(int), c->stream);
    launch(c, "k_sample_candidates", k_sample_candidates, dim3(div_up(count, 256)), dim3(256), 0, sp,
           (unsigned long long)d->pcg_state_hi, (unsigned long long)d->pcg_state_lo,
           (unsigned long long)d->pcg_inc_hi, (unsigned long long)d->pcg_inc_lo, row0, count, cand.as<double>(),
           flag.as<int>(), pcg_dev);
    BZG_CHECK_CUDA(cudaMemsetAsync(flag.as<int>() + count, 0, sizeof(int), c->stream));
    exclusive_scan_i(c, flag.as<int>(), pos.as<int>(), count + 1);
    launch(c, "k_sample_scatter", k_sample_scatter, dim3(div_up(count, 256)), dim3(256), 0, cand.as<double>(),
           flag.as<int>(), pos.as<int>(), count, n, need, d_vertices + got * n);
    if (single_round) {  // accepted count checked by build_pairs (Ctx::sample_check)
      c->sample_check = pos.as<int>() + count;
      c->sample_need = need;
      c->sample_count = count;
      return;
    }
    BZG_CHECK_CUDA(cudaMemcpyAsync(h, pos.as<int>() + count, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
    const long long acc = h[0];
    // Rows past the N-th acceptance were drawn but are never used, exactly like the
    // reference whose rounds only ever draw `needed` rows (graph.py:150-156): the kept
    // set is the first N accepted rows of the stream either way.
    const long long take = std::min(acc, need);
    got += take;
    need -= take;
    row0 += count;
    est = std::max(1e-3, (double)acc / (double)count);
  }
  c->sample_est = est;
}

void sample_regions(Ctx* c, int n, int R, const int64_t* N, const uint64_t* pcg, const double* lo, const double* hi,
                    const int32_t* row_off, const double* A, const double* b, double eps_geo, double* d_out,
                    double* est_out) {
  BZG_REQUIRE(n >= 1 && n <= kMaxN, BZG_EUNSUPPORTED, "state dimension too large for the device sampler");
  BZG_REQUIRE(R >= 1, BZG_EINVAL, "need at least one region");
  std::vector<double> range((size_t)R * n), beps(row_off[R]);
  for (size_t k = 0; k < range.size(); ++k) range[k] = hi[k] - lo[k];  // np.subtract(high, low)
  for (int q = 0; q < row_off[R]; ++q) beps[q] = b[q] + eps_geo;
  c->arena->reset();
  TmpBuf d_pcg(c), d_lo(c), d_rng(c), d_off(c), d_A(c), d_b(c), d_coff(c), d_row0(c), d_dest(c), d_need(c), d_acc(c);
  DevBuf &cand = c->ws[WS_CAND], &flag = c->ws[WS_FLAG], &pos = c->ws[WS_POS];
  auto up = [&](TmpBuf& buf, const void* src, size_t bytes) {
    buf.alloc(std::max<size_t>(bytes, 8), c->stream);
    if (bytes) BZG_CHECK_CUDA(cudaMemcpyAsync(buf.ptr, src, bytes, cudaMemcpyHostToDevice, c->stream));
  };
  up(d_pcg, pcg, (size_t)R * 4 * sizeof(uint64_t));
  up(d_lo, lo, (size_t)R * n * sizeof(double));
  up(d_rng, range.data(), (size_t)R * n * sizeof(double));
  up(d_off, row_off, (size_t)(R + 1) * sizeof(int32_t));
  up(d_A, A, (size_t)row_off[R] * n * sizeof(double));
  up(d_b, beps.data(), beps.size() * sizeof(double));
  std::vector<long long> need(N, N + R), got(R, 0), row0(R, 0), base(R + 1, 0), coff(R + 1), dest(R);
  std::vector<double> est(R, 1.0);
  for (int r = 0; r < R; ++r) base[r + 1] = base[r] + N[r];
  d_coff.alloc((R + 1) * sizeof(long long), c->stream);
  d_row0.alloc(R * sizeof(long long), c->stream);
  d_dest.alloc(R * sizeof(long long), c->stream);
  d_need.alloc(R * sizeof(long long), c->stream);
  d_acc.alloc(R * sizeof(long long), c->stream);
  long long* hacc = static_cast<long long*>(c->host_scratch(R * sizeof(long long)));
  for (int round = 0;; ++round) {
    bool any = false;
    coff[0] = 0;
    for (int r = 0; r < R; ++r) {
      long long cnt = 0;
      if (need[r] > 0) {
        any = true;
        cnt = std::min<long long>((long long)std::ceil((double)need[r] / std::max(est[r], 1e-3) * 1.05) + 64, 1ll << 24);
      }
      coff[r + 1] = coff[r] + cnt;
      dest[r] = base[r] + got[r];
    }
    if (!any) break;
    BZG_REQUIRE(round < 10000, BZG_EINVAL, "sampler made no progress: a region's state set misses its sampling box");
    const long long total = coff[R];
    BZG_REQUIRE(total < (1ll << 30), BZG_EUNSUPPORTED, "too many sampler candidates in one round");
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_coff.ptr, coff.data(), (R + 1) * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_row0.ptr, row0.data(), R * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_dest.ptr, dest.data(), R * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_need.ptr, need.data(), R * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
    cand.alloc(total * n * sizeof(double), c->stream);
    flag.alloc((total + 1) * sizeof(int), c->stream);
    pos.alloc((total + 1) * sizeof(int), c->stream);
    RegionSampleDev rs{d_pcg.as<unsigned long long>(), d_lo.as<double>(), d_rng.as<double>(), d_off.as<int>(),
                       d_A.as<double>(), d_b.as<double>(), d_coff.as<long long>(), d_row0.as<long long>(), n, R};
    launch(c, "k_sample_regions", k_sample_regions, dim3(div_up(total, 256)), dim3(256), 0, rs, total,
           cand.as<double>(), flag.as<int>());
    BZG_CHECK_CUDA(cudaMemsetAsync(flag.as<int>() + total, 0, sizeof(int), c->stream));
    exclusive_scan_i(c, flag.as<int>(), pos.as<int>(), total + 1);
    launch(c, "k_scatter_regions", k_scatter_regions, dim3(div_up(total, 256)), dim3(256), 0, cand.as<double>(),
           flag.as<int>(), pos.as<int>(), d_coff.as<long long>(), R, total, n, d_dest.as<long long>(),
           d_need.as<long long>(), d_out);
    launch(c, "k_region_acc", k_region_acc, dim3(div_up(R, 256)), dim3(256), 0, pos.as<int>(), d_coff.as<long long>(),
           R, d_acc.as<long long>());
    BZG_CHECK_CUDA(cudaMemcpyAsync(hacc, d_acc.ptr, R * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
    for (int r = 0; r < R; ++r) {
      if (need[r] <= 0) continue;
      const long long cnt = coff[r + 1] - coff[r];
      const long long take = std::min(hacc[r], need[r]);  // the first need[r] acceptances of the stream
      got[r] += take;
      need[r] -= take;
      row0[r] += cnt;
      est[r] = std::max(1e-3, (double)hacc[r] / (double)cnt);
    }
  }
  if (est_out)
    for (int r = 0; r < R; ++r) est_out[r] = est[r];
}

// ---- keep-in sampling for a captured plan: ONE round whose per-region candidate counts come
// from acceptance estimates (1.3x margin), every array but the PCG words uploaded once; the
// per-region acceptance counts reach h_acc (pinned) for the plan's check after the launch.
struct RegionSamplePlan {
  int n = 0, R = 0;
  long long total = 0;
  DevBuf lo, range, row_off, A, b_eps, cand_off, row0, dest, need, acc;
};

RegionSamplePlan* region_sample_plan_create(Ctx* c, int n, int R, const int64_t* N, const double* lo,
                                            const double* hi, const int32_t* row_off, const double* A,
                                            const double* b, double eps_geo, const double* est) {
  RegionSamplePlan* s = new RegionSamplePlan();
  s->n = n;
  s->R = R;
  std::vector<double> range((size_t)R * n), beps(row_off[R]);
  for (size_t k = 0; k < range.size(); ++k) range[k] = hi[k] - lo[k];  // np.subtract(high, low)
  for (int q = 0; q < row_off[R]; ++q) beps[q] = b[q] + eps_geo;
  std::vector<long long> coff(R + 1, 0), row0(R, 0), dest(R, 0), need(R);
  long long base = 0;
  for (int r = 0; r < R; ++r) {
    const long long cnt = N[r] > 0 ? std::min<long long>(
        (long long)std::ceil((double)N[r] / std::max(est[r], 1e-3) * 1.3) + 64, 1ll << 24) : 0;
    coff[r + 1] = coff[r] + cnt;
    dest[r] = base;
    need[r] = N[r];
    base += N[r];
  }
  s->total = coff[R];
  auto up = [&](DevBuf& buf, const void* src, size_t bytes) {
    buf.alloc(std::max<size_t>(bytes, 8), c->stream);
    if (bytes) BZG_CHECK_CUDA(cudaMemcpyAsync(buf.ptr, src, bytes, cudaMemcpyHostToDevice, c->stream));
  };
  up(s->lo, lo, (size_t)R * n * sizeof(double));
  up(s->range, range.data(), range.size() * sizeof(double));
  up(s->row_off, row_off, (size_t)(R + 1) * sizeof(int32_t));
  up(s->A, A, (size_t)row_off[R] * n * sizeof(double));
  up(s->b_eps, beps.data(), beps.size() * sizeof(double));
  up(s->cand_off, coff.data(), coff.size() * sizeof(long long));
  up(s->row0, row0.data(), row0.size() * sizeof(long long));
  up(s->dest, dest.data(), dest.size() * sizeof(long long));
  up(s->need, need.data(), need.size() * sizeof(long long));
  s->acc.alloc(R * sizeof(long long), c->stream);
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));  // (host vectors leave scope)
  return s;
}

void region_sample_plan_enqueue(Ctx* c, RegionSamplePlan* s, const unsigned long long* d_pcg, double* d_out,
                                long long* h_acc) {
  DevBuf &cand = c->ws[WS_CAND], &flag = c->ws[WS_FLAG], &pos = c->ws[WS_POS];
  const long long total = s->total;
  cand.alloc(total * s->n * sizeof(double), c->stream);
  flag.alloc((total + 1) * sizeof(int), c->stream);
  pos.alloc((total + 1) * sizeof(int), c->stream);
  RegionSampleDev rs{d_pcg, s->lo.as<double>(), s->range.as<double>(), s->row_off.as<int>(), s->A.as<double>(),
                     s->b_eps.as<double>(), s->cand_off.as<long long>(), s->row0.as<long long>(), s->n, s->R};
  launch(c, "k_sample_regions", k_sample_regions, dim3(div_up(total, 256)), dim3(256), 0, rs, total,
         cand.as<double>(), flag.as<int>());
  BZG_CHECK_CUDA(cudaMemsetAsync(flag.as<int>() + total, 0, sizeof(int), c->stream));
  exclusive_scan_i(c, flag.as<int>(), pos.as<int>(), total + 1);
  launch(c, "k_scatter_regions", k_scatter_regions, dim3(div_up(total, 256)), dim3(256), 0, cand.as<double>(),
         flag.as<int>(), pos.as<int>(), s->cand_off.as<long long>(), s->R, total, s->n, s->dest.as<long long>(),
         s->need.as<long long>(), d_out);
  launch(c, "k_region_acc", k_region_acc, dim3(div_up(s->R, 256)), dim3(256), 0, pos.as<int>(),
         s->cand_off.as<long long>(), s->R, s->acc.as<long long>());
  BZG_CHECK_CUDA(cudaMemcpyAsync(h_acc, s->acc.ptr, s->R * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
}

void region_sample_plan_destroy(RegionSamplePlan* s) { delete s; }

// the keep-in rows of the pair test (one-sided source / destination rows per region, with the
// eps-shifted thresholds), prepared on the host
struct RegionRowsHost {
  std::vector<int> soff{0}, doff{0};
  std::vector<double> sF, sth, dF, dth;
};
RegionRowsHost region_rows_host(const bzg_build_desc* d, int n, double th_shift) {
  RegionRowsHost h;
  const int R = d->n_regions;
  for (int r = 0; r < R; ++r) {
    bool never_r = false;
    for (int q = d->region_row_off[r]; q < d->region_row_off[r + 1]; ++q) {
      const double* f = d->region_F + (size_t)q * 2 * n;
      bool z1 = true, z2 = true;
      for (int k = 0; k < n; ++k) { z1 &= f[k] == 0.0; z2 &= f[n + k] == 0.0; }
      double th = d->region_G[q] + d->eps_geo;  // check_edges: G + eps (reachability.py:142)
      if (th_shift != 0.0) th = th + th_shift;
      BZG_REQUIRE(z1 || z2, BZG_EUNSUPPORTED, "a keep-in region row couples both endpoints");
      if (z1 && z2) { never_r |= !(0.0 <= th); continue; }
      if (z2) { h.sF.insert(h.sF.end(), f, f + n); h.sth.push_back(th); }
      else { h.dF.insert(h.dF.end(), f + n, f + 2 * n); h.dth.push_back(th); }
    }
    if (never_r) {  // a constant row that fails: the region admits no edge
      h.sF.insert(h.sF.end(), n, 0.0);
      h.sth.push_back(-1.0);
    }
    h.soff.push_back((int)h.sth.size());
    h.doff.push_back((int)h.dth.size());
  }
  return h;
}

// a captured plan's keep-in rows and region boxes, uploaded once
struct RegionRowsCache {
  DevBuf soff, sF, sth, doff, dF, dth, blo, bhi;
  int R = 0;
  bool boxes = false;
};

RegionRowsCache* region_rows_cache_create(Ctx* c, const bzg_build_desc* d) {
  const int n = d->m * d->gamma, m = d->m, R = d->n_regions;
  BZG_REQUIRE(R <= 64 * kMaxRegionWords, BZG_EUNSUPPORTED, "at most 256 keep-in regions");
  BZG_REQUIRE(d->region_row_off && d->region_F && d->region_G, BZG_EINVAL, "region rows missing");
  const RegionRowsHost h = region_rows_host(d, n, 0.0);
  RegionRowsCache* rc = new RegionRowsCache();
  rc->R = R;
  auto up = [&](DevBuf& buf, const void* src, size_t bytes) {
    buf.alloc(std::max<size_t>(bytes, 8), c->stream);
    if (bytes) BZG_CHECK_CUDA(cudaMemcpyAsync(buf.ptr, src, bytes, cudaMemcpyHostToDevice, c->stream));
  };
  up(rc->soff, h.soff.data(), h.soff.size() * sizeof(int));
  up(rc->sF, h.sF.data(), h.sF.size() * sizeof(double));
  up(rc->sth, h.sth.data(), h.sth.size() * sizeof(double));
  up(rc->doff, h.doff.data(), h.doff.size() * sizeof(int));
  up(rc->dF, h.dF.data(), h.dF.size() * sizeof(double));
  up(rc->dth, h.dth.data(), h.dth.size() * sizeof(double));
  if (d->region_box_lo && d->region_box_hi) {
    rc->boxes = true;
    up(rc->blo, d->region_box_lo, (size_t)R * m * sizeof(double));
    up(rc->bhi, d->region_box_hi, (size_t)R * m * sizeof(double));
  }
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));  // (host vectors leave scope)
  return rc;
}

void region_rows_cache_destroy(RegionRowsCache* rc) { delete rc; }

bool build_pairs(Ctx* c, const bzg_build_desc* d, Graph* g, double th_shift, long long* count_only,
                 const BuildCapture* bc) {
  const int n = g->n;
  const int nF = d->n_F;
  const long long V = g->V;
  const long long r0 = g->row_begin, r1 = g->row_end;
  const long long rows = r1 - r0;

  // ---- host row plan: classify F rows (one-sided / negation-paired / unpaired)
  RowPlan rp{};
  Bounds bd{};
  rp.n = n;
  std::vector<double> th(nF);
  for (int r = 0; r < nF; ++r) th[r] = d->G[r] + d->eps_geo;  // oracle.G + EPS_GEO (graph.py:176)
  if (th_shift != 0.0)  // eps-band count (bzg_graph_eps_band): every threshold moved by +-eps
    for (int r = 0; r < nF; ++r) th[r] = th[r] + th_shift;
  auto zero = [&](int r, int off) {
    for (int k = 0; k < n; ++k)
      if (d->F[(size_t)r * 2 * n + off + k] != 0.0) return false;
    return true;
  };
  bool never = false;  // a constant row 0 <= thresh that fails kills every pair
  std::vector<int> used(nF, 0);
  std::vector<std::pair<int, std::pair<double, double>>> iv;  // row, (lo, hi)
  for (int r = 0; r < nF; ++r) {
    const bool z1 = zero(r, 0), z2 = zero(r, n);
    if (z1 && z2) { if (!(0.0 <= th[r])) never = true; used[r] = 1; continue; }
    if (z2) { BZG_REQUIRE(rp.n_src < kMaxIntervals, BZG_EUNSUPPORTED, "too many oracle rows"); rp.row_src[rp.n_src] = r; rp.th_src[rp.n_src++] = th[r]; used[r] = 1; continue; }
    if (z1) { BZG_REQUIRE(rp.n_dst < kMaxIntervals, BZG_EUNSUPPORTED, "too many oracle rows"); rp.row_dst[rp.n_dst] = r; rp.th_dst[rp.n_dst++] = th[r]; used[r] = 1; continue; }
  }
  for (int r = 0; r < nF; ++r) {
    if (used[r]) continue;
    used[r] = 1;
    double lo = -INFINITY;
    for (int s = r + 1; s < nF; ++s) {
      if (used[s]) continue;
      bool neg = true;
      for (int k = 0; k < 2 * n && neg; ++k) neg = d->F[(size_t)s * 2 * n + k] == -d->F[(size_t)r * 2 * n + k];
      if (neg) {  // lhs_s = -lhs_r exactly, so lhs_s <= th_s  <=>  lhs_r >= -th_s
        used[s] = 1;
        lo = -th[s];
        break;
      }
    }
    iv.push_back({r, {lo, th[r]}});
  }
  BZG_REQUIRE((int)iv.size() <= kMaxIntervals, BZG_EUNSUPPORTED, "too many coupled oracle rows");
  rp.K = (int)iv.size();
  static const int kSizes[] = {4, 8, 12, 16, 24, 32, 48, 64};
  int Kpad = 0;
  for (int s : kSizes)
    if (s >= rp.K) { Kpad = s; break; }
  for (int q = 0; q < Kpad; ++q) {
    if (q < rp.K) {
      rp.row_iv[q] = iv[q].first;
      bd.lo[q] = iv[q].second.first;
      bd.hi[q] = iv[q].second.second;
    } else {
      bd.lo[q] = -INFINITY;
      bd.hi[q] = INFINITY;
    }
  }

  c->arena->reset();
  TmpBuf dF(c);
  if (bc) {  // a captured plan: the oracle rows were uploaded once
    dF.ptr = const_cast<double*>(bc->dF);
    dF.bytes = (size_t)nF * 2 * n * sizeof(double);
  } else {
    dF.alloc((size_t)nF * 2 * n * sizeof(double), c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(dF.ptr, d->F, (size_t)nF * 2 * n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  DevBuf &a1c = c->ws[WS_A1C], &a2t = c->ws[WS_A2T];
  TmpBuf sok(c), dok(c);
  a1c.alloc((size_t)V * Kpad * sizeof(double), c->stream);
  a2t.alloc((size_t)V * Kpad * sizeof(double), c->stream);
  sok.alloc(V, c->stream);
  dok.alloc(V, c->stream);
  const long long W = (V + 31) / 32;
  DevBuf &bits = c->ws[WS_BITS], &rowcnt = c->ws[WS_ROWCNT], &rptr = c->ws[WS_RPTR];
  bits.alloc((size_t)std::max(rows, 1ll) * W * sizeof(uint32_t), c->stream);
  rowcnt.alloc((size_t)(rows + 1) * sizeof(unsigned long long), c->stream);
  rptr.alloc((size_t)(rows + 1) * sizeof(long long), c->stream);
  BZG_CHECK_CUDA(cudaMemsetAsync(rowcnt.ptr, 0, (rows + 1) * sizeof(unsigned long long), c->stream));
  BZG_CHECK_CUDA(cudaMemsetAsync(bits.ptr, 0, (size_t)std::max(rows, 1ll) * W * sizeof(uint32_t), c->stream));
  c->trace("pairs: alloc+memset");

  // ---- Morton order of the positions (first m coordinates); the box only steers tiling
  const int m = g->m;
  double plo[3] = {0, 0, 0}, phi[3] = {1, 1, 1};
  for (int k = 0; k < m && k < 3; ++k) {
    double lo = INFINITY, hi = -INFINITY;
    if (d->vertices) {
      for (long long i = 0; i < d->N; ++i) { lo = std::min(lo, d->vertices[i * n + k]); hi = std::max(hi, d->vertices[i * n + k]); }
    } else {
      lo = d->sample_lo[k];
      hi = d->sample_hi[k];
    }
    for (long long i = 0; i < d->n_include; ++i) {
      lo = std::min(lo, d->include[i * n + k]);
      hi = std::max(hi, d->include[i * n + k]);
    }
    plo[k] = lo;
    phi[k] = hi > lo ? hi : lo + 1.0;
  }
  const double cells = m == 1 ? 1073741823.0 : (m == 2 ? 65535.0 : 1023.0);
  TmpBuf key(c), key2(c), idx(c), perm(c);
  key.alloc(V * sizeof(unsigned), c->stream);
  key2.alloc(V * sizeof(unsigned), c->stream);
  idx.alloc(V * sizeof(int), c->stream);
  perm.alloc(V * sizeof(int), c->stream);
  launch(c, "k_morton", k_morton, dim3(div_up(V, 256)), dim3(256), 0, g->vertices.as<double>(), V, n, std::min(m, 3),
         plo[0], plo[1], plo[2], cells / (phi[0] - plo[0]), cells / (phi[1] - plo[1]), cells / (phi[2] - plo[2]),
         key.as<unsigned>(), idx.as<int>());
  {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.as<unsigned>(), key2.as<unsigned>(), idx.as<int>(),
                                    perm.as<int>(), V, 0, 32, c->stream);
    c->ws[WS_SCRATCH].alloc(bytes, c->stream);
    ScopedLibLaunch l(c, "cub_sort_morton", 4);
    BZG_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(c->ws[WS_SCRATCH].ptr, bytes, key.as<unsigned>(), key2.as<unsigned>(),
                                                   idx.as<int>(), perm.as<int>(), V, 0, 32, c->stream));
  }
  ensure_dyn_smem((const void*)k_project_sorted, (size_t)nF * 2 * n * sizeof(double));
  launch(c, "k_project_sorted", k_project_sorted, dim3(div_up(V, 128)), dim3(128), (size_t)nF * 2 * n * sizeof(double),
         rp, dF.as<double>(), nF,
         g->vertices.as<double>(), perm.as<int>(), V, Kpad, r0, r1, a1c.as<double>(), a2t.as<double>(),
         sok.as<uint8_t>(), dok.as<uint8_t>());
  const long long ng = (V + kTile - 1) / kTile;
  // ---- keep-in regions: per-vertex membership masks from the one-sided added rows
  RegionMasks rm{nullptr, nullptr, nullptr, nullptr, 0};
  TmpBuf r_soff(c), r_sF(c), r_sth(c), r_doff(c), r_dF(c), r_dth(c), smask(c), dmask(c), tor(c), gor(c);
  const int R = d->n_regions;
  BZG_REQUIRE(!bc || R == 0 || bc->rows, BZG_EINVAL, "a captured plan's keep-in rows are missing");
  if (R > 0) {
    BZG_REQUIRE(R <= 64 * kMaxRegionWords, BZG_EUNSUPPORTED, "at most 256 keep-in regions");
    BZG_REQUIRE(d->region_row_off && d->region_F && d->region_G, BZG_EINVAL, "region rows missing");
    auto up = [&](TmpBuf& buf, const void* src, size_t bytes) {
      buf.alloc(std::max<size_t>(bytes, 8), c->stream);
      if (bytes) BZG_CHECK_CUDA(cudaMemcpyAsync(buf.ptr, src, bytes, cudaMemcpyHostToDevice, c->stream));
    };
    auto view = [](TmpBuf& buf, const DevBuf& src) { buf.ptr = src.ptr; buf.bytes = src.bytes; };
    TmpBuf rblo(c), rbhi(c);
    if (bc) {  // a captured plan: uploaded once (region_rows_cache_create)
      const RegionRowsCache* rc = bc->rows;
      view(r_soff, rc->soff); view(r_sF, rc->sF); view(r_sth, rc->sth);
      view(r_doff, rc->doff); view(r_dF, rc->dF); view(r_dth, rc->dth);
      if (rc->boxes) { view(rblo, rc->blo); view(rbhi, rc->bhi); }
    } else {
      const RegionRowsHost h = region_rows_host(d, n, th_shift);
      up(r_soff, h.soff.data(), h.soff.size() * sizeof(int));
      up(r_sF, h.sF.data(), h.sF.size() * sizeof(double));
      up(r_sth, h.sth.data(), h.sth.size() * sizeof(double));
      up(r_doff, h.doff.data(), h.doff.size() * sizeof(int));
      up(r_dF, h.dF.data(), h.dF.size() * sizeof(double));
      up(r_dth, h.dth.data(), h.dth.size() * sizeof(double));
      if (d->region_box_lo && d->region_box_hi) {
        up(rblo, d->region_box_lo, (size_t)R * m * sizeof(double));
        up(rbhi, d->region_box_hi, (size_t)R * m * sizeof(double));
      }
    }
    RegionRowsDev rr{r_soff.as<int>(), r_sF.as<double>(), r_sth.as<double>(), r_doff.as<int>(), r_dF.as<double>(),
                     r_dth.as<double>(), R, (R + 63) / 64, n};
    smask.alloc(V * rr.RW * sizeof(unsigned long long), c->stream);
    dmask.alloc(V * rr.RW * sizeof(unsigned long long), c->stream);
    tor.alloc(ng * rr.RW * sizeof(unsigned long long), c->stream);
    gor.alloc(ng * rr.RW * sizeof(unsigned long long), c->stream);
    // lanes per vertex: V x G up to ~1,150 threads per SM (cfg5 k_region_masks, G = 1/4/8/16/32:
    // 10 k vertices 99/55/43/38/43 us, 100 k 93/96/111/166/247 us); BZG_REGION_LANES forces G
    static const int g_env = std::getenv("BZG_REGION_LANES") ? std::atoi(std::getenv("BZG_REGION_LANES")) : 0;
    int gl = 1;
    while (gl < 32 && V * gl * 2 <= 1152ll * c->num_sms) gl *= 2;
    if (g_env == 1 || g_env == 2 || g_env == 4 || g_env == 8 || g_env == 16 || g_env == 32) gl = g_env;
    launch(c, "k_region_masks", k_region_masks, dim3(div_up(V * gl, 128)), dim3(128), 0, rr, g->vertices.as<double>(),
           perm.as<int>(), V, m, rblo.as<double>(), rbhi.as<double>(), smask.as<unsigned long long>(),
           dmask.as<unsigned long long>(), sok.as<uint8_t>(), dok.as<uint8_t>(), gl);
    launch(c, "k_mask_or", k_mask_or, dim3(div_up(ng * rr.RW, 256), 2), dim3(256), 0, smask.as<unsigned long long>(),
           sok.as<uint8_t>(), V, rr.RW, tor.as<unsigned long long>(), dmask.as<unsigned long long>(),
           dok.as<uint8_t>(), gor.as<unsigned long long>());
    rm = RegionMasks{smask.as<unsigned long long>(), dmask.as<unsigned long long>(), tor.as<unsigned long long>(),
                     gor.as<unsigned long long>(), rr.RW};
  }
  c->trace("pairs: morton+proj+regions");
  // ---- the row block's sources, densely tiled in Morton order (multi-GPU row split: with the
  // full order a 32-source tile would hold ~32 / G sources of this block, and the cull, list
  // and staging work would not shrink with G); destinations stay the full sorted order
  const bool split = rows < V && rows > 0;
  BZG_REQUIRE(!bc || !split, BZG_EUNSUPPORTED, "a captured plan builds the whole graph");
  const long long Vs = split ? rows : V;
  const long long ngs = (Vs + kTile - 1) / kTile;
  TmpBuf s_perm(c), s_a1c(c), s_ok(c), s_smask(c), s_flag(c), s_pos(c), s_tor(c);
  const int* perm_src = perm.as<int>();
  const double* a1c_src = a1c.as<double>();
  const uint8_t* ok_src = sok.as<uint8_t>();
  RegionMasks rms = rm;
  if (split) {
    s_flag.alloc((V + 1) * sizeof(int), c->stream);
    s_pos.alloc((V + 1) * sizeof(int), c->stream);
    launch(c, "k_src_flags", k_src_flags, dim3(div_up(V, 256)), dim3(256), 0, perm.as<int>(), V, r0, r1,
           s_flag.as<int>());
    BZG_CHECK_CUDA(cudaMemsetAsync(s_flag.as<int>() + V, 0, sizeof(int), c->stream));
    exclusive_scan_i(c, s_flag.as<int>(), s_pos.as<int>(), V + 1);
    s_perm.alloc(Vs * sizeof(int), c->stream);
    s_a1c.alloc((size_t)Vs * Kpad * sizeof(double), c->stream);
    s_ok.alloc(Vs, c->stream);
    s_smask.alloc(std::max<long long>(R > 0 ? Vs * rm.RW : 1, 1) * sizeof(unsigned long long), c->stream);
    launch(c, "k_src_gather", k_src_gather, dim3(div_up(V, 256)), dim3(256), 0, perm.as<int>(), s_flag.as<int>(),
           s_pos.as<int>(), V, Kpad, a1c.as<double>(), sok.as<uint8_t>(), rm.smask, R > 0 ? rm.RW : 0,
           s_perm.as<int>(), s_a1c.as<double>(), s_ok.as<uint8_t>(), s_smask.as<unsigned long long>());
    perm_src = s_perm.as<int>();
    a1c_src = s_a1c.as<double>();
    ok_src = s_ok.as<uint8_t>();
    if (R > 0) {
      s_tor.alloc(ngs * rm.RW * sizeof(unsigned long long), c->stream);
      launch(c, "k_mask_or", k_mask_or, dim3(div_up(ngs * rm.RW, 256)), dim3(256), 0, s_smask.as<unsigned long long>(),
             ok_src, Vs, rm.RW, s_tor.as<unsigned long long>(), (const unsigned long long*)nullptr,
             (const uint8_t*)nullptr, (unsigned long long*)nullptr);
      rms.smask = s_smask.as<unsigned long long>();
      rms.tile_or = s_tor.as<unsigned long long>();
    }
  }
  TmpBuf tmin(c), tmax(c), gmin(c), gmax(c);
  tmin.alloc(ngs * Kpad * sizeof(double), c->stream);
  tmax.alloc(ngs * Kpad * sizeof(double), c->stream);
  gmin.alloc(ng * Kpad * sizeof(double), c->stream);
  gmax.alloc(ng * Kpad * sizeof(double), c->stream);
  launch(c, "k_group_bounds", k_group_bounds, dim3(div_up(ngs * Kpad, 256)), dim3(256), 0, a1c_src, 0, Vs, Kpad,
         ok_src, tmin.as<double>(), tmax.as<double>());
  launch(c, "k_group_bounds", k_group_bounds, dim3(div_up(ng * Kpad, 256)), dim3(256), 0, a2t.as<double>(), 1, V, Kpad,
         dok.as<uint8_t>(), gmin.as<double>(), gmax.as<double>());
  const bool use_list = (double)ngs * (double)ng * 8.0 <= 1.0e9;  // worst-case list fits 1 GB
  if (!never && rows > 0 && use_list) {
    // culls over every (tile, group) into a compact list, then one warp per survivor
    DevBuf& list = c->ws[WS_PAIRLIST];
    list.alloc((size_t)ngs * ng * sizeof(unsigned long long), c->stream);
    TmpBuf nlist(c);
    nlist.alloc(sizeof(unsigned long long), c->stream);
    BZG_CHECK_CUDA(cudaMemsetAsync(nlist.ptr, 0, sizeof(unsigned long long), c->stream));
    const bool reg = R > 0;
    launch(c, "k_tile_group_cull", k_tile_group_cull, dim3(div_up(ng, 256), (unsigned)ngs), dim3(256), 0, bd,
           tmin.as<double>(), tmax.as<double>(), gmin.as<double>(), gmax.as<double>(), ng, Kpad, rms, (int)reg,
           list.as<unsigned long long>(), nlist.as<unsigned long long>());
    auto go = [&](auto kern, size_t smem) {
      ensure_dyn_smem((const void*)kern, smem);
      launch(c, "k_pair_list", kern, dim3((unsigned)(c->num_sms * 3)), dim3(kPairThreads), smem, bd,
             a1c_src, a2t.as<double>(), ok_src, dok.as<uint8_t>(), perm.as<int>(),
             gmin.as<double>(), gmax.as<double>(), V, r0, W, bits.as<uint32_t>(), rowcnt.as<unsigned long long>(), rms,
             list.as<unsigned long long>(), nlist.as<unsigned long long>(), perm_src, Vs);
    };
#define BZG_K(k)                                                                                        \
  case k:                                                                                               \
    if (reg) go(k_pair_list<k, true>, pair_list_smem<k, true>()); else go(k_pair_list<k, false>, pair_list_smem<k, false>()); \
    break;
    switch (Kpad) {
      BZG_K(4) BZG_K(8) BZG_K(12) BZG_K(16) BZG_K(24) BZG_K(32) BZG_K(48)
      default:
        if (reg) go(k_pair_list<64, true>, pair_list_smem<64, true>()); else go(k_pair_list<64, false>, pair_list_smem<64, false>());
        break;
    }
#undef BZG_K
  } else if (!never && rows > 0) {
    dim3 grid(div_up(V, kPairThreads), (unsigned)ngs);
    auto go = [&](auto kern) {
      launch(c, "k_pair_tiles", kern, grid, dim3(kPairThreads), 0, bd, a1c_src, a2t.as<double>(),
             ok_src, dok.as<uint8_t>(), perm.as<int>(), tmin.as<double>(), tmax.as<double>(),
             gmin.as<double>(), gmax.as<double>(), V, r0, W, bits.as<uint32_t>(), rowcnt.as<unsigned long long>(), rms,
             perm_src, Vs);
    };
    const bool reg = R > 0;
#define BZG_K(k) \
  case k: if (reg) go(k_pair_tiles<k, true>); else go(k_pair_tiles<k, false>); break;
    switch (Kpad) {
      BZG_K(4) BZG_K(8) BZG_K(12) BZG_K(16) BZG_K(24) BZG_K(32) BZG_K(48)
      default: if (reg) go(k_pair_tiles<64, true>); else go(k_pair_tiles<64, false>); break;
    }
#undef BZG_K
  }
  if (d->k_nearest >= 0 && !never && rows > 0 && !count_only) {
    BZG_REQUIRE(m <= 3, BZG_EUNSUPPORTED, "k_nearest prefilter supports m <= 3");
    const long long k = std::min<long long>(d->k_nearest, V - 1);
    launch(c, "k_knn_rows", k_knn_rows, dim3((unsigned)rows), dim3(kKnnThreads), 0, g->vertices.as<double>(), V, n, m,
           k, r0, W, bits.as<uint32_t>(), rowcnt.as<unsigned long long>());
  }
  c->trace("pairs: tiles(+knn)");
  exclusive_scan_ll(c, rowcnt.as<unsigned long long>(), rptr.as<long long>(), rows + 1);
  if (bc) {
    // captured plan: no read-back here.  The CSR arrays already have the plan's capacity (E on
    // the host); the edge count stays on the device (rptr[rows], read by the cut and search
    // kernels through Graph::dE) and reaches the host with the sampler's acceptance count at
    // the end of the launch, where the plan checks both.
    BZG_CHECK_CUDA(cudaMemcpyAsync(bc->h_out, rptr.as<long long>() + rows, sizeof(long long), cudaMemcpyDeviceToHost,
                                   c->stream));
    if (c->sample_check)
      BZG_CHECK_CUDA(cudaMemcpyAsync(bc->h_sampled, c->sample_check, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sample_check = nullptr;
    DParams dp{};
    for (size_t k = 0; k < g->D.size(); ++k) dp.D[k] = g->D[k];
    dispatch_gm(g->gamma, g->m, [&](auto G_, auto M_) {
      constexpr int Gc = decltype(G_)::value, Mc = decltype(M_)::value;
      launch(c, "k_expand", k_expand<Gc, Mc>, dim3(div_up(rows * 32, kExpandThreads)), dim3(kExpandThreads), 0, dp,
             g->vertices.as<double>(), r0, r1, W, bits.as<uint32_t>(), rptr.as<long long>(), g->src.as<int>(),
             g->dst.as<int>(), g->cost.as<double>(), (long long)g->E);
    });
    launch(c, "k_row_ptr_global", k_row_ptr_global, dim3(div_up(V + 1, 256)), dim3(256), 0, rptr.as<long long>(),
           V, r0, r1, g->row_ptr.as<long long>(), (long long)g->E);
    return true;
  }
  long long* h = static_cast<long long*>(c->host_scratch(2 * sizeof(long long)));
  BZG_CHECK_CUDA(cudaMemcpyAsync(h, rptr.as<long long>() + rows, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  int* sampled = c->sample_check;
  if (sampled) {
    h[1] = 0;
    BZG_CHECK_CUDA(cudaMemcpyAsync(h + 1, sampled, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  }
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  if (sampled) {  // the single sampler round of this build (sample_states): enough acceptances?
    c->sample_check = nullptr;
    const long long acc = (long long)(int)h[1];
    c->sample_est = std::max(1e-3, (double)acc / (double)c->sample_count);
    if (acc < c->sample_need) return false;  // the caller resamples with the checked loop
  }
  const long long E = h[0];
  if (count_only) {
    *count_only = E;
    return true;
  }
  BZG_REQUIRE(E < (1ll << 31), BZG_EUNSUPPORTED, "edge count exceeds the int32 CSR index range");
  g->E = E;
  ++g->version;
  g->src.alloc(E * sizeof(int), c->stream);
  g->dst.alloc(E * sizeof(int), c->stream);
  g->cost.alloc(E * sizeof(double), c->stream);
  g->row_ptr.alloc((V + 1) * sizeof(long long), c->stream);
  c->trace("pairs: scan+csr alloc");
  DParams dp{};
  for (size_t k = 0; k < g->D.size(); ++k) dp.D[k] = g->D[k];
  if (E > 0) {
    dispatch_gm(g->gamma, g->m, [&](auto G_, auto M_) {
      constexpr int Gc = decltype(G_)::value, Mc = decltype(M_)::value;
      launch(c, "k_expand", k_expand<Gc, Mc>, dim3(div_up(rows * 32, kExpandThreads)), dim3(kExpandThreads), 0, dp,
             g->vertices.as<double>(), r0, r1, W, bits.as<uint32_t>(), rptr.as<long long>(), g->src.as<int>(),
             g->dst.as<int>(), g->cost.as<double>(), E);
    });
  }
  launch(c, "k_row_ptr_global", k_row_ptr_global, dim3(div_up(V + 1, 256)), dim3(256), 0, rptr.as<long long>(),
         V, r0, r1, g->row_ptr.as<long long>(), E);
  return true;
}

void set_edges(Ctx* c, Graph* g, long long E, const int* src, const int* dst, const double* cost, bool on_device) {
  const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  BZG_REQUIRE(E >= 0 && E < (1ll << 31), BZG_EINVAL, "edge count out of range");
  g->E = E;
  ++g->version;
  g->row_begin = 0;
  g->row_end = g->V;
  g->points_ready = false;
  g->cut_cache.clear();  // the cached cut outcomes belong to the old edge set
  g->cut_cache.Wb = 0;
  g->src.alloc(std::max(E, 1ll) * sizeof(int), c->stream);
  g->dst.alloc(std::max(E, 1ll) * sizeof(int), c->stream);
  g->cost.alloc(std::max(E, 1ll) * sizeof(double), c->stream);
  if (E > 0) {
    BZG_CHECK_CUDA(cudaMemcpyAsync(g->src.ptr, src, E * sizeof(int), kind, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(g->dst.ptr, dst, E * sizeof(int), kind, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(g->cost.ptr, cost, E * sizeof(double), kind, c->stream));
  }
  g->row_ptr.alloc((g->V + 1) * sizeof(long long), c->stream);
  launch(c, "k_row_ptr_from_src", k_row_ptr_from_src, dim3(div_up(g->V + 1, 256)), dim3(256), 0, g->src.as<int>(), E,
         g->V, g->row_ptr.as<long long>());
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
}

void materialize_points(Ctx* c, Graph* g) {
  if (g->points_ready) return;
  const long long E = g->E;
  g->points.alloc((size_t)std::max(E, 1ll) * g->m * (g->p + 1) * sizeof(double), c->stream);
  DParams dp{};
  for (size_t k = 0; k < g->D.size(); ++k) dp.D[k] = g->D[k];
  if (E > 0) {
    dispatch_gm(g->gamma, g->m, [&](auto G_, auto M_) {
      constexpr int Gc = decltype(G_)::value, Mc = decltype(M_)::value;
      launch(c, "k_points", k_points<Gc, Mc>, dim3(div_up(E, 256)), dim3(256), 0, dp, g->vertices.as<double>(), E,
             g->src.as<int>(), g->dst.as<int>(), g->points.as<double>());
    });
  }
  g->points_ready = true;
}

void check_edges(Ctx* c, int n, int n_F, const double* F, const double* G, double eps, int64_t k,
                 const double* X1, const double* X2, uint8_t* out) {
  if (k <= 0) return;
  std::vector<double> th(n_F);
  for (int r = 0; r < n_F; ++r) th[r] = G[r] + eps;
  c->arena->reset();
  TmpBuf dF(c), dT(c), d1(c), d2(c), dout(c);
  dF.alloc((size_t)n_F * 2 * n * 8, c->stream);
  dT.alloc((size_t)n_F * 8, c->stream);
  d1.alloc((size_t)k * n * 8, c->stream);
  d2.alloc((size_t)k * n * 8, c->stream);
  dout.alloc(k, c->stream);
  BZG_CHECK_CUDA(cudaMemcpyAsync(dF.ptr, F, (size_t)n_F * 2 * n * 8, cudaMemcpyHostToDevice, c->stream));
  BZG_CHECK_CUDA(cudaMemcpyAsync(dT.ptr, th.data(), (size_t)n_F * 8, cudaMemcpyHostToDevice, c->stream));
  BZG_CHECK_CUDA(cudaMemcpyAsync(d1.ptr, X1, (size_t)k * n * 8, cudaMemcpyHostToDevice, c->stream));
  BZG_CHECK_CUDA(cudaMemcpyAsync(d2.ptr, X2, (size_t)k * n * 8, cudaMemcpyHostToDevice, c->stream));
  launch(c, "k_check_edges", k_check_edges, dim3(div_up(k, 256)), dim3(256), 0, dF.as<double>(), dT.as<double>(),
         n, n_F, (long long)k, d1.as<double>(), d2.as<double>(), dout.as<uint8_t>());
  BZG_CHECK_CUDA(cudaMemcpyAsync(out, dout.ptr, k, cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace bzg
