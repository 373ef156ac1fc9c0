// Shortest path on device: start/goal snapping, (reverse) reachability, min-plus
// Bellman-Ford relaxation to the fixed point, Dijkstra-equivalent parent rule and
// backtracking.
//
// Replaces reference graph.py:353-430 (find_path) and graph.py:433-450 (_reaches_goal).
// The fixed point d[v] = min_u fl(d[u] + c_uv) equals the heapq Dijkstra distances
// (fl(x + c) is monotone in x and costs are positive), and parent[v] =
// argmin_(d[u], u) over alive tight in-edges reproduces the heap's pop order, so the
// node sequence and dist[vg] are bitwise those of the reference.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "bzg_internal.cuh"
#include "bzg_math.cuh"

namespace cg = cooperative_groups;

namespace bzg {

namespace {

constexpr unsigned long long kInfBits = 0x7FF0000000000000ull;

struct SnapParams {
  double target[16];
  double tlo[16], thi[16];  // start - v tube window: diff >= -hi - eps, diff <= -lo + eps
  int n, m_norm;            // components entering the norm (n, or m when position-only)
  int mode;                 // 0: goal (all vertices), 1: tube filter, 2: reach filter
};

// norm of (v - target) over the first m_norm components, numpy order (graph.py:375/379):
// sqrt of the sequential sum of squares.
__device__ __forceinline__ double snap_norm(const double* v, const SnapParams& sp) {
  // np.linalg.norm(axis=1) = sqrt(add.reduce(d*d)) over each contiguous row: numpy's pairwise
  // sum, which is a left fold below 8 terms and, from 8 to 128 terms, eight interleaved
  // partial sums combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a left-folded tail
  // (checked against numpy for n = 4, 6, 8, 9, 12 on 200k rows).
  const int n = sp.m_norm;
  double sq[16];
  for (int k = 0; k < n; ++k) {
    const double dk = __dsub_rn(v[k], sp.target[k]);
    sq[k] = __dmul_rn(dk, dk);
  }
  double s;
  int k0;
  if (n < 8) {
    s = sq[0];
    k0 = 1;
  } else {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = sq[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sq[i + j]);
    s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                  __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    k0 = i;
  }
  for (int k = k0; k < n; ++k) s = __dadd_rn(s, sq[k]);
  return __dsqrt_rn(s);
}

// first argmin (value, index) over candidates; infinite values are skipped so an
// all-excluded set returns index -1.
// spd: the parameters in device memory (a captured query, whose start/goal change per launch),
// else the by-value sp
__global__ void k_snap(SnapParams sp_val, const SnapParams* __restrict__ spd, const double* __restrict__ Vx,
                       long long V, const uint8_t* __restrict__ reach, unsigned long long* __restrict__ best) {
  BZG_PDL_ENTRY();
  const SnapParams& sp = spd ? *spd : sp_val;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double val = INFINITY;
  long long idx = -1;
  if (i < V) {
    const double* v = Vx + i * sp.n;
    bool ok = true;
    if (sp.mode == 1) {
      for (int k = 0; k < sp.n; ++k) {
        const double d = __dsub_rn(v[k], sp.target[k]);
        ok = ok && d >= sp.tlo[k] && d <= sp.thi[k];
      }
    } else if (sp.mode == 2) {
      ok = reach[i] != 0;
    }
    if (ok) {
      val = snap_norm(v, sp);
      idx = i;
    }
  }
  // warp then block argmin, ties to the lower index
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, val, off);
    const long long oi = __shfl_down_sync(0xffffffffu, idx, off);
    if (oi >= 0 && (idx < 0 || ov < val || (ov == val && oi < idx))) { val = ov; idx = oi; }
  }
  __shared__ double sv[32];
  __shared__ long long si[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sv[w] = val; si[w] = idx; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    val = lane < nw ? sv[lane] : INFINITY;
    idx = lane < nw ? si[lane] : -1;
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, val, off);
      const long long oi = __shfl_down_sync(0xffffffffu, idx, off);
      if (oi >= 0 && (idx < 0 || ov < val || (ov == val && oi < idx))) { val = ov; idx = oi; }
    }
    if (lane == 0 && idx >= 0) {
      // best[0]: min value bits (values are >= 0, so bit order == value order)
      atomicMin(best, dbits(val));
      best[1 + blockIdx.x] = ((unsigned long long)dbits(val));
      best[1 + gridDim.x + blockIdx.x] = (unsigned long long)idx;
    } else if (lane == 0) {
      best[1 + blockIdx.x] = kInfBits + 1;  // marks "no candidate" (above +inf bits)
    }
  }
}

__global__ void k_snap_final(unsigned long long* __restrict__ best, int nblocks, long long* __restrict__ out) {
  BZG_PDL_ENTRY();
  // single warp: lowest index among blocks whose local minimum equals the global minimum
  const int lane = threadIdx.x;
  const unsigned long long m = best[0];
  long long idx = -1;
  for (int b = lane; b < nblocks; b += 32) {
    if (best[1 + b] == m && m != kInfBits + 2) {
      const long long bi = (long long)best[1 + nblocks + b];
      if (idx < 0 || bi < idx) idx = bi;
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const long long oi = __shfl_down_sync(0xffffffffu, idx, off);
    if (oi >= 0 && (idx < 0 || oi < idx)) idx = oi;
  }
  if (lane == 0) *out = idx;
}

// Reverse reachability to vg (graph.py:433-450, _reaches_goal) in one cooperative launch: vg
// from the device plan; sweeps over the alive edges mark src when dst is marked, a grid barrier
// per sweep, until a sweep marks nothing.  Cached per (mask, vg) through `key` on the device.
// Small graphs (V <= kSnapBlockV): a snap as ONE block per parameter set -- the strided scan
// keeps each thread's first minimum, the block reduction the lowest index among equal values,
// i.e. k_snap + k_snap_final's first argmin -- so the goal and (tube) start snaps are one
// launch instead of six.  Block b handles parameter set first + b and writes out[b].
constexpr long long kSnapBlockV = 16384;
__global__ void __launch_bounds__(1024) k_snap_block(SnapParams s0, SnapParams s1, const SnapParams* __restrict__ spd,
                                                     int first, const double* __restrict__ Vx, long long V,
                                                     const uint8_t* __restrict__ reach, long long* __restrict__ out) {
  BZG_PDL_ENTRY();
  const int set = first + blockIdx.x;
  const SnapParams& sp = spd ? spd[set] : (set == 0 ? s0 : s1);
  double val = INFINITY;
  long long idx = -1;
  for (long long i = threadIdx.x; i < V; i += blockDim.x) {
    const double* v = Vx + i * sp.n;
    bool ok = true;
    if (sp.mode == 1) {
      for (int k = 0; k < sp.n; ++k) {
        const double d = __dsub_rn(v[k], sp.target[k]);
        ok = ok && d >= sp.tlo[k] && d <= sp.thi[k];
      }
    } else if (sp.mode == 2) {
      ok = reach[i] != 0;
    }
    if (ok) {
      const double nv = snap_norm(v, sp);
      if (idx < 0 || nv < val) { val = nv; idx = i; }  // ascending i: keep the first minimum
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, val, off);
    const long long oi = __shfl_down_sync(0xffffffffu, idx, off);
    if (oi >= 0 && (idx < 0 || ov < val || (ov == val && oi < idx))) { val = ov; idx = oi; }
  }
  __shared__ double sv[32];
  __shared__ long long si[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sv[w] = val; si[w] = idx; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    val = lane < nw ? sv[lane] : INFINITY;
    idx = lane < nw ? si[lane] : -1;
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, val, off);
      const long long oi = __shfl_down_sync(0xffffffffu, idx, off);
      if (oi >= 0 && (idx < 0 || ov < val || (ov == val && oi < idx))) { val = ov; idx = oi; }
    }
    if (lane == 0) out[blockIdx.x] = idx;
  }
}

// GRID: one cooperative grid and grid barriers; else ONE thread-block cluster (the launch's
// whole grid) and cluster barriers -- far cheaper per sweep for small graphs (k_bf_cluster).
template <bool GRID>
__global__ void k_reach_sweeps(long long E, long long V, const int* __restrict__ src, const int* __restrict__ dst,
                               const uint8_t* __restrict__ alive, uint8_t* __restrict__ reach,
                               long long* __restrict__ key, const long long* __restrict__ plan, int* __restrict__ flags,
                               const long long* __restrict__ dE) {
  BZG_PDL_ENTRY();
  if (dE) E = min(E, *dE);  // a captured plan's edge count (E = its capacity)
  const long long vg = plan[0];
  if (*(volatile long long*)key == vg) return;  // uniform: the cached set is vg's
  auto sync = [] {
    if constexpr (GRID) cg::this_grid().sync(); else cg::this_cluster().sync();
  };
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  for (long long i = tid; i < V; i += nt) reach[i] = i == vg ? 1 : 0;
  if (tid < 3) flags[tid] = 0;
  sync();
  for (int sweep = 0; sweep <= V + 1; ++sweep) {
    if (tid == 0) flags[(sweep + 1) % 3] = 0;
    bool any = false;
    for (long long e = tid; e < E; e += nt) {
      if (alive && !alive[e]) continue;
      const int u = src[e];
      if (reach[dst[e]] && !reach[u]) {
        reach[u] = 1;
        any = true;
      }
    }
    if (any) flags[sweep % 3] = 1;
    sync();
    if (*(volatile int*)&flags[sweep % 3] == 0) break;
  }
  sync();
  if (tid == 0) *key = vg;
}

// The same reverse reachability pulled bottom-up over the forward CSR: one warp per still-
// unmarked vertex scans its alive out-edges 32 at a time and stops at the first marked dst;
// marked vertices are skipped, so a sweep reads only the unmarked vertices' edges (up to their
// first hit) where the edge sweeps read all E edges every sweep; a grid barrier per sweep,
// until a sweep marks nothing.  Marks only grow and each is a vertex with an alive route to vg:
// the set is the edge sweeps' fixed point.  (A top-down frontier over a reverse CSR for the
// first sweeps measured no faster on cfg3: 111 vs 113 us per search.)
__global__ void k_reach_pull(long long V, const long long* __restrict__ fptr, const int* __restrict__ fdst,
                             const uint8_t* __restrict__ alive, uint8_t* __restrict__ reach,
                             long long* __restrict__ key, const long long* __restrict__ plan, int* __restrict__ flags,
                             const long long* __restrict__ dE) {
  BZG_PDL_ENTRY();
  const long long vg = plan[0];
  if (*(volatile long long*)key == vg) return;  // uniform: the cached set is vg's
  cg::grid_group grid = cg::this_grid();
  const long long Ecl = dE ? *dE : LLONG_MAX;  // a captured plan's edge count
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const long long wg = tid / 32, nw = nt / 32;
  for (long long i = tid; i < V; i += nt) reach[i] = i == vg ? 1 : 0;
  if (tid < 3) flags[tid] = 0;
  grid.sync();
  volatile uint8_t* vr = reach;
  // flags[t % 3]: "sweep t marked something", cleared one sweep ahead
  for (long long t = 0; t <= V + 1; ++t) {
    if (tid == 0) flags[(t + 1) % 3] = 0;
    bool any = false;
    for (long long u = wg; u < V; u += nw) {
      if (__shfl_sync(0xffffffffu, (int)vr[u], 0)) continue;  // warp-uniform
      const long long k0 = fptr[u], k1 = min(fptr[u + 1], Ecl);
      bool hit = false;
      for (long long k = k0; k < k1 && !hit; k += 32) {
        const long long kk = k + lane;
        const bool ok = kk < k1 && (!alive || alive[kk]) && vr[fdst[kk]];
        hit = __any_sync(0xffffffffu, ok);
      }
      if (hit) {
        if (lane == 0) vr[u] = 1;
        any = true;
      }
    }
    if (any && lane == 0) flags[t % 3] = 1;
    grid.sync();
    if (*(volatile int*)&flags[t % 3] == 0) break;
  }
  grid.sync();
  if (tid == 0) *key = vg;
}

// Frontier Bellman-Ford as one persistent cooperative kernel: a queue of the vertices
// improved in the previous sweep (each enqueued once per sweep through its stamp); one warp
// per queued vertex relaxes its alive out-edges with fl(d[u] + c) and atomicMin on the
// (non-negative) double bits; grid-wide barriers between sweeps; stops when a sweep improves
// nothing.  No host round trip per sweep.
__global__ void k_bf_persistent(long long V, const long long* __restrict__ row_ptr, const int* __restrict__ dst,
                                const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                                unsigned long long* __restrict__ dist, int* __restrict__ stamp, int* __restrict__ qa,
                                int* __restrict__ qb, int* __restrict__ counts, int max_sweeps,
                                const long long* __restrict__ plan) {
  BZG_PDL_ENTRY();
  if (!plan[2]) return;  // grid-uniform
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const long long wg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const long long nw = ((long long)gridDim.x * blockDim.x) / 32;
  // frontier sizes rotate through counts[0..2]: sweep s reads counts[(s-1)%3], appends to
  // counts[s%3] and zeroes counts[(s+1)%3] (last read in sweep s-1, next written in sweep s+1),
  // so one grid-wide barrier per sweep suffices
  int sweep = 1;
  for (; sweep <= max_sweeps; ++sweep) {
    const int* qin = (sweep & 1) ? qa : qb;
    int* qout = (sweep & 1) ? qb : qa;
    const int cin = *(volatile int*)&counts[(sweep - 1) % 3];
    if (cin == 0) break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      counts[(sweep + 1) % 3] = 0;
      counts[4] += cin;  // frontier vertices expanded (diagnostic)
    }
    int* cout = counts + sweep % 3;
    for (long long k = wg; k < cin; k += nw) {
      const int u = qin[k];
      const double du = __longlong_as_double((long long)__ldcg(dist + u));
      const long long e1 = row_ptr[u + 1];
      // four edges per lane per pass, their loads issued together (the sweep is latency-bound)
      for (long long eb = row_ptr[u] + lane; eb < e1; eb += 128) {
        int vv[4];
        double cc[4];
        bool ok[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long long e = eb + 32 * q;
          ok[q] = e < e1 && (!alive || alive[e]);
          vv[q] = ok[q] ? dst[e] : 0;
          cc[q] = ok[q] ? cost[e] : 0.0;
        }
        unsigned long long dv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) dv[q] = ok[q] ? __ldcg(dist + vv[q]) : 0ull;
        const unsigned am = __activemask();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bool push = false;
          if (ok[q]) {
            const unsigned long long nb = dbits(__dadd_rn(du, cc[q]));
            if (nb < dv[q]) {
              const unsigned long long old = atomicMin(dist + vv[q], nb);
              push = nb < old && atomicExch(stamp + vv[q], sweep) != sweep;
            }
          }
          // warp-aggregated enqueue: one atomic on the frontier counter per warp and round
          // (a per-lane atomicAdd on the single counter serialised the sweep at large V)
          const unsigned want = __ballot_sync(am, push);
          if (want) {
            const int leader = __ffs(want) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(cout, __popc(want));
            base = __shfl_sync(am, base, leader);
            if (push) qout[base + __popc(want & ((1u << lane) - 1u))] = vv[q];
          }
        }
      }
    }
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[3] = sweep - 1;
}

// Same frontier Bellman-Ford with the improvement detection moved out of the relax loop:
// the relax phase issues fire-and-forget atomicMin (RED) on the distance bits, and after a
// grid barrier a scan over all vertices enqueues those whose distance dropped since the last
// scan (prev[]), deduplicated by construction.  The queue variant above waits on two
// returning atomics (atomicMin, then the stamp exchange) per improvement, which at large V
// made every sweep latency-bound.  Two barriers per sweep; same fixpoint.
__global__ void k_bf_scan(long long V, const long long* __restrict__ row_ptr, const int* __restrict__ dst,
                          const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                          unsigned long long* __restrict__ dist, unsigned long long* __restrict__ prev,
                          int* __restrict__ qa, int* __restrict__ qb, int* __restrict__ counts, int max_sweeps,
                          const long long* __restrict__ plan) {
  BZG_PDL_ENTRY();
  if (!plan[2]) return;  // grid-uniform
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const long long wg = tid / 32, nw = nt / 32;
  int sweep = 1;
  for (; sweep <= max_sweeps; ++sweep) {
    const int* qin = (sweep & 1) ? qa : qb;
    int* qout = (sweep & 1) ? qb : qa;
    const int cin = *(volatile int*)&counts[(sweep - 1) % 3];
    if (cin == 0) break;
    if (tid == 0) {
      counts[(sweep + 1) % 3] = 0;
      counts[4] += cin;
    }
    for (long long k = wg; k < cin; k += nw) {
      const int u = qin[k];
      const double du = __longlong_as_double((long long)__ldcg(dist + u));
      const long long e1 = row_ptr[u + 1];
      for (long long eb = row_ptr[u] + lane; eb < e1; eb += 128) {
        int vv[4];
        double cc[4];
        bool ok[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const long long e = eb + 32 * q;
          ok[q] = e < e1 && (!alive || alive[e]);
          vv[q] = ok[q] ? dst[e] : 0;
          cc[q] = ok[q] ? cost[e] : 0.0;
        }
        unsigned long long dv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) dv[q] = ok[q] ? __ldcg(dist + vv[q]) : 0ull;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const unsigned long long nb = dbits(__dadd_rn(du, cc[q]));
          if (ok[q] && nb < dv[q]) atomicMin(dist + vv[q], nb);
        }
      }
    }
    grid.sync();
    int* cout = counts + sweep % 3;
    for (long long v0 = tid - lane; v0 < V; v0 += nt) {  // warp-uniform trip count
      const long long v = v0 + lane;
      bool push = false;
      if (v < V) {
        const unsigned long long d = __ldcg(dist + v);
        if (d != prev[v]) {
          prev[v] = d;
          push = true;
        }
      }
      const unsigned want = __ballot_sync(0xffffffffu, push);
      if (want) {
        const int leader = __ffs(want) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(cout, __popc(want));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (push) qout[base + __popc(want & ((1u << lane) - 1u))] = (int)v;
      }
    }
    grid.sync();
  }
  if (tid == 0) counts[3] = sweep - 1;
}

// Tiny graphs (V <= kBfCtaMaxV, E <= kBfCtaMaxE): the frontier Bellman-Ford in ONE thread
// block with the distances, stamps and both frontier queues in shared memory -- every sweep is a
// block barrier and the relaxations are shared-memory atomics; only the edges come from L2.
constexpr int kBfCtaThreads = 1024;
constexpr long long kBfCtaMaxV = 4096, kBfCtaMaxE = 32768;
__global__ void __launch_bounds__(kBfCtaThreads, 1)
k_bf_cta(long long V, const long long* __restrict__ row_ptr, const int* __restrict__ dst,
         const double* __restrict__ cost, const uint8_t* __restrict__ alive, unsigned long long* __restrict__ dist,
         int* __restrict__ counts, int max_sweeps, const long long* __restrict__ plan) {
  BZG_PDL_ENTRY();
  if (!plan[2]) return;  // block-uniform
  extern __shared__ unsigned long long smem_u64[];
  unsigned long long* sd = smem_u64;               // V distances (double bits)
  int* sstamp = reinterpret_cast<int*>(sd + V);    // V stamps: last sweep that enqueued the vertex
  int* qa = sstamp + V;                            // two frontier queues of V entries
  int* qb = qa + V;
  __shared__ int scount[3];
  const int v0 = (int)plan[1];
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    sd[i] = i == v0 ? 0ull : kInfBits;
    sstamp[i] = i == v0 ? 0 : -1;
  }
  if (threadIdx.x == 0) {
    qa[0] = v0;
    scount[0] = 1;
    scount[1] = 0;
    scount[2] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int sweep = 1;
  for (; sweep <= max_sweeps; ++sweep) {
    const int* qin = (sweep & 1) ? qa : qb;
    int* qout = (sweep & 1) ? qb : qa;
    const int cin = scount[(sweep - 1) % 3];
    if (cin == 0) break;
    if (threadIdx.x == 0) scount[(sweep + 1) % 3] = 0;
    int* cout = scount + sweep % 3;
    for (int k = wid; k < cin; k += nw) {
      const int u = qin[k];
      const double du = __longlong_as_double((long long)sd[u]);
      const long long e1 = row_ptr[u + 1];
      for (long long eb = row_ptr[u] + lane; eb < e1; eb += 64) {
        int vv[2];
        double cc[2];
        bool ok[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const long long e = eb + 32 * t;
          ok[t] = e < e1 && (!alive || alive[e]);
          vv[t] = ok[t] ? dst[e] : 0;
          cc[t] = ok[t] ? cost[e] : 0.0;
        }
        const unsigned am = __activemask();
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          bool push = false;
          if (ok[t]) {
            const unsigned long long nb = dbits(__dadd_rn(du, cc[t]));
            if (nb < sd[vv[t]]) {
              const unsigned long long old = atomicMin(sd + vv[t], nb);
              push = nb < old && atomicExch(sstamp + vv[t], sweep) != sweep;
            }
          }
          const unsigned want = __ballot_sync(am, push);
          if (want) {
            const int leader = __ffs(want) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(cout, __popc(want));
            base = __shfl_sync(am, base, leader);
            if (push) qout[base + __popc(want & ((1u << lane) - 1u))] = vv[t];
          }
        }
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < V; i += blockDim.x) dist[i] = sd[i];
  if (threadIdx.x == 0) {
    counts[3] = sweep - 1;
    counts[4] = 0;
  }
}

// Thread-block-cluster Bellman-Ford (graphs up to kBfClusterMaxV vertices): the frontier
// Bellman-Ford of k_bf_scan on the CTAs of ONE cluster, so a sweep ends with a cluster barrier
// (barrier.cluster, far cheaper than the cooperative grid barrier, which costs ~2 us per sweep
// and is most of a small graph's search).  CTA r owns the vertex slice [r*chunk, (r+1)*chunk):
// one phase per sweep, each CTA scans its slice for vertices whose distance dropped since its
// last scan (prev, in shared memory), queues them in shared memory, relaxes their alive
// out-edges with fire-and-forget atomicMin on the global distance bits (L2), and adds its queue
// length to a cluster-wide counter in CTA 0's shared memory; the search ends after the barrier
// that shows a sweep with an empty frontier everywhere.  Same fixed point as the other schedules.
constexpr int kBfClusterThreads = 1024;
constexpr long long kBfClusterMaxV = 16 * 16 * 1024;
// default range of the cluster schedule: cfg2 (V = 2k, 249k edges) 0.056 ms vs 0.084 for the
// grid rescan; cfg3 (20k, 4.5M) 0.201 vs 0.203 -- even; cfg5 100k (14M edges) 13 ms: 16 SMs are
// far too few for the relaxations there
constexpr long long kBfClusterDefaultV = 16384, kBfClusterDefaultE = 2ll << 20;
__global__ void __launch_bounds__(kBfClusterThreads, 1)
k_bf_cluster(long long V, long long chunk, const long long* __restrict__ row_ptr, const int* __restrict__ dst,
             const double* __restrict__ cost, const uint8_t* __restrict__ alive, unsigned long long* __restrict__ dist,
             int* __restrict__ counts, int max_sweeps, const long long* __restrict__ plan) {
  BZG_PDL_ENTRY();
  if (!plan[2]) return;  // cluster-uniform
  cg::cluster_group cl = cg::this_cluster();  // barriers: barrier.cluster arrive.release / wait.acquire
  extern __shared__ unsigned long long smem_u64[];
  unsigned long long* sprev = smem_u64;            // chunk: the owned distances at the last scan
  int* q = reinterpret_cast<int*>(sprev + chunk);  // the local frontier (global vertex ids)
  __shared__ int tot[3];                           // rank 0's: frontier totals per phase (mod 3)
  __shared__ int qn;
  const unsigned rank = cl.block_rank();
  const long long v_lo = (long long)rank * chunk;
  const long long n_own = max(0ll, min(chunk, V - v_lo));
  // k_init_tree set dist (0 at v0, +inf elsewhere); prev = +inf everywhere, so v0 shows up as
  // dropped in the first scan
  for (long long i = threadIdx.x; i < chunk; i += blockDim.x) sprev[i] = kInfBits;
  if (threadIdx.x < 3) tot[threadIdx.x] = 0;
  int* tot0 = cl.map_shared_rank(tot, 0);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  cl.sync();
  int phase = 0;
  for (; phase <= max_sweeps; ++phase) {
    if (phase > 0 && *(volatile int*)&tot0[(phase - 1) % 3] == 0) break;  // last sweep relaxed nothing
    if (rank == 0 && threadIdx.x == 0) tot[(phase + 1) % 3] = 0;
    // scan the owned slice: vertices whose distance dropped form this sweep's frontier
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
    for (long long i0 = (long long)threadIdx.x - lane; i0 < n_own; i0 += blockDim.x) {  // warp-uniform
      const long long i = i0 + lane;
      bool push = false;
      if (i < n_own) {
        const unsigned long long d = __ldcg(dist + v_lo + i);
        if (d != sprev[i]) {
          sprev[i] = d;
          push = true;
        }
      }
      const unsigned want = __ballot_sync(0xffffffffu, push);
      if (want) {
        const int leader = __ffs(want) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&qn, __popc(want));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (push) q[base + __popc(want & ((1u << lane) - 1u))] = (int)(v_lo + i);
      }
    }
    __syncthreads();
    const int cin = qn;
    if (threadIdx.x == 0 && cin) atomicAdd(&tot0[phase % 3], cin);
    // relax the frontier's alive out-edges (a stale, larger du only gives a larger candidate;
    // the later drop is caught by the next scan)
    for (int k = wid; k < cin; k += nw) {
      const int u = q[k];
      const double du = __longlong_as_double((long long)sprev[u - v_lo]);
      const long long e1 = row_ptr[u + 1];
      for (long long eb = row_ptr[u] + lane; eb < e1; eb += 128) {
        int vv[4];
        double cc[4];
        bool ok[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const long long e = eb + 32 * t;
          ok[t] = e < e1 && (!alive || alive[e]);
          vv[t] = ok[t] ? dst[e] : 0;
          cc[t] = ok[t] ? cost[e] : 0.0;
        }
        unsigned long long dv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) dv[t] = ok[t] ? __ldcg(dist + vv[t]) : 0ull;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const unsigned long long nb = dbits(__dadd_rn(du, cc[t]));
          if (ok[t] && nb < dv[t]) atomicMin(dist + vv[t], nb);
        }
      }
    }
    cl.sync();
  }
  if (rank == 0 && threadIdx.x == 0) {
    counts[3] = phase;
    counts[4] = 0;
  }
  cl.sync();  // no CTA leaves while others may still read CTA 0's counters
}

__global__ void k_fill_u64(unsigned long long* p, long long n, unsigned long long v) {
  BZG_PDL_ENTRY();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// ---------------------------------------------------------------- device-resident plan
// find_path keeps (vg, v0) and the decisions that depend on them on the device, so a search is
// one stream of launches and one host synchronisation (the path read-back).
//   plan[0] = vg, plan[1] = v0 (-1: no snappable start), plan[2] = 1 when the shortest-path
//   tree must be (re)built, plan[3] = 1 when the mask's cached tree (tree_key = its v0) is
//   reused.  Kernels that build the tree return at once when plan[2] == 0.
__global__ void k_plan(long long* __restrict__ plan, long long* __restrict__ tree_key) {
  BZG_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long vg = plan[0], v0 = plan[1];
  const bool trivial = v0 < 0 || v0 == vg;
  const bool cached = !trivial && tree_key && *tree_key == v0;
  plan[2] = (!trivial && !cached) ? 1 : 0;
  plan[3] = cached ? 1 : 0;
  plan[5] = 0;  // tight in-edges listed by k_parent_dist
  if (plan[2] && tree_key) *tree_key = v0;  // the tree built below is the cache from now on
}

// mode 3 (k_bf_async): in-queue flags (stamp) 0 but v0, ring queue slot 0 = v0 + 1 (qa holds
//   the Q ring slots, zeroed by the caller), 64-bit head / tail / pending counters in counts;
// mode 1 (k_bf_persistent): stamps -1 but v0, frontier queue = [v0], counts = {1, 0, ...};
// mode 2 (k_bf_scan): prev = dist, frontier queue = [v0], counts = {1, 0, ...}.
__global__ void k_init_tree(long long V, const long long* __restrict__ plan, int mode,
                            unsigned long long* __restrict__ dist, unsigned long long* __restrict__ prev,
                            int* __restrict__ stamp, int* __restrict__ parent, unsigned long long* __restrict__ pd,
                            int* __restrict__ counts, int* __restrict__ qa) {
  BZG_PDL_ENTRY();
  if (!plan[2]) return;
  const long long v0 = plan[1];
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (mode == 3) {
    unsigned long long* c64 = reinterpret_cast<unsigned long long*>(counts);
    if (i == 0) { c64[0] = 0; c64[1] = 1; c64[2] = 1; c64[3] = 0; qa[0] = (int)v0 + 1; }  // head, tail, pending
  } else {
    if (i < 8) counts[i] = (i == 0) ? 1 : 0;
    if (i == 0 && mode != 0) qa[0] = (int)v0;
  }
  if (i >= V) return;
  const unsigned long long d = i == v0 ? 0ull : kInfBits;
  dist[i] = d;
  if (mode == 1) stamp[i] = i == v0 ? 0 : -1;
  if (mode == 3) stamp[i] = i == v0 ? 1 : 0;
  if (mode == 2) prev[i] = d;
  parent[i] = 0x7fffffff;
  pd[i] = ~0ull;
}

// Bellman-Ford without barriers: the same fixed point by asynchronous relaxation.  A ring queue
// of vertices whose distance dropped (each at most once at a time: the in-queue flag), one warp
// per popped vertex relaxing its alive out-edges with returning atomicMin, improved targets
// pushed back (warp-aggregated); `pending` counts pushed-but-unfinished items, and the kernel
// ends when it reaches zero.  Relaxation order does not matter: every d[v] only ever decreases
// to min over paths of the left-fold fl sums, which is what the sweeps reach too.
// Ordering: a popper clears the flag, fences, then reads d[v]; a pusher lowers d[w], fences,
// then tests the flag -- so a drop after the read always re-enqueues the vertex.
__global__ void k_bf_async(long long V, const long long* __restrict__ row_ptr, const int* __restrict__ dst,
                           const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                           unsigned long long* __restrict__ dist, int* __restrict__ inq, int* __restrict__ ring,
                           unsigned long long* __restrict__ ctr, long long Q, const long long* __restrict__ plan) {
  BZG_PDL_ENTRY();
  if (!plan[2]) return;
  const int lane = threadIdx.x & 31;
  volatile int* vring = ring;
  volatile unsigned long long* vpend = ctr + 2;
  while (true) {
    unsigned long long h = 0;
    if (lane == 0) h = atomicAdd(ctr + 0, 1ull);
    h = __shfl_sync(0xffffffffu, h, 0);
    const long long slot = (long long)(h % (unsigned long long)Q);
    int v = -1;
    while (true) {  // wait for index h to be published, or for the end
      int sv = 0;
      if (lane == 0) sv = vring[slot];
      sv = __shfl_sync(0xffffffffu, sv, 0);
      if (sv != 0) { v = sv - 1; break; }
      unsigned long long pd = 0;
      if (lane == 0) pd = *vpend;
      pd = __shfl_sync(0xffffffffu, pd, 0);
      if (pd == 0) return;
      __nanosleep(64);
    }
    if (lane == 0) {
      vring[slot] = 0;
      atomicExch(inq + v, 0);
      __threadfence();
    }
    __syncwarp();
    const double du = __longlong_as_double((long long)atomicAdd(dist + v, 0ull));
    const long long e1 = row_ptr[v + 1];
    for (long long e = row_ptr[v] + lane; e - lane < e1; e += 32) {
      bool push = false;
      int w = 0;
      if (e < e1 && (!alive || alive[e])) {
        w = dst[e];
        const unsigned long long nb = dbits(__dadd_rn(du, cost[e]));
        if (nb < __ldcg(dist + w)) {
          const unsigned long long old = atomicMin(dist + w, nb);
          if (nb < old) {
            __threadfence();
            push = atomicExch(inq + w, 1) == 0;
          }
        }
      }
      const unsigned want = __ballot_sync(0xffffffffu, push);
      if (want) {
        const int leader = __ffs(want) - 1;
        unsigned long long base = 0;
        if (lane == leader) {
          atomicAdd(ctr + 2, (unsigned long long)__popc(want));  // pending first, then publish
          base = atomicAdd(ctr + 1, (unsigned long long)__popc(want));
        }
        base = __shfl_sync(0xffffffffu, base, leader);
        if (push) {
          const unsigned long long t = base + __popc(want & ((1u << lane) - 1u));
          vring[(long long)(t % (unsigned long long)Q)] = w + 1;
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicAdd(ctr + 2, ~0ull);  // this item is done (-1)
    }
  }
}

// parent[v] = argmin (d[u], u) over alive in-edges with fl(d[u] + c) == d[v] (two passes):
// the first takes the min d[u] per v over the tight in-edges and lists those edges (about one
// per reached vertex), the second picks the min u among the listed edges with d[u] == that
// minimum -- all E edges again only if the list overflowed its capacity.
__global__ void k_parent_dist(long long E, const int* __restrict__ src, const int* __restrict__ dst,
                              const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                              const unsigned long long* __restrict__ dist, unsigned long long* __restrict__ pd,
                              const long long* __restrict__ plan, const long long* __restrict__ dE,
                              int* __restrict__ tight, unsigned long long* __restrict__ n_tight, long long cap) {
  BZG_PDL_ENTRY();
  if (dE) E = min(E, *dE);
  if (plan && !plan[2]) return;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  if (alive && !alive[e]) return;
  const int u = src[e], v = dst[e];
  const unsigned long long bu = dist[u];
  if (bu >= kInfBits) return;
  const double nd = __dadd_rn(__longlong_as_double((long long)bu), cost[e]);
  if (dbits(nd) == dist[v]) {
    atomicMin(pd + v, bu);
    const unsigned long long k = atomicAdd(n_tight, 1ull);
    if ((long long)k < cap) tight[k] = (int)e;
  }
}

__device__ __forceinline__ void parent_edge(long long e, const int* __restrict__ src, const int* __restrict__ dst,
                                            const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                                            const unsigned long long* __restrict__ dist,
                                            const unsigned long long* __restrict__ pd, int* __restrict__ parent) {
  if (alive && !alive[e]) return;
  const int u = src[e], v = dst[e];
  const unsigned long long bu = dist[u];
  if (bu >= kInfBits || bu != pd[v]) return;
  const double nd = __dadd_rn(__longlong_as_double((long long)bu), cost[e]);
  if (dbits(nd) == dist[v]) atomicMin(parent + v, u);
}

__global__ void k_parent_idx(long long E, const int* __restrict__ src, const int* __restrict__ dst,
                             const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                             const unsigned long long* __restrict__ dist, const unsigned long long* __restrict__ pd,
                             int* __restrict__ parent, const long long* __restrict__ plan,
                             const long long* __restrict__ dE, const int* __restrict__ tight,
                             const unsigned long long* __restrict__ n_tight, long long cap) {
  BZG_PDL_ENTRY();
  if (dE) E = min(E, *dE);
  if (plan && !plan[2]) return;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const long long n = (long long)*n_tight;
  if (n <= cap) {
    for (long long k = tid; k < n; k += nt) parent_edge(tight[k], src, dst, cost, alive, dist, pd, parent);
  } else {  // the list overflowed: every edge
    for (long long e = tid; e < E; e += nt) parent_edge(e, src, dst, cost, alive, dist, pd, parent);
  }
}

// out[0] = path length (-1: None), out[1] = dist bits, out[2..] = the path from v0 to vg
__global__ void k_backtrack(long long V, const long long* __restrict__ plan, const int* __restrict__ parent,
                            const unsigned long long* __restrict__ dist, long long* __restrict__ out) {
  BZG_PDL_ENTRY();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const long long vg = plan[0], v0 = plan[1];
  long long* path = out + 2;
  if (v0 < 0) { out[0] = -1; return; }
  if (v0 == vg) { out[0] = 1; out[1] = 0; path[0] = v0; return; }
  if (dist[vg] >= kInfBits) { out[0] = -1; return; }
  long long n = 0, v = vg;
  path[n++] = v;
  while (v != v0 && n <= V) {
    v = parent[v];
    if (v < 0 || v >= V) { n = -2; break; }
    path[n++] = v;
  }
  if (n > 0)
    for (long long a = 0, b = n - 1; a < b; ++a, --b) {  // vg .. v0 -> v0 .. vg
      const long long t = path[a];
      path[a] = path[b];
      path[b] = t;
    }
  out[0] = n;
  out[1] = (long long)dist[vg];
}

size_t bf_cluster_smem(long long chunk) { return (size_t)chunk * (sizeof(unsigned long long) + sizeof(int)); }

// cluster size for k_bf_cluster on V vertices: the smallest of 1, 2, 4, 8, 16 whose slice fits
// the shared memory (16 needs the non-portable cluster size) -- small clusters for small graphs,
// fewer CTAs to synchronise; 0 when V is too large or the device refuses the configuration
int bf_cluster_size(long long V) {
  if (V > kBfClusterMaxV) return 0;
  const long long per_cta = 192 * 1024 / (sizeof(unsigned long long) + sizeof(int));
  static int max_size = -1;
  if (max_size < 0) {  // 16 CTAs at the largest slice, if the device schedules such a cluster
    max_size = 8;
    if (cudaFuncSetAttribute((const void*)k_bf_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess &&
        cudaFuncSetAttribute((const void*)k_bf_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)bf_cluster_smem(per_cta)) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(16);
      cfg.blockDim = dim3(kBfClusterThreads);
      cfg.dynamicSmemBytes = bf_cluster_smem(per_cta);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 16;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (const void*)k_bf_cluster, &cfg) == cudaSuccess && n > 0) max_size = 16;
    }
    cudaGetLastError();
  }
  const int env = std::getenv("BZG_BF_CLUSTER") ? std::atoi(std::getenv("BZG_BF_CLUSTER")) : 0;  // per call
  int cs = env > 0 ? env : 16;
  // default: 16 CTAs (the relaxation streams the edges through 16 SMs)
  if (div_up(V, cs) > per_cta) return 0;
  return cs <= max_size ? cs : 0;
}

// k_snap over the vertices, the result (first argmin index, -1 if none) written to *out
void snap_launch(Ctx* c, Graph* g, const SnapParams& sp, const SnapParams* spd, const uint8_t* reach, DevBuf& best,
                 long long* out) {
  const long long V = g->V;
  const unsigned nb = div_up(V, 256);
  best.alloc((1 + 2 * (size_t)nb) * sizeof(unsigned long long), c->stream);
  launch(c, "k_fill_best", k_fill_u64, dim3(1), dim3(32), 0, best.as<unsigned long long>(), 1ll, kInfBits + 2);
  launch(c, "k_snap", k_snap, dim3(nb), dim3(256), 0, sp, spd, g->vertices.as<double>(), V, reach,
         best.as<unsigned long long>());
  launch(c, "k_snap_final", k_snap_final, dim3(1), dim3(32), 0, best.as<unsigned long long>(), (int)nb, out);
}

constexpr long long kHead = 510;  // path entries in the first read-back

// goal (mode 0) and start (mode 1 tube / 2 reach) snapping parameters of one search
void snap_params(const Graph* g, const double* start, const double* goal, const double* tube_lo,
                 const double* tube_hi, double eps, int pos_only, int require_tube, SnapParams sp[2]) {
  const int n = g->n;
  for (int j = 0; j < 2; ++j) {
    sp[j] = SnapParams{};
    sp[j].n = n;
    sp[j].m_norm = pos_only ? g->m : n;
  }
  for (int k = 0; k < n; ++k) {
    sp[0].target[k] = goal[k];
    sp[1].target[k] = start[k];
    sp[1].tlo[k] = -tube_hi[k] - eps;  // (diff >= -tube.hi - EPS_GEO)   graph.py:381
    sp[1].thi[k] = -tube_lo[k] + eps;  // (diff <= -tube.lo + EPS_GEO)
  }
  sp[0].mode = 0;
  sp[1].mode = require_tube ? 1 : 2;
}

// Enqueue one search on c->stream: snapping, the shortest-path tree (skipped on the device when
// cached or trivial), parents, backtrack, and the read-back of the first kHead + 2 entries of
// [len, dist bits, path...] into h_out (pinned).  Every buffer comes from c->ws or the mask, so
// the same sequence can be captured (bzg_query).  h_sp (pinned, 2 SnapParams) non-null: the
// snapping parameters are copied to the device and read there instead of sp.
void path_enqueue(Ctx* c, Graph* g, Mask* mk, const SnapParams sp[2], const SnapParams* h_sp, long long* h_out) {
  const long long V = g->V, E = g->E;
  const uint8_t* alive = mk ? mk->alive.as<uint8_t>() : nullptr;
  DevBuf& d_plan = c->ws[WS_PLAN];
  d_plan.alloc(8 * sizeof(long long), c->stream);
  long long* plan = d_plan.as<long long>();
  const SnapParams* spd = nullptr;
  if (h_sp) {
    DevBuf& d_sp = c->ws[WS_SNAP];
    d_sp.alloc(2 * sizeof(SnapParams), c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(d_sp.ptr, h_sp, 2 * sizeof(SnapParams), cudaMemcpyHostToDevice, c->stream));
    spd = d_sp.as<SnapParams>();
  }
  const bool small = V <= kSnapBlockV && !std::getenv("BZG_SNAP_GRID");  // (tests compare both)
  if (small) {  // goal and, for tube snapping, the start in one launch of one block each
    launch(c, "k_snap_block", k_snap_block, dim3(sp[1].mode == 1 ? 2 : 1), dim3(1024), 0, sp[0], sp[1], spd, 0,
           g->vertices.as<double>(), V, (const uint8_t*)nullptr, plan);
  } else {
    snap_launch(c, g, sp[0], spd, nullptr, c->ws[WS_BEST0], plan + 0);
  }

  if (sp[1].mode == 1) {
    if (!small) snap_launch(c, g, sp[1], spd ? spd + 1 : nullptr, nullptr, c->ws[WS_BEST1], plan + 1);
  } else {
    // relaxed mid-run snap: nearest vertex that can still reach vg (graph.py:388-392); the
    // reverse reachability runs on the device (k_reach_coop), cached per (mask, vg) there
    uint8_t* reach;
    long long* rkey;
    if (mk) {
      mk->reach.alloc(V, c->stream);
      reach = mk->reach.as<uint8_t>();
      if (!mk->reach_key.ptr) {
        mk->reach_key.alloc(sizeof(long long), c->stream);
        BZG_CHECK_CUDA(cudaMemsetAsync(mk->reach_key.ptr, 0xFF, sizeof(long long), c->stream));
      }
      rkey = mk->reach_key.as<long long>();
    } else {  // no mask, no cache: the key is reset every search
      DevBuf &t_reach = c->ws[WS_NM_REACH], &t_key = c->ws[WS_NM_KEY];
      t_reach.alloc(V, c->stream);
      reach = t_reach.as<uint8_t>();
      t_key.alloc(sizeof(long long), c->stream);
      BZG_CHECK_CUDA(cudaMemsetAsync(t_key.ptr, 0xFF, sizeof(long long), c->stream));
      rkey = t_key.as<long long>();
    }
    DevBuf& rflags = c->ws[WS_REACH_FLAGS];
    rflags.alloc(4 * sizeof(int), c->stream);
    long long El = E, Vl2 = V;
    const long long* dEp = g->dE;
    const int* rs = g->src.as<int>();
    const int* rd = g->dst.as<int>();
    const long long* cpl = plan;
    int* rf = rflags.as<int>();
    // small graphs: one cluster (BZG_REACH_IMPL=grid|cluster forces a schedule)
    const char* re = std::getenv("BZG_REACH_IMPL");
    const std::string rs_env = re ? std::string(re) : std::string();
    const int rcs = bf_cluster_size(V) > 0 ? (E <= kBfCtaMaxE ? 1 : 16) : 0;
    const bool rcl = rcs > 0 && (rs_env == "cluster" || (rs_env.empty() && V <= kBfClusterDefaultV &&
                                                         E <= kBfClusterDefaultE));
    // larger graphs: the bottom-up pull (BZG_REACH_IMPL=grid: the edge sweeps)
    if (!rcl && rs_env != "grid") {
      const long long* fp = g->row_ptr.as<long long>();
      static int pull_per_sm = 0;
      if (!pull_per_sm)
        BZG_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pull_per_sm, (const void*)k_reach_pull, 256, 0));
      const int pblocks = std::max(1, std::min(pull_per_sm, 4) * c->num_sms);
      void* args[] = {&Vl2, &fp, &rd, &alive, &reach, &rkey, &cpl, &rf, &dEp};
      launch_coop(c, "k_reach_pull", (const void*)k_reach_pull, dim3(pblocks), dim3(256), args);
    } else if (rcl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(rcs);
      cfg.blockDim = dim3(1024);
      cfg.stream = c->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = rcs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      static bool attr_set = false;
      if (!attr_set) {
        BZG_CHECK_CUDA(cudaFuncSetAttribute((const void*)k_reach_sweeps<false>,
                                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_set = true;
      }
      cudaEvent_t ea = nullptr;
      const bool timed = c->timed("k_reach_cluster");
      if (timed) { ea = c->take_event(); BZG_CHECK_CUDA(cudaEventRecord(ea, c->stream)); }
      BZG_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_reach_sweeps<false>, El, Vl2, rs, rd, alive, reach, rkey, cpl, rf, dEp));
      c->launches++;
      if (timed) {
        cudaEvent_t eb = c->take_event();
        BZG_CHECK_CUDA(cudaEventRecord(eb, c->stream));
        c->pending.push_back({"k_reach_cluster", ea, eb});
      }
    } else {
      int per_sm = 0;
      BZG_CHECK_CUDA(
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_reach_sweeps<true>, 256, 0));
      const int rblocks = std::max(1, std::min(per_sm, 2) * c->num_sms);
      void* args[] = {&El, &Vl2, &rs, &rd, &alive, &reach, &rkey, &cpl, &rf, &dEp};
      launch_coop(c, "k_reach_coop", (const void*)k_reach_sweeps<true>, dim3(rblocks), dim3(256), args);
    }
    if (small)
      launch(c, "k_snap_block", k_snap_block, dim3(1), dim3(1024), 0, sp[0], sp[1], spd, 1, g->vertices.as<double>(), V,
             (const uint8_t*)reach, plan + 1);
    else
      snap_launch(c, g, sp[1], spd ? spd + 1 : nullptr, reach, c->ws[WS_BEST1], plan + 1);
  }

  // ---- the shortest-path tree from v0 (skipped on the device when cached or trivial)
  unsigned long long* dist;
  int* parent;
  long long* key = nullptr;
  if (mk) {
    if (mk->dist.bytes < (size_t)V * sizeof(unsigned long long)) mk->tree_key.release();
    mk->dist.alloc(V * sizeof(unsigned long long), c->stream);
    mk->parent.alloc(V * sizeof(int), c->stream);
    if (!mk->tree_key.ptr) {
      mk->tree_key.alloc(sizeof(long long), c->stream);
      BZG_CHECK_CUDA(cudaMemsetAsync(mk->tree_key.ptr, 0xFF, sizeof(long long), c->stream));  // -1: no tree
    }
    dist = mk->dist.as<unsigned long long>();
    parent = mk->parent.as<int>();
    key = mk->tree_key.as<long long>();
  } else {
    DevBuf &t_dist = c->ws[WS_NM_DIST], &t_parent = c->ws[WS_NM_PARENT];
    t_dist.alloc(V * sizeof(unsigned long long), c->stream);
    t_parent.alloc(V * sizeof(int), c->stream);
    dist = t_dist.as<unsigned long long>();
    parent = t_parent.as<int>();
  }
  launch(c, "k_plan", k_plan, dim3(1), dim3(32), 0, plan, key);
  DevBuf &t_prev = c->ws[WS_SSSP_PREV], &t_pd = c->ws[WS_SSSP_PD], &t_aux = c->ws[WS_SSSP_AUX];
  t_prev.alloc(std::max(V, 1ll) * sizeof(unsigned long long), c->stream);
  t_pd.alloc(std::max(V, 1ll) * sizeof(unsigned long long), c->stream);
  // BZG_BF_IMPL=queue|scan|async: k_bf_persistent (frontier queue, returning atomics), k_bf_scan
  // (fire-and-forget relaxation + rescan, two barriers per sweep) or k_bf_async (no barriers).
  const char* bf_env = std::getenv("BZG_BF_IMPL");
  const std::string bfs = bf_env ? std::string(bf_env) : std::string();
  // default: the rescan variant (cfg2 0.086 ms vs queue 0.098, cfg3 0.20 vs 0.30, cfg5 100k 0.80
  // vs 1.17); the queue for tiny graphs.  The barrier-free k_bf_async reaches the same fixed
  // point but re-relaxes far more (cfg3 0.46 ms, cfg5 100k 2.7 ms), and a one-barrier rescan
  // (relax the last frontier and rescan without waiting) measured the same as two barriers
  // (cfg3 0.201 vs 0.208 ms): the sweeps are bound by their dependent loads.
  // tiny graphs: one block in shared memory (k_bf_cta); graphs up to kBfClusterDefaultV: one
  // cluster (k_bf_cluster); larger: the grid-wide rescan (k_bf_scan)
  const int cl_size = bf_cluster_size(V);
  const bool cta_ok = V <= kBfCtaMaxV && E <= kBfCtaMaxE;
  const int mode = bfs == "queue" ? 1
                   : bfs == "scan" ? 2
                   : bfs == "async" ? 3
                   : bfs == "cta" && cta_ok ? 5
                   : bfs == "cluster" && cl_size > 0 ? 4
                   : !bfs.empty() ? 2
                   : cta_ok ? 5
                   : cl_size > 0 && V <= kBfClusterDefaultV && E <= kBfClusterDefaultE ? 4
                   : 2;
  const long long Q = V + 8192 + 64;  // ring: <= V queued (flags) + claimed-unread (one per warp)
  // aux: counts (8 ints) | stamp (V ints) | qa (V ints) | qb (V ints); async: counts | stamp | ring
  if (mode == 3)
    t_aux.alloc((8 + (size_t)std::max(V, 1ll) + (size_t)Q) * sizeof(int), c->stream);
  else
    t_aux.alloc((8 + 3 * (size_t)std::max(V, 1ll)) * sizeof(int), c->stream);
  int* counts = t_aux.as<int>();
  int* stamp = counts + 8;
  int* qa = stamp + V;
  int* qb = qa + V;
  if (mode == 3) BZG_CHECK_CUDA(cudaMemsetAsync(qa, 0, (size_t)Q * sizeof(int), c->stream));
  launch(c, "k_init_tree", k_init_tree, dim3(div_up(std::max(V, 8ll), 256)), dim3(256), 0, V, (const long long*)plan,
         mode, dist, t_prev.as<unsigned long long>(), stamp, parent, t_pd.as<unsigned long long>(), counts, qa);
  const void* bf_kern = mode == 1 ? (const void*)k_bf_persistent
                                  : (mode == 3 ? (const void*)k_bf_async : (const void*)k_bf_scan);
  int per_sm = 0;
  if (mode != 4) BZG_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bf_kern, 256, 0));
  static const int bf_per_sm_env =
      std::getenv("BZG_BF_BLOCKS_PER_SM") ? std::atoi(std::getenv("BZG_BF_BLOCKS_PER_SM")) : 0;
  // blocks per SM: fewer blocks make the grid barriers cheaper, more hide the relax latency
  // (scan: cfg3 0.228 / 0.208 ms at 4 / 2 per SM; cfg5 100k 0.79 / 0.86)
  const int want_per_sm = bf_per_sm_env > 0 ? bf_per_sm_env : (V < 50000 ? 2 : 4);
  const int blocks = std::max(1, std::min(per_sm, want_per_sm) * c->num_sms);
  long long Vl = V;
  const long long* rp = g->row_ptr.as<long long>();
  const int* dd = g->dst.as<int>();
  const double* cc = g->cost.as<double>();
  unsigned long long* pv = t_prev.as<unsigned long long>();
  int maxs = (int)std::min<long long>(V + 2, 1 << 30);
  const long long* cplan = plan;
  if (mode == 5) {
    const size_t smem = (size_t)V * (sizeof(unsigned long long) + 3 * sizeof(int));
    ensure_dyn_smem((const void*)k_bf_cta, smem);
    launch(c, "k_bf_cta", k_bf_cta, dim3(1), dim3(kBfCtaThreads), smem, Vl, rp, dd, cc, alive, dist, counts, maxs,
           cplan);
  } else if (mode == 4) {
    const long long chunk = div_up(V, cl_size);
    const size_t smem = bf_cluster_smem(chunk);
    ensure_dyn_smem((const void*)k_bf_cluster, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl_size);
    cfg.blockDim = dim3(kBfClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl_size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t ea = nullptr;
    const bool timed = c->timed("k_bf_cluster");
    if (timed) { ea = c->take_event(); BZG_CHECK_CUDA(cudaEventRecord(ea, c->stream)); }
    BZG_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_bf_cluster, Vl, chunk, rp, dd, cc, alive, dist, counts, maxs, cplan));
    c->launches++;
    if (timed) {
      cudaEvent_t eb = c->take_event();
      BZG_CHECK_CUDA(cudaEventRecord(eb, c->stream));
      c->pending.push_back({"k_bf_cluster", ea, eb});
    }
  } else if (mode == 1) {
    void* args[] = {&Vl, &rp, &dd, &cc, &alive, &dist, &stamp, &qa, &qb, &counts, &maxs, &cplan};
    launch_coop(c, "k_bf_persistent", bf_kern, dim3(blocks), dim3(256), args);
  } else if (mode == 3) {
    launch(c, "k_bf_async", k_bf_async, dim3(blocks), dim3(256), 0, Vl, rp, dd, cc, alive, dist, stamp, qa,
           reinterpret_cast<unsigned long long*>(counts), Q, cplan);
  } else {
    void* args[] = {&Vl, &rp, &dd, &cc, &alive, &dist, &pv, &qa, &qb, &counts, &maxs, &cplan};
    launch_coop(c, "k_bf_scan", bf_kern, dim3(blocks), dim3(256), args);
  }
  if (c->trace_on && !g_capturing) {
    int hc[8];
    long long hp[4];
    BZG_CHECK_CUDA(cudaMemcpyAsync(hc, counts, sizeof(hc), cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(hp, plan, sizeof(hp), cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
    std::fprintf(stderr, "[bzg path] vg %lld v0 %lld build %lld cached %lld; Bellman-Ford sweeps %d (V = %lld)\n",
                 hp[0], hp[1], hp[2], hp[3], hc[3], V);
  }
  // tight in-edge list (counter plan[5], zeroed by k_plan): ~one entry per reached vertex
  const long long tcap = std::max(1ll, std::min(E, 2 * V + 1024));
  DevBuf& t_tight = c->ws[WS_TIGHT];
  t_tight.alloc(tcap * sizeof(int), c->stream);
  unsigned long long* n_tight = reinterpret_cast<unsigned long long*>(plan + 5);
  launch(c, "k_parent_dist", k_parent_dist, dim3(div_up(std::max(E, 1ll), 256)), dim3(256), 0, E, g->src.as<int>(),
         g->dst.as<int>(), g->cost.as<double>(), alive, (const unsigned long long*)dist, t_pd.as<unsigned long long>(),
         cplan, (const long long*)g->dE, t_tight.as<int>(), n_tight, tcap);
  launch(c, "k_parent_idx", k_parent_idx,
         dim3((unsigned)std::min<long long>(div_up(std::max(E, 1ll), 256), 8ll * c->num_sms)), dim3(256), 0, E,
         g->src.as<int>(), g->dst.as<int>(), g->cost.as<double>(), alive, (const unsigned long long*)dist,
         (const unsigned long long*)t_pd.as<unsigned long long>(), parent, cplan, (const long long*)g->dE,
         (const int*)t_tight.as<int>(), (const unsigned long long*)n_tight, tcap);

  // ---- backtrack and the single read-back: [len, dist bits, path...], the first kHead entries
  DevBuf& d_out = c->ws[WS_SSSP_OUT];
  d_out.alloc((V + 3) * sizeof(long long), c->stream);
  launch(c, "k_backtrack", k_backtrack, dim3(1), dim3(32), 0, V, cplan, (const int*)parent,
         (const unsigned long long*)dist, d_out.as<long long>());
  const long long head = std::min<long long>(V + 2, kHead + 2);
  BZG_CHECK_CUDA(cudaMemcpyAsync(h_out, d_out.ptr, head * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
}

// After the stream reached the read-back: the path (empty: None) and its distance; a path
// longer than the head is completed from d_out with a second copy.
void path_collect(Ctx* c, const Graph* g, const long long* h, const long long* d_out, std::vector<int64_t>& path,
                  double* dist_out) {
  path.clear();
  *dist_out = INFINITY;
  const long long head = std::min<long long>(g->V + 2, kHead + 2);
  const long long len = h[0];
  BZG_REQUIRE(len != -2, BZG_ECUDA, "parent chain broken during backtrack");
  if (len < 0) return;  // no snappable start or vg unreachable -> None
  double dv;
  memcpy(&dv, h + 1, sizeof(double));
  path.assign(h + 2, h + 2 + std::min(len, head - 2));
  if (len > head - 2) {  // long path: the rest in a second copy
    path.resize(len);
    BZG_CHECK_CUDA(cudaMemcpyAsync(path.data() + (head - 2), d_out + head, (len - (head - 2)) * sizeof(long long),
                                   cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  }
  *dist_out = dv;
}

}  // namespace

// One host synchronisation per search (the path read-back).  (vg, v0) stay on the device
// (plan); the tree kernels skip themselves when the mask's cached shortest-path tree already
// belongs to v0 (cfg4 goal updates) or the answer is trivial.  Relaxed snapping computes the
// reverse reachability to vg on the device (cached per (mask, vg)).
void find_path(Ctx* c, Graph* g, Mask* mk, const double* start, const double* goal, const double* tube_lo,
               const double* tube_hi, double eps, int pos_only, int require_tube, std::vector<int64_t>& path,
               double* dist_out) {
  BZG_REQUIRE(g->n <= 16, BZG_EUNSUPPORTED, "state dimension too large");
  BZG_REQUIRE(g->V >= 1, BZG_EINVAL, "graph has no vertices");
  SnapParams sp[2];
  snap_params(g, start, goal, tube_lo, tube_hi, eps, pos_only, require_tube, sp);
  long long* h = static_cast<long long*>(c->host_scratch((size_t)(kHead + 2) * sizeof(long long)));
  path_enqueue(c, g, mk, sp, nullptr, h);
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  path_collect(c, g, h, c->ws[WS_SSSP_OUT].as<long long>(), path, dist_out);
}

// ---- PathStage: the search with start/goal in pinned staging (capturable enqueue)
struct PathStage {
  int pos_only = 0, require_tube = 0;
  double eps = 0.0;
  std::vector<double> tube_lo, tube_hi;
  SnapParams* h_sp = nullptr;  // pinned: [goal, start] parameters, read by the enqueued H2D copy
  long long* h_out = nullptr;  // pinned: the head of the read-back
};

PathStage* path_stage_create(const Graph* g, const double* tube_lo, const double* tube_hi, double eps, int pos_only,
                             int require_tube) {
  BZG_REQUIRE(g->n <= 16, BZG_EUNSUPPORTED, "state dimension too large");
  BZG_REQUIRE(g->V >= 1, BZG_EINVAL, "graph has no vertices");
  PathStage* s = new PathStage();
  s->pos_only = pos_only;
  s->require_tube = require_tube;
  s->eps = eps;
  s->tube_lo.assign(tube_lo, tube_lo + g->n);
  s->tube_hi.assign(tube_hi, tube_hi + g->n);
  if (cudaMallocHost(&s->h_sp, 2 * sizeof(SnapParams)) != cudaSuccess ||
      cudaMallocHost(&s->h_out, (size_t)(kHead + 2) * sizeof(long long)) != cudaSuccess) {
    path_stage_destroy(s);
    throw Error(BZG_ECUDA, "pinned staging allocation failed");
  }
  std::vector<double> zero(g->n, 0.0);
  path_stage_set(s, g, zero.data(), zero.data());
  return s;
}

// (the caller guarantees that no launch reading the staging is still pending)
void path_stage_set(PathStage* s, const Graph* g, const double* start, const double* goal) {
  snap_params(g, start, goal, s->tube_lo.data(), s->tube_hi.data(), s->eps, s->pos_only, s->require_tube, s->h_sp);
}

void path_stage_enqueue(Ctx* c, Graph* g, Mask* mk, PathStage* s) { path_enqueue(c, g, mk, s->h_sp, s->h_sp, s->h_out); }

void path_stage_collect(Ctx* c, const Graph* g, PathStage* s, std::vector<int64_t>& path, double* dist) {
  path_collect(c, g, s->h_out, c->ws[WS_SSSP_OUT].as<long long>(), path, dist);
}

void path_stage_destroy(PathStage* s) {
  if (!s) return;
  if (s->h_sp) cudaFreeHost(s->h_sp);
  if (s->h_out) cudaFreeHost(s->h_out);
  delete s;
}

// ---- bzg_query: the search above captured once per (graph, mask, snapping options)
struct Query {
  Ctx* c = nullptr;
  Graph* g = nullptr;
  Mask* mk = nullptr;
  uint64_t version = 0;
  int64_t E = 0;
  PathStage* st = nullptr;
  DevBuf ws[kWsSlots];  // the query's own workspaces (the graph reads their addresses)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long kernels = 0;  // kernel nodes per launch
};

void query_destroy(Query* q) {
  if (!q) return;
  if (q->c) cudaStreamSynchronize(q->c->stream);
  if (q->exec) cudaGraphExecDestroy(q->exec);
  if (q->graph) cudaGraphDestroy(q->graph);
  for (auto& w : q->ws) w.release();
  path_stage_destroy(q->st);
  delete q;
}

Query* query_create(Ctx* c, Graph* g, Mask* mk, const double* tube_lo, const double* tube_hi, double eps,
                    int pos_only, int require_tube) {
  Query* q = new Query();
  try {
    q->c = c;
    q->g = g;
    q->mk = mk;
    q->version = g->version;
    q->E = g->E;
    q->st = path_stage_create(g, tube_lo, tube_hi, eps, pos_only, require_tube);
    // warm-up: one eager search sizes every workspace and initialises the mask's cache keys
    with_ws(c, q->ws, [&] {
      path_stage_enqueue(c, g, mk, q->st);
      BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
      q->exec = capture_graph(c, [&] { path_stage_enqueue(c, g, mk, q->st); }, &q->kernels, &q->graph);
    });
  } catch (...) {
    query_destroy(q);
    throw;
  }
  return q;
}

void query_run(Query* q, const double* start, const double* goal, std::vector<int64_t>& path, double* dist) {
  Ctx* c = q->c;
  Graph* g = q->g;
  BZG_REQUIRE(g->version == q->version && g->E == q->E && (!q->mk || (q->mk->g == g && q->mk->E == g->E)),
              BZG_EINVAL, "stale query: the graph's edge set changed after it was captured");
  path_stage_set(q->st, g, start, goal);  // the previous launch finished (query_run synchronises)
  BZG_CHECK_CUDA(cudaGraphLaunch(q->exec, c->stream));
  c->launches += q->kernels;
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  with_ws(c, q->ws, [&] { path_stage_collect(c, g, q->st, path, dist); });
}

long long query_kernels(const Query* q) { return q->kernels; }
Ctx* query_ctx(const Query* q) { return q->c; }

}  // namespace bzg
