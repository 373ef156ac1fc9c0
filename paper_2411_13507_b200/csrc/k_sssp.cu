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
__global__ void k_snap(SnapParams sp, const double* __restrict__ Vx, long long V, const uint8_t* __restrict__ reach,
                       unsigned long long* __restrict__ best) {
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

// reverse reachability sweep over alive edges: reach[u] |= reach[v] for u -> v
__global__ void k_reach_sweep(long long E, const int* __restrict__ src, const int* __restrict__ dst,
                              const uint8_t* __restrict__ alive, uint8_t* __restrict__ reach, int* __restrict__ changed) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  if (alive && !alive[e]) return;
  const int v = dst[e];
  if (!reach[v]) return;
  const int u = src[e];
  if (!reach[u]) {
    reach[u] = 1;
    *changed = 1;
  }
}

// Frontier Bellman-Ford as one persistent cooperative kernel: a queue of the vertices
// improved in the previous sweep (each enqueued once per sweep through its stamp); one warp
// per queued vertex relaxes its alive out-edges with fl(d[u] + c) and atomicMin on the
// (non-negative) double bits; grid-wide barriers between sweeps; stops when a sweep improves
// nothing.  No host round trip per sweep.
__global__ void k_bf_persistent(long long V, const long long* __restrict__ row_ptr, const int* __restrict__ dst,
                                const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                                unsigned long long* __restrict__ dist, int* __restrict__ stamp, int* __restrict__ qa,
                                int* __restrict__ qb, int* __restrict__ counts, int max_sweeps) {
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
                          int* __restrict__ qa, int* __restrict__ qb, int* __restrict__ counts, int max_sweeps) {
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

// parent[v] = argmin (d[u], u) over alive in-edges with fl(d[u] + c) == d[v] (two passes)
__global__ void k_parent_dist(long long E, const int* __restrict__ src, const int* __restrict__ dst,
                              const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                              const unsigned long long* __restrict__ dist, unsigned long long* __restrict__ pd) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  if (alive && !alive[e]) return;
  const int u = src[e], v = dst[e];
  const unsigned long long bu = dist[u];
  if (bu >= kInfBits) return;
  const double nd = __dadd_rn(__longlong_as_double((long long)bu), cost[e]);
  if (dbits(nd) == dist[v]) atomicMin(pd + v, bu);
}

__global__ void k_parent_idx(long long E, const int* __restrict__ src, const int* __restrict__ dst,
                             const double* __restrict__ cost, const uint8_t* __restrict__ alive,
                             const unsigned long long* __restrict__ dist, const unsigned long long* __restrict__ pd,
                             int* __restrict__ parent) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  if (alive && !alive[e]) return;
  const int u = src[e], v = dst[e];
  const unsigned long long bu = dist[u];
  if (bu >= kInfBits || bu != pd[v]) return;
  const double nd = __dadd_rn(__longlong_as_double((long long)bu), cost[e]);
  if (dbits(nd) == dist[v]) atomicMin(parent + v, u);
}

__global__ void k_backtrack(long long V, long long v0, long long vg, const int* __restrict__ parent,
                            const unsigned long long* __restrict__ dist, long long* __restrict__ path,
                            long long* __restrict__ len, double* __restrict__ dout) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (dist[vg] >= kInfBits) {
    *len = -1;
    return;
  }
  long long n = 0, v = vg;
  path[n++] = v;
  while (v != v0 && n <= V) {
    v = parent[v];
    if (v < 0 || v >= V) { n = -2; break; }
    path[n++] = v;
  }
  *len = n;
  *dout = __longlong_as_double((long long)dist[vg]);
}

__global__ void k_fill_u64(unsigned long long* p, long long n, unsigned long long v) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void k_init_sssp(long long V, long long v0, unsigned long long* dist, int* stamp, int* parent,
                            unsigned long long* pd) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= V) return;
  dist[i] = i == v0 ? 0ull : kInfBits;
  stamp[i] = i == v0 ? 0 : -1;
  parent[i] = 0x7fffffff;
  pd[i] = ~0ull;
}

long long snap_launch(Ctx* c, Graph* g, const SnapParams& sp, const uint8_t* reach) {
  const long long V = g->V;
  const unsigned nb = div_up(V, 256);
  DevBuf best, out;
  best.alloc((1 + 2 * (size_t)nb) * sizeof(unsigned long long), c->stream);
  out.alloc(sizeof(long long), c->stream);
  const unsigned long long init = kInfBits + 2;
  BZG_CHECK_CUDA(cudaMemcpyAsync(best.ptr, &init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
  launch(c, "k_snap", k_snap, dim3(nb), dim3(256), 0, sp, g->vertices.as<double>(), V, reach,
         best.as<unsigned long long>());
  launch(c, "k_snap_final", k_snap_final, dim3(1), dim3(32), 0, best.as<unsigned long long>(), (int)nb,
         out.as<long long>());
  long long* h = static_cast<long long*>(c->host_scratch(sizeof(long long)));
  BZG_CHECK_CUDA(cudaMemcpyAsync(h, out.ptr, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  return h[0];
}

}  // namespace

void find_path(Ctx* c, Graph* g, Mask* mk, const double* start, const double* goal, const double* tube_lo,
               const double* tube_hi, double eps, int pos_only, int require_tube, std::vector<int64_t>& path,
               double* dist_out) {
  const long long V = g->V, E = g->E;
  const int n = g->n;
  BZG_REQUIRE(n <= 16, BZG_EUNSUPPORTED, "state dimension too large");
  const uint8_t* alive = mk ? mk->alive.as<uint8_t>() : nullptr;
  path.clear();
  *dist_out = INFINITY;

  SnapParams sp{};
  sp.n = n;
  sp.m_norm = pos_only ? g->m : n;
  for (int k = 0; k < n; ++k) sp.target[k] = goal[k];
  sp.mode = 0;
  const long long vg = snap_launch(c, g, sp, nullptr);
  BZG_REQUIRE(vg >= 0, BZG_EINVAL, "graph has no vertices");

  for (int k = 0; k < n; ++k) {
    sp.target[k] = start[k];
    sp.tlo[k] = -tube_hi[k] - eps;  // (diff >= -tube.hi - EPS_GEO)   graph.py:381
    sp.thi[k] = -tube_lo[k] + eps;  // (diff <= -tube.lo + EPS_GEO)
  }
  long long v0;
  DevBuf tmp_reach;
  if (require_tube) {
    sp.mode = 1;
    v0 = snap_launch(c, g, sp, nullptr);
  } else {
    // relaxed mid-run snap: nearest vertex that can still reach vg (graph.py:388-392)
    uint8_t* reach;
    if (mk) {
      mk->reach.alloc(V, c->stream);
      reach = mk->reach.as<uint8_t>();
    } else {
      tmp_reach.alloc(V, c->stream);
      reach = tmp_reach.as<uint8_t>();
    }
    if (!mk || mk->reach_vg != vg) {
      DevBuf changed;
      changed.alloc(sizeof(int), c->stream);
      BZG_CHECK_CUDA(cudaMemsetAsync(reach, 0, V, c->stream));
      const uint8_t one = 1;
      BZG_CHECK_CUDA(cudaMemcpyAsync(reach + vg, &one, 1, cudaMemcpyHostToDevice, c->stream));
      int* h = static_cast<int*>(c->host_scratch(sizeof(int)));
      for (int guard = 0;; ++guard) {
        BZG_CHECK_CUDA(cudaMemsetAsync(changed.ptr, 0, sizeof(int), c->stream));
        for (int s = 0; s < 8; ++s)
          launch(c, "k_reach_sweep", k_reach_sweep, dim3(div_up(E, 256)), dim3(256), 0, E, g->src.as<int>(),
                 g->dst.as<int>(), alive, reach, changed.as<int>());
        BZG_CHECK_CUDA(cudaMemcpyAsync(h, changed.ptr, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
        if (!h[0] || E == 0) break;
        BZG_REQUIRE(guard < V + 8, BZG_ECUDA, "reachability sweep did not converge");
      }
      if (mk) mk->reach_vg = vg;
    }
    sp.mode = 2;
    v0 = snap_launch(c, g, sp, reach);
  }
  if (v0 < 0) return;  // no snappable start -> None
  if (v0 == vg) {
    path.push_back(v0);
    *dist_out = 0.0;
    return;
  }

  DevBuf lpath, llen, ldist;
  DevBuf t_dist, t_parent, t_stamp, t_pd, t_last;
  unsigned long long* dist;
  int* parent;
  const bool cached = mk && mk->tree_v0 == v0;
  if (mk) {
    mk->dist.alloc(V * sizeof(unsigned long long), c->stream);
    mk->parent.alloc(V * sizeof(int), c->stream);
    dist = mk->dist.as<unsigned long long>();
    parent = mk->parent.as<int>();
  } else {
    t_dist.alloc(V * sizeof(unsigned long long), c->stream);
    t_parent.alloc(V * sizeof(int), c->stream);
    dist = t_dist.as<unsigned long long>();
    parent = t_parent.as<int>();
  }
  if (!cached) {
    t_stamp.alloc(V * sizeof(int), c->stream);
    t_pd.alloc(V * sizeof(unsigned long long), c->stream);
    t_last.alloc(sizeof(int), c->stream);
    launch(c, "k_init_sssp", k_init_sssp, dim3(div_up(V, 256)), dim3(256), 0, V, v0, dist, t_stamp.as<int>(), parent,
           t_pd.as<unsigned long long>());
    BZG_CHECK_CUDA(cudaMemsetAsync(t_last.ptr, 0, sizeof(int), c->stream));
    // frontier Bellman-Ford in one cooperative launch (all blocks resident)
    DevBuf qa, qb, cnt;
    qa.alloc(std::max(V, 1ll) * sizeof(int), c->stream);
    qb.alloc(std::max(V, 1ll) * sizeof(int), c->stream);
    cnt.alloc(8 * sizeof(int), c->stream);
    const int init[8] = {1, 0, 0, 0, 0, 0, 0, 0};
    const int v0i = (int)v0;
    BZG_CHECK_CUDA(cudaMemcpyAsync(cnt.ptr, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    BZG_CHECK_CUDA(cudaMemcpyAsync(qa.ptr, &v0i, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    // the scan variant's second barrier and V-wide scan cost more than the queue's returning
    // atomics on small graphs (cfg5 10k: 0.22 vs 0.19 ms); from ~16 k vertices it wins
    // (cfg3 0.33 -> 0.24 ms, cfg5 100k 1.18 -> 0.80 ms).  BZG_BF_IMPL=queue|scan overrides.
    static const char* bf_env = std::getenv("BZG_BF_IMPL");
    const bool bf_queue = bf_env ? std::string(bf_env) == "queue" : V < 16384;
    const void* bf_kern = bf_queue ? (const void*)k_bf_persistent : (const void*)k_bf_scan;
    int per_sm = 0;
    BZG_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bf_kern, 256, 0));
    static const int bf_per_sm_env =
        std::getenv("BZG_BF_BLOCKS_PER_SM") ? std::atoi(std::getenv("BZG_BF_BLOCKS_PER_SM")) : 0;
    const int blocks = std::max(1, std::min(per_sm, bf_per_sm_env > 0 ? bf_per_sm_env : 4) * c->num_sms);
    long long Vl = V;
    const long long* rp = g->row_ptr.as<long long>();
    const int* dd = g->dst.as<int>();
    const double* cc = g->cost.as<double>();
    int* st = t_stamp.as<int>();
    int* pa = qa.as<int>();
    int* pb = qb.as<int>();
    int* pc = cnt.as<int>();
    int maxs = (int)std::min<long long>(V + 2, 1 << 30);
    if (bf_queue) {
      void* args[] = {&Vl, &rp, &dd, &cc, &alive, &dist, &st, &pa, &pb, &pc, &maxs};
      launch_coop(c, "k_bf_persistent", bf_kern, dim3(blocks), dim3(256), args);
    } else {
      // prev = dist at init (v0 = 0, others +inf), so the first scan sees only v0's improvements
      unsigned long long* pv = t_pd.as<unsigned long long>();
      BZG_CHECK_CUDA(cudaMemcpyAsync(pv, dist, V * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, c->stream));
      void* args[] = {&Vl, &rp, &dd, &cc, &alive, &dist, &pv, &pa, &pb, &pc, &maxs};
      launch_coop(c, "k_bf_scan", bf_kern, dim3(blocks), dim3(256), args);
      launch(c, "k_fill_pd", k_fill_u64, dim3(div_up(V, 256)), dim3(256), 0, pv, V, ~0ull);  // k_parent_dist's init
    }
    if (c->trace_on) {
      int hc[8];
      BZG_CHECK_CUDA(cudaMemcpyAsync(hc, cnt.ptr, sizeof(hc), cudaMemcpyDeviceToHost, c->stream));
      BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
      std::fprintf(stderr, "[bzg path] Bellman-Ford sweeps %d, frontier vertices expanded %d (V = %lld)\n", hc[3],
                   hc[4], V);
    }
    launch(c, "k_parent_dist", k_parent_dist, dim3(div_up(E, 256)), dim3(256), 0, E, g->src.as<int>(),
           g->dst.as<int>(), g->cost.as<double>(), alive, dist, t_pd.as<unsigned long long>());
    launch(c, "k_parent_idx", k_parent_idx, dim3(div_up(E, 256)), dim3(256), 0, E, g->src.as<int>(), g->dst.as<int>(),
           g->cost.as<double>(), alive, dist, t_pd.as<unsigned long long>(), parent);
    if (mk) mk->tree_v0 = v0;
  }
  lpath.alloc((V + 1) * sizeof(long long), c->stream);
  llen.alloc(sizeof(long long), c->stream);
  ldist.alloc(sizeof(double), c->stream);
  launch(c, "k_backtrack", k_backtrack, dim3(1), dim3(32), 0, V, v0, vg, parent, dist, lpath.as<long long>(),
         llen.as<long long>(), ldist.as<double>());
  long long* h = static_cast<long long*>(c->host_scratch(2 * sizeof(long long)));
  BZG_CHECK_CUDA(cudaMemcpyAsync(h, llen.ptr, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaMemcpyAsync(h + 1, ldist.ptr, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  const long long len = h[0];
  double dv;
  memcpy(&dv, h + 1, sizeof(double));
  BZG_REQUIRE(len != -2, BZG_ECUDA, "parent chain broken during backtrack");
  if (len < 0) return;  // vg unreachable -> None
  std::vector<long long> rev(len);
  BZG_CHECK_CUDA(cudaMemcpyAsync(rev.data(), lpath.ptr, len * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  path.resize(len);
  for (long long i = 0; i < len; ++i) path[i] = rev[len - 1 - i];
  *dist_out = dv;
}

}  // namespace bzg
