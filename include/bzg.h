/*
 * bzg.h — C ABI of the B200-native graph-construction stage for
 * reachable-Bezier-polytope kinodynamic planning (arXiv 2411.13507).
 *
 * The reference (beziergraph, /root/reference/pkg/src/beziergraph) is pure
 * Python and has no FFI; the entry points below are the boundary a
 * maintainer binds (ctypes stub in INTEGRATION.md) to replace the hot
 * functions of graph.py.  Each declaration cites the reference interface it
 * replaces.
 *
 * Conventions
 *   - every call returns 0 on success or a negative BZG_E* code;
 *     bzg_last_error() returns a thread-local message for the last failure;
 *   - host pointers are owned by the caller; opaque handles are owned by the
 *     library and released with the matching *_destroy call;
 *   - arrays are C-order float64 / int64 exactly as numpy holds them;
 *   - work is stream-ordered on the context's stream; calls that return host
 *     data synchronise that stream before returning;
 *   - there is no CPU fallback: without a usable sm_100 device every compute
 *     call fails with BZG_ENODEV.
 */
#ifndef BZG_H
#define BZG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BZG_ABI_VERSION 1

enum {
  BZG_OK = 0,
  BZG_EINVAL = -1,      /* argument error (reference raises ValueError) */
  BZG_ENODEV = -2,      /* no usable CUDA device */
  BZG_ECUDA = -3,       /* CUDA runtime error */
  BZG_EUNSUPPORTED = -4,/* input outside what the device path implements */
  BZG_ENOMEM = -5
};

/* provenance codes, reference graph.py:35-39 (CutProvenance) */
enum { BZG_HEURISTIC_UNSAFE = 0, BZG_HEURISTIC_SAFE = 1, BZG_QP_SAFE = 2, BZG_QP_UNSAFE = 3 };
/* QP status codes, reference qpsolver.py:29-33 (SolveStatus) */
enum { BZG_SOLVED = 0, BZG_MAX_ITER = 1, BZG_INFEASIBLE = 2, BZG_ERROR = 3 };

typedef struct bzg_ctx bzg_ctx;
typedef struct bzg_graph bzg_graph;
typedef struct bzg_mask bzg_mask;
typedef struct bzg_query bzg_query;
typedef struct bzg_replanner bzg_replanner;
typedef struct bzg_planner bzg_planner;

int bzg_abi_version(void);
const char* bzg_last_error(void);

/* ---- context ----------------------------------------------------------- */
/* stream: a cudaStream_t to run on, or NULL for a library-owned stream. */
int bzg_ctx_create(int device, void* stream, bzg_ctx** out);
int bzg_ctx_destroy(bzg_ctx* ctx);
int bzg_ctx_stream(bzg_ctx* ctx, void** stream_out);
int bzg_ctx_synchronize(bzg_ctx* ctx);
/* per-kernel CUDA-event timing of every launch (off by default) */
int bzg_ctx_set_profiling(bzg_ctx* ctx, int enabled);
/* restrict profiling to launches of one kernel (NULL or "" = all), so timing a step adds
 * only two event records per launch of that kernel */
int bzg_ctx_profile_only(bzg_ctx* ctx, const char* kernel);
/* launches since creation/reset; with profiling, per-kernel totals.
 * names: buffer of n_cap*64 chars; ms/launches: n_cap entries; *n_out = kernels seen. */
int bzg_ctx_stats(bzg_ctx* ctx, long long* launches, int n_cap, char* names, double* ms,
                  long long* counts, int* n_out);
int bzg_ctx_reset_stats(bzg_ctx* ctx);

/* ---- a1..a5: build_graph (reference graph.py:129-199) ------------------- */
typedef struct {
  int32_t m, gamma, p;        /* BezierSpec (bezier.py:22-44); n = m*gamma, p = 2*gamma-1 */
  int32_t n_F;                /* rows of the reachability oracle */
  const double* F;            /* (n_F, 2n) ReachOracle.F (reachability.py:53) */
  const double* G;            /* (n_F,)    ReachOracle.G */
  double eps_geo;             /* EPS_GEO (geometry.py:14): thresh = G + eps_geo */
  const double* D;            /* (p+1, 2*gamma) boundary_matrix (bezier.py:201) */
  /* sampler (graph.py:147-157): first N accepted rows of one PCG64 stream */
  int64_t N;
  uint64_t pcg_state_hi, pcg_state_lo;  /* numpy PCG64 bit_generator.state['state'] */
  uint64_t pcg_inc_hi, pcg_inc_lo;      /* ... ['inc'] */
  const double* sample_lo;    /* (n,) Box.lo of the sampling bounds */
  const double* sample_hi;    /* (n,) Box.hi */
  int32_t xd_rows;            /* oracle.Xd: (xd_rows, n) A and (xd_rows,) b */
  const double* xd_A;
  const double* xd_b;
  /* optional vertices appended after the samples (graph.py:158-159) */
  int64_t n_include;
  const double* include;      /* (n_include, n) or NULL */
  /* optional: skip sampling and take these vertices verbatim (N rows); NULL = sample */
  const double* vertices;
  /* source-row block [row_begin, row_end) of the pair matrix this call evaluates
   * (multi-GPU row sharding); row_end <= 0 means all rows */
  int64_t row_begin, row_end;
  /* optional keep-in free regions (north-star configs 1 and 5, paper_2411_13507_b200/regions.py):
   * region r adds rows [region_row_off[r], region_row_off[r+1]) of region_F (rows, 2n) and
   * region_G to the base oracle; edge i->j needs the base test AND some region r whose added
   * rows all hold.  Added rows must be one-sided (position rows of a minimal-degree curve are:
   * the first gamma control points depend on x1 only, the last gamma on x2 only). */
  int32_t n_regions;
  const int32_t* region_row_off;
  const double* region_F;
  const double* region_G;
  /* optional (n_regions, m) position bounding boxes of the regions, NULL = none: a vertex
   * outside a region's box (by more than 1e-6) is not tested against its rows */
  const double* region_box_lo;
  const double* region_box_hi;
  /* k_nearest prefilter (graph.py:162-170): < 0 = off; else edge i->j also needs j among
   * the min(k_nearest, V-1) nearest vertices of i by fl(sum_k (p_ik - p_jk)^2) over the m
   * position coordinates.  Ties at the k-th distance keep the lowest indices (the
   * reference's argpartition tie order is implementation-defined). */
  int64_t k_nearest;
} bzg_build_desc;

/* north-star eps-band report: ordered pairs (i != j) whose minimum constraint slack
 * min_r (G_r + eps_geo - (F1 x_i + F2 x_j)_r) lies in (-eps, eps], counted over g's source-row
 * block as counts[1] - counts[2] with counts[1] = #pairs feasible with every threshold
 * fl(G_r + eps_geo) + eps and counts[2] = # with fl(G_r + eps_geo) - eps; counts[0] = the band.
 * desc = the descriptor g was built from (its vertices are g's; k_nearest is ignored). */
int bzg_graph_eps_band(bzg_graph* g, const bzg_build_desc* desc, double eps, int64_t counts[3]);

/* the sampler alone (graph.py:147-157): N accepted states of one PCG64 stream written to a
 * host buffer (N, n); uses desc's m, gamma, N, pcg_*, sample_lo/hi, xd_*, eps_geo */
int bzg_sample_states(bzg_ctx* ctx, const bzg_build_desc* desc, double* out_host);
/* the sampler for several keep-in regions in one call (regions.py sample_region_states):
 * region r draws N[r] states from its own PCG64 stream (pcg[4r..4r+3] = state_hi, state_lo,
 * inc_hi, inc_lo of default_rng([seed, r])) in the box lo/hi (n_regions x n), accepting in
 * rows [row_off[r], row_off[r+1]) of A (rows x n) / b; out_host = (sum N, n) in region order */
int bzg_sample_region_states(bzg_ctx* ctx, int32_t n, int32_t n_regions, const int64_t* N, const uint64_t* pcg,
                             const double* lo, const double* hi, const int32_t* row_off, const double* A,
                             const double* b, double eps_geo, double* out_host);

/* replaces graph.build_graph (graph.py:129-199), k_nearest prefilter included */
int bzg_build_graph(bzg_ctx* ctx, const bzg_build_desc* desc, bzg_graph** out);
/* assemble a graph from an existing edge list (device or host pointers), used by
 * the multi-GPU gather on rank 0; edges must be in row-major (src, dst) order */
int bzg_graph_from_edges(bzg_ctx* ctx, int32_t m, int32_t gamma, int32_t p, const double* D, int64_t V,
                         const double* vertices_host, int64_t E, const int32_t* src, const int32_t* dst,
                         const double* cost, int on_device, bzg_graph** out);
/* a new graph over the vertices of `like` (copied on the device) with the given edge list
 * (row-major (src, dst) + cost; device or host pointers): rank 0's graph of the gathered row
 * blocks.  `like` and its masks stay valid. */
int bzg_graph_with_edges(const bzg_graph* like, int64_t E, const int32_t* src, const int32_t* dst,
                         const double* cost, int on_device, bzg_graph** out);
/* replace the edge set of g (row-major ordered (src, dst) + cost; device or host pointers);
 * the row block becomes [0, V).  Masks cut before the change become stale: bzg_find_path,
 * bzg_mask_copy and bzg_mask_export_device reject them with BZG_EINVAL. */
int bzg_graph_set_edges(bzg_graph* g, int64_t E, const int32_t* src, const int32_t* dst, const double* cost,
                        int on_device);
/* re-cut cache (device-resident replanning, sim.py:324-330): while max_obstacles > 0, every
 * bzg_cut_graph on g keeps per-obstacle outcome bits (3 x E bits per obstacle) for up to
 * max_obstacles distinct obstacles (least recently used evicted); obstacles seen before --
 * same normalised rows, bounds and cut configuration, bit for bit -- are not screened or QP'd
 * again, only recombined, so a replanning cycle in which a few obstacles moved costs the cut
 * of those few.  The mask is identical to a full cut's; its QP records cover the QPs this
 * call solved.  Lists longer than max_obstacles are cut without the cache.  0 = off. */
int bzg_graph_set_cut_cache(bzg_graph* g, int32_t max_obstacles);
int bzg_graph_destroy(bzg_graph* g);
int bzg_graph_info(const bzg_graph* g, int64_t* V, int64_t* E, int64_t* row_begin, int64_t* row_end);
/* host copies (BezierGraph fields, graph.py:61-68); any pointer may be NULL */
int bzg_graph_copy_vertices(bzg_graph* g, double* vertices /* (V, n) */);
int bzg_graph_copy_edges(bzg_graph* g, int64_t* edges /* (E, 2) */, double* costs /* (E,) */);
int bzg_graph_copy_points(bzg_graph* g, double* points /* (E, m, p+1) */);
int bzg_graph_copy_csr(bzg_graph* g, int64_t* row_ptr /* (V+1,) */, int32_t* col /* (E,) */);
/* device-to-device export into caller-allocated device buffers (NCCL gather) */
int bzg_graph_export_device(bzg_graph* g, int32_t* src, int32_t* dst, double* cost);

/* replaces reachability.check_edges (reachability.py:139-142): out[k] = 1 iff
 * X1[k] F1' + X2[k] F2' <= G + eps row-wise (same separable arithmetic as the build) */
int bzg_check_edges(bzg_ctx* ctx, int32_t n, int32_t n_F, const double* F, const double* G, double eps,
                    int64_t k, const double* X1, const double* X2, uint8_t* out);

/* ---- a7..a10: cut_graph (reference graph.py:302-350) -------------------- */
typedef struct {
  double eps_cut;     /* CutConfig.eps_cut (graph.py:44) */
  double heur_margin; /* CutConfig.heur_margin (graph.py:45) */
  double eps_geo;     /* CutConfig.eps_geo (graph.py:46) */
  int32_t qp_max_iter;/* CutConfig.qp (graph.py:47-49) -> SolveConfig (qpsolver.py:60-72) */
  double qp_eps_abs, qp_eps_rel, qp_rho, qp_sigma, qp_alpha, qp_eps_pinf;
  int32_t qp_polish;
} bzg_cut_config;

/* Obstacles in list order.  Rows of obstacle o are rows [row_off[o], row_off[o+1])
 * of A (rows x m) / b, ALREADY NORMALISED (Polytope.normalized, geometry.py:135-137).
 * is_box[o] != 0 marks obstacles recovered by Polytope.as_box (geometry.py:155-185)
 * with the recovered bounds box_lo/box_hi (o*m ... o*m+m-1); they take the closed-form
 * screen (graph.py:249-264).  Other obstacles (1..32 rows) take the per-edge cut_heuristic
 * (graph.py:202-221, projection QPs of geometry.py:202-252).  More than 32 rows:
 * BZG_EUNSUPPORTED.  An obstacle whose projection QP certifies it empty: BZG_EINVAL
 * (the reference raises ValueError). */
int bzg_cut_graph(bzg_ctx* ctx, bzg_graph* g, int32_t n_obs, const int32_t* row_off, const double* A,
                  const double* b, const uint8_t* is_box, const double* box_lo, const double* box_hi,
                  const bzg_cut_config* cfg, bzg_mask** out);
/* The scalar entry points on explicit control points: B sets of (m x J) control points
 * (row-major, J = p + 1 even), set i tested against obstacle obs_index[i] of the list
 * (same obstacle arrays as bzg_cut_graph).
 *   mode 0 = cut_heuristic (graph.py:202-221): code[i] = 0 unsafe / 1 safe / 2 indeterminate;
 *   mode 1 = cut_qp (graph.py:285-299): code[i] = safe flag, delta[i] = ||delta*||,
 *            status[i] = solver status (BZG_SOLVED ...).  delta/status may be NULL. */
int bzg_cut_points(bzg_ctx* ctx, int32_t m, int32_t J, int64_t B, const double* points, const int32_t* obs_index,
                   int32_t n_obs, const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box,
                   const double* box_lo, const double* box_hi, const bzg_cut_config* cfg, int32_t mode, int8_t* code,
                   double* delta, int8_t* status);
int bzg_mask_destroy(bzg_mask* mk);
/* edge count the mask was cut for, and its QP instance count */
int bzg_mask_info(const bzg_mask* mk, int64_t* E, int64_t* n_qp);
/* counters: pairs_total, pairs_point_hit, pairs_hyperplane, pairs_qp, qp_safe, qp_unsafe (graph.py:97-102) */
int bzg_mask_copy(bzg_mask* mk, uint8_t* alive /* (E,) */, uint8_t* provenance /* (E,) */, int64_t counters[6]);
/* QP diagnostics of the last cut: per solved instance (edge, obstacle, status, iterations, ||delta||) */
int bzg_mask_qp_count(bzg_mask* mk, int64_t* n);
int bzg_mask_copy_qp(bzg_mask* mk, int64_t* edge, int32_t* obstacle, int8_t* status, int32_t* iters, double* delta);
/* assemble a mask from alive/provenance arrays (multi-GPU gather) */
int bzg_mask_from_arrays(bzg_ctx* ctx, bzg_graph* g, const uint8_t* alive, const uint8_t* provenance,
                         const int64_t counters[6], int on_device, bzg_mask** out);
int bzg_mask_export_device(bzg_mask* mk, uint8_t* alive, uint8_t* provenance);

/* ---- a11..a13: find_path (reference graph.py:353-430) ------------------- */
/* path_out: caller buffer of path_cap entries; *path_len = -1 means None (no path).
 * tube_lo/tube_hi: oracle.tube.error box (n,).  *dist_out = path cost (graph.py:453-458). */
int bzg_find_path(bzg_ctx* ctx, bzg_graph* g, bzg_mask* mk, const double* start, const double* goal,
                  const double* tube_lo, const double* tube_hi, double eps_geo, int position_only_snap,
                  int require_tube_snap, int64_t* path_out, int64_t path_cap, int64_t* path_len,
                  double* dist_out);
/* repeated find_path on one (graph, mask) -- the 200 Hz goal/start updates of a replanning
 * loop (sim.py:275-408 calls graph.find_path every cycle): bzg_query_create warms the search
 * up once and captures it as a CUDA graph; bzg_query_run(start, goal) is then one graph
 * launch and one synchronisation, with the same result as bzg_find_path with these options.
 * mk may be NULL (no mask).  A query is stale (BZG_EINVAL) once g's edge set changes; destroy
 * it before its graph and mask. */
int bzg_query_create(bzg_ctx* ctx, bzg_graph* g, bzg_mask* mk, const double* tube_lo, const double* tube_hi,
                     double eps_geo, int position_only_snap, int require_tube_snap, bzg_query** out);
int bzg_query_run(bzg_query* q, const double* start, const double* goal, int64_t* path_out, int64_t path_cap,
                  int64_t* path_len, double* dist_out);
/* kernels per bzg_query_run (the captured graph's kernel nodes) */
int bzg_query_kernels(const bzg_query* q, int64_t* n);
int bzg_query_destroy(bzg_query* q);

/* ---- f2: the replanning cycle as one captured CUDA graph -------------------- */
/* A cycle of sim.run_closed_loop (sim.py:324-330: re-cut with the moved obstacles, then
 * graph.find_path, graph.py:302-430) on a fixed graph: bzg_replanner_create runs the first cycle
 * with the given obstacles eagerly and captures cut + search as one CUDA graph; every
 * bzg_replanner_run is then one graph launch and one synchronisation, with the obstacle records
 * and the snapping targets passed through pinned staging.  Results equal bzg_cut_graph +
 * bzg_find_path on the same inputs.  The obstacle list keeps its count; when its shape (row
 * counts, box / general kinds) changes or a work list outgrows its capacity, that cycle runs
 * eagerly (*eager = 1) and the graph is re-captured.  counters: as bzg_mask_copy.  The
 * replanner's mask holds no per-QP records.  dynamic (n_obs flags, NULL = all): obstacles
 * flagged 0 are static -- cut once, their per-obstacle outcome rows kept on the device (as
 * the re-cut cache keeps them) -- and a cycle cuts only the dynamic ones and rebuilds the mask
 * in list order; a static obstacle passed changed to a later run is re-cut then.  A run may
 * pass the dynamic obstacles alone (n_obs = their count, in list order): the static ones then
 * stand as last given. */
int bzg_replanner_create(bzg_ctx* ctx, bzg_graph* g, int32_t n_obs, const int32_t* row_off, const double* A,
                         const double* b, const uint8_t* is_box, const double* box_lo, const double* box_hi,
                         const uint8_t* dynamic, const bzg_cut_config* cfg, const double* tube_lo, const double* tube_hi, double eps_geo,
                         int position_only_snap, int require_tube_snap, bzg_replanner** out);
int bzg_replanner_run(bzg_replanner* rp, int32_t n_obs, const int32_t* row_off, const double* A, const double* b,
                      const uint8_t* is_box, const double* box_lo, const double* box_hi, const double* start,
                      const double* goal, int64_t* path_out, int64_t path_cap, int64_t* path_len, double* dist_out,
                      int64_t counters[6], int32_t* eager);
/* a new mask (owned by the caller) holding the last cycle's alive set, provenance and counters */
int bzg_replanner_mask(bzg_replanner* rp, bzg_mask** out);
/* info: kernels per captured cycle, cycles run, cycles run eagerly, captures */
int bzg_replanner_info(const bzg_replanner* rp, int64_t info[4]);
int bzg_replanner_destroy(bzg_replanner* rp);

/* ---- the whole stage as one captured CUDA graph ---------------------------- */
/* build_graph -> cut_graph -> find_path (graph.py:129-430, the order of sim.plan_once) for one
 * scene shape: desc fixes the oracle, N, curve, sampling bounds and include count (keep-in
 * regions take a bzg_region_sampler; no row block); the obstacle list keeps its count.
 * bzg_planner_create runs the first call (desc's seed and include rows, the given obstacles)
 * eagerly and captures the stage; each bzg_planner_run (pcg = the seed's PCG64 words as in
 * bzg_build_desc, 4 per region with keep-in regions; include rows; obstacles; start; goal) is
 * then one graph launch and one synchronisation, with the results of bzg_build_graph +
 * bzg_cut_graph + bzg_find_path on the same inputs.  The build's edge count stays on the
 * device; the CSR arrays have a capacity (1.5 x the last edge count, at most every ordered
 * pair); a call whose sampler round fell short, whose edges outgrew the capacity, whose work
 * lists overflowed or whose obstacle list changed shape runs eagerly (*eager = 1) and
 * re-captures.  counters as bzg_mask_copy; *num_edges = the graph's E. */
/* keep-in regions (desc->n_regions > 0): the per-region sampler of bzg_sample_region_states --
 * N[r] states of region r from its own PCG64 stream (pcg: 4 words per region, this call's
 * seed), box lo/hi (n_regions x n), state-set rows [row_off[r], row_off[r+1]) of A / b; the N[r]
 * add up to desc->N.  A planner's run then takes 4 words per region. */
typedef struct {
  int32_t n_regions;
  const int64_t* N;
  const uint64_t* pcg;
  const double* lo;
  const double* hi;
  const int32_t* row_off;
  const double* A;
  const double* b;
} bzg_region_sampler;
int bzg_planner_create(bzg_ctx* ctx, const bzg_build_desc* desc, const bzg_region_sampler* regions, int32_t n_obs,
                       const int32_t* row_off,
                       const double* A, const double* b, const uint8_t* is_box, const double* box_lo,
                       const double* box_hi, const bzg_cut_config* cfg, const double* tube_lo, const double* tube_hi,
                       double eps_geo, int position_only_snap, int require_tube_snap, bzg_planner** out);
int bzg_planner_run(bzg_planner* pl, const uint64_t* pcg, const double* include, int32_t n_obs,
                    const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box,
                    const double* box_lo, const double* box_hi, const double* start, const double* goal,
                    int64_t* path_out, int64_t path_cap, int64_t* path_len, double* dist_out, int64_t counters[6],
                    int64_t* num_edges, int32_t* eager);
/* copies (owned by the caller) of the last call's graph and (m_out non-NULL) its mask */
int bzg_planner_result(bzg_planner* pl, bzg_graph** g_out, bzg_mask** m_out);
/* info: kernels per captured call, calls, eager calls, captures, edge capacity, and why the
 * last eager call was eager (0 it was not / the first call, 1 obstacle-list shape, 2 sampler
 * round short, 3 edge capacity, 4 cut work lists) */
int bzg_planner_info(const bzg_planner* pl, int64_t info[6]);
int bzg_planner_destroy(bzg_planner* pl);

/* replaces sim._project_on_path (sim.py:220-239): the grid time tau = k h (k < (L-1) *
 * steps_per_hop, steps_per_hop = round(T / h)) along the curve chain through the L path states
 * (L, n) whose position is closest to state[:m]; first minimum, same arithmetic as the
 * reference (bezier.py boundary_points / de_casteljau, 1-D norm).  L <= 1: 0. */
int bzg_project_on_path(bzg_ctx* ctx, int32_t m, int32_t gamma, double T, const double* D, int64_t L,
                        const double* path_states, double h, int32_t steps_per_hop, const double* state,
                        double* best_t);

/* ---- diagnostics (not a reference entry point) -------------------------- */
/* sustained FP64 instruction issue rate (DFMA if use_fma else DADD), instructions/s:
 * the roofline denominator of the FP64-pipe-bound kernels (pair test, box cut, QP). */
int bzg_probe_fp64(bzg_ctx* ctx, int use_fma, double* instr_per_s);

#ifdef __cplusplus
}
#endif
#endif /* BZG_H */
