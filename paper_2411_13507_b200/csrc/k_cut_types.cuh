// Types shared by the cut translation units (k_cut.cu: screen + aggregation; k_qp_g*.cu:
// the Cut-QP per gamma).  Kept in an anonymous namespace like the kernels that use them;
// across translation units the obstacle records travel as raw device pointers.
#pragma once

#include "bzg_internal.cuh"

namespace bzg {

// Everything the batched Cut-QP of one cut needs (k_qp_impl.cuh qp_solve_t).
struct QpJob {
  const Graph* g;
  double D[64];                       // boundary matrix (p+1) x 2*gamma, row-major
  const void* d_obs;                  // ObsRec<M>[n_obs] on the device
  bool canon;                         // every obstacle a canonical box (A = [I; -I])
  const unsigned long long* d_pend;   // work list (e << 20 | o)
  long long n_inst;                   // capacity of the work list and of every per-instance buffer
  const unsigned long long* d_n;      // device-side instance count (nullptr: n_inst itself)
  const bzg_cut_config* cfg;
  int polish_mode;                    // 0 none, 1 SOLVED, 2 SOLVED and MAX_ITER
  double screen;                      // polish screen (k_qp_select)
  Mask* mk;                           // receives n_polished (-1 unless read back)
  DevBuf* d_safe;                     // receives the verdicts (n_inst capacity)
  int8_t* st_out;                     // solver status, iterations, ||delta|| per instance
  int* it_out;
  double* delta_out;
};
// C = padded obstacle rows of the launch (2m or kObsRows); defined in k_qp_g<gamma>.cu
void qp_solve_g1(Ctx* c, int M, int C, const QpJob& j);
void qp_solve_g2(Ctx* c, int M, int C, const QpJob& j);
void qp_solve_g3(Ctx* c, int M, int C, const QpJob& j);
void qp_solve_g4(Ctx* c, int M, int C, const QpJob& j);
inline void qp_solve(Ctx* c, int G, int M, int C, const QpJob& j) {
  switch (G) {
    case 1: qp_solve_g1(c, M, C, j); return;
    case 2: qp_solve_g2(c, M, C, j); return;
    case 3: qp_solve_g3(c, M, C, j); return;
    case 4: qp_solve_g4(c, M, C, j); return;
    default: throw Error(BZG_EUNSUPPORTED, "device cut supports gamma in 1..4");
  }
}

namespace {

struct DParams {
  double D[64];
};

// Row capacities of the obstacle records: kObsRows for boxes and small polytopes (the records
// the screen stages in shared memory), kObsRowsBig for the rest (convex hulls with many faces,
// e.g. the paper's segmented obstacles): those take the general screen and a Cut-QP launch
// with C = kObsRowsBig.  More rows: BZG_EUNSUPPORTED.
constexpr int kObsRows = 8;
constexpr int kObsRowsBig = 32;
// record capacity a Cut-QP launch with C padded rows reads
template <int C>
constexpr int obs_cap() { return C > kObsRows ? kObsRowsBig : kObsRows; }

// Per-obstacle record.  Rows past `rows` are padding (A = 0, b = 1e300): inert in every
// test and in the Cut-QP (k_qp_common.cuh).  In an RC = kObsRows record of an obstacle with
// more rows only `rows` (and is_box = 0) is meaningful: the screen sends its pairs to the
// general path, which reads the kObsRowsBig record.
template <int M, int RC = kObsRows>
struct ObsRec {
  double A[RC][M];         // normalised rows (geometry.py:135-137)
  double b[RC];
  double b_eps[RC];        // fl(b + eps_geo)   (graph.py:234)
  double norm2[RC];        // row norms of the normalised rows (Polytope._row_norms of O)
  double lo[M], hi[M];     // Polytope.as_box bounds (geometry.py:155-185)
  double canon;            // 1 when A == [I; -I] exactly (Box.to_polytope row order)
  double act_hi[M];        // hi - 1e-6: a point below it cannot make face +k active
  double act_lo[M];        // lo + 1e-6
  double thin[M];          // 1 when hi - lo <= 1e-6 (both faces of axis k may be active)
  double rows;             // constraint rows
  double is_box;           // 1 when as_box() recovers a box (the closed-form branch applies)
};

}  // namespace
}  // namespace bzg
