// Internal runtime of libbzg: context, device buffers, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <stdexcept>
#include <string>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/bzg.h"
#include <nvtx3/nvToolsExt.h>

namespace bzg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BZG_CHECK_CUDA(call)                                                                  \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw ::bzg::Error(BZG_ECUDA, std::string(#call) + " failed: " + cudaGetErrorString(e_)); \
  } while (0)

#define BZG_REQUIRE(cond, code, msg)          \
  do {                                        \
    if (!(cond)) throw ::bzg::Error(code, msg); \
  } while (0)

struct Ctx;

// NVTX range around a public entry point (header-only NVTX v3: a no-op unless a profiler such as
// ncu --nvtx or nsys attaches), so captures can be filtered by call.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Programmatic dependent launch: every kernel of the library begins with BZG_PDL_ENTRY -- wait
// for the preceding grid's completion (and memory flush), then let the next grid launch -- and
// launch() marks its launches programmatic-serialisation-allowed, so a kernel's blocks are
// scheduled while its predecessor's last wave drains instead of after it (in captured graphs,
// a programmatic edge).  Nothing runs before the wait, so stream order is preserved; a launch
// without the attribute (cooperative, cluster, CUB) makes the wait a no-op.  BZG_PDL=0: off.
#define BZG_PDL_ENTRY() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BZG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Set while a stream capture (bzg_query) records work: a workspace that would have to grow
// then is an error (the graph would bake in a fresh allocation), so captures are preceded by
// an eager warm-up that sizes every buffer.
inline thread_local bool g_capturing = false;

// Stream-ordered device allocation owned by the library.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr; bytes = o.bytes; stream = o.stream;
      o.ptr = nullptr; o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFreeAsync(ptr, stream);
    ptr = nullptr;
    bytes = 0;
  }
  void alloc(size_t nbytes, cudaStream_t s) {
    if (nbytes <= bytes && ptr) return;
    if (g_capturing) throw Error(BZG_ECUDA, "workspace grew during a stream capture");
    release();
    stream = s;
    if (nbytes == 0) nbytes = 16;
    BZG_CHECK_CUDA(cudaMallocAsync(&ptr, nbytes, s));
    bytes = nbytes;
  }
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
};

// workspace slots of Ctx::ws (each used by one buffer of one phase at a time)
enum WsSlot {
  WS_CAND, WS_FLAG, WS_POS,                                          // samplers
  WS_BITS, WS_A1C, WS_A2T, WS_ROWCNT, WS_RPTR, WS_PAIRLIST,          // pair test
  WS_KILL, WS_QKILL, WS_SAVED, WS_PEND, WS_GEN, WS_OBSGRID,          // cut screen
  WS_QX, WS_QZY, WS_QSAFE, WS_QLIST, WS_QCONST, WS_QRESUME, WS_QSTATUS, WS_QITERS, WS_QDELTA,             // Cut-QP
  WS_PLAN, WS_SSSP_PREV, WS_SSSP_PD, WS_SSSP_AUX, WS_SSSP_OUT,       // find_path
  WS_CUTBITS, WS_CUTSLOTS,                                           // re-cut cache
  WS_PROJ,                                                           // project_on_path
  WS_REACH_FLAGS,
  WS_SNAP, WS_BEST0, WS_BEST1, WS_NM_REACH, WS_NM_KEY, WS_NM_DIST, WS_NM_PARENT,  // find_path
  WS_OBSGRIDHDR, WS_CUTCNT, WS_CUTOBS, WS_QNEXT,                     // cut staging, counters
  WS_TIGHT,                                                          // find_path tight in-edges
  WS_SCRATCH,                                                        // CUB temporary storage
  kWsSlots
};

// Per-call device temporaries without a cudaMallocAsync / cudaFreeAsync pair each (a small
// scene's build did ~25 of them, tens of microseconds of host time): grow-only chunks handed
// out bump-style and reused by the next call.  Like the ws slots this is safe because every
// use is stream-ordered on the context's one stream; reset() at the start of each user.
struct Arena {
  std::vector<DevBuf> chunks;
  size_t cur = 0, off = 0;
  void reset() {
    cur = 0;
    off = 0;
  }
  void* take(size_t bytes, cudaStream_t s) {
    bytes = std::max<size_t>((bytes + 255) & ~(size_t)255, 256);
    while (true) {
      if (cur == chunks.size()) chunks.emplace_back();
      DevBuf& ch = chunks[cur];
      if (off == 0 && ch.bytes < bytes) ch.alloc(std::max<size_t>(bytes, (size_t)1 << 20), s);
      if (off + bytes <= ch.bytes) {
        void* p = static_cast<char*>(ch.ptr) + off;
        off += bytes;
        return p;
      }
      ++cur;
      off = 0;
    }
  }
};

struct KernelStat {
  double ms = 0.0;
  long long count = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  bool profiling = false;
  std::string profile_only;  // when non-empty, time only launches of this kernel
  long long launches = 0;
  bool timed(const char* name) const { return profiling && (profile_only.empty() || profile_only == name); }
  // BZG_TRACE=1: synchronising host wall-time trace of library phases (diagnosing launch gaps)
  bool trace_on = std::getenv("BZG_TRACE") != nullptr;
  std::chrono::steady_clock::time_point trace_t = std::chrono::steady_clock::now();
  void trace(const char* what) {
    if (!trace_on || g_capturing) return;
    cudaStreamSynchronize(stream);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bzg] %-24s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - trace_t).count());
    trace_t = now;
  }
  struct Pending { std::string name; cudaEvent_t a, b; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> spare;
  std::vector<std::string> order;
  std::unordered_map<std::string, KernelStat> stats;
  DevBuf flag;          // small device scalars
  // Grow-only workspaces for the per-call temporaries (pair bit matrix, sampler candidates,
  // cut work lists, QP state): reused across calls on this stream, so repeated builds and
  // cuts do not refragment the stream-ordered pool (a fresh 1 GB bit matrix per step made the
  // pool map new memory at random steps, milliseconds each).
  // ws points at ws_own except while a bzg_query warms up or captures with its own set.
  DevBuf ws_own[kWsSlots];
  DevBuf* ws = ws_own;
  Arena arena_own;         // per-call temporaries (TmpBuf)
  Arena* arena = &arena_own;  // switched with ws by a captured plan
  // last obstacle-grid decision (k_cut.cu): obstacle count and xy bounds -> grid sparse enough
  int grid_nobs = -1;
  double grid_key[4] = {0, 0, 0, 0};
  bool grid_sparse = false;
  long long qp_hint = 0;   // QP instances of the last cut: sizes the next cut's QP buffers
  unsigned long long cut_last_pend = 0, cut_last_gen = 0;  // the last cut's work-list lengths
  double sample_est = 1.0; // acceptance rate of the last sampler run (sizes a single round)
  int* sample_check = nullptr;  // pending single-round sampler count (device), need, candidates
  long long sample_need = 0, sample_count = 0;
  void* pinned = nullptr;  // small pinned host staging area
  size_t pinned_bytes = 0;

  cudaEvent_t take_event() {
    if (!spare.empty()) { cudaEvent_t e = spare.back(); spare.pop_back(); return e; }
    cudaEvent_t e;
    BZG_CHECK_CUDA(cudaEventCreate(&e));
    return e;
  }
  void drain_profile() {
    if (pending.empty()) return;
    BZG_CHECK_CUDA(cudaStreamSynchronize(stream));
    for (auto& p : pending) {
      float ms = 0.f;
      BZG_CHECK_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
      auto it = stats.find(p.name);
      if (it == stats.end()) { order.push_back(p.name); it = stats.emplace(p.name, KernelStat{}).first; }
      it->second.ms += ms;
      it->second.count += 1;
      spare.push_back(p.a);
      spare.push_back(p.b);
    }
    pending.clear();
  }
  void* host_scratch(size_t bytes) {
    if (bytes > pinned_bytes) {
      if (pinned) cudaFreeHost(pinned);
      BZG_CHECK_CUDA(cudaMallocHost(&pinned, bytes));
      pinned_bytes = bytes;
    }
    return pinned;
  }
};

// A DevBuf-like view of arena memory, valid until the next Arena::reset of its context.
struct TmpBuf {
  Ctx* c;
  void* ptr = nullptr;
  size_t bytes = 0;
  explicit TmpBuf(Ctx* c_) : c(c_) {}
  void alloc(size_t n, cudaStream_t s) {
    if (ptr && n <= bytes) return;
    ptr = c->arena->take(n, s);
    bytes = n;
  }
  template <typename T> T* as() const { return static_cast<T*>(ptr); }
};

// Raise a kernel's dynamic shared-memory limit only when a launch needs more than before: the
// driver call costs tens of microseconds, which shows up as a gap whenever the stream is empty.
inline void ensure_dyn_smem(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, size_t> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long key = (unsigned long long)(uintptr_t)kern ^ ((unsigned long long)dev << 56);
  std::lock_guard<std::mutex> lk(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return;
  BZG_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  done[key] = bytes;
}

// Launch a kernel on the context stream, counting it and (when profiling) timing it
// with a pair of CUDA events recorded on the same stream.
template <typename... KArgs, typename... Args>
inline void launch(Ctx* c, const char* name, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   Args&&... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  cudaEvent_t a = nullptr, b = nullptr;
  const bool timed = c->timed(name);
  if (timed) { a = c->take_event(); BZG_CHECK_CUDA(cudaEventRecord(a, c->stream)); }
  if (pdl_enabled()) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BZG_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  } else {
    kern<<<grid, block, smem, c->stream>>>(std::forward<Args>(args)...);
    BZG_CHECK_CUDA(cudaGetLastError());
  }
  c->launches++;
  if (timed) {
    b = c->take_event();
    BZG_CHECK_CUDA(cudaEventRecord(b, c->stream));
    c->pending.push_back({name, a, b});
  }
}

// Cooperative launch (all blocks co-resident, grid-wide sync allowed), counted and timed like launch().
inline void launch_coop(Ctx* c, const char* name, const void* kern, dim3 grid, dim3 block, void** args) {
  cudaEvent_t a = nullptr, b = nullptr;
  const bool timed = c->timed(name);
  if (timed) { a = c->take_event(); BZG_CHECK_CUDA(cudaEventRecord(a, c->stream)); }
  BZG_CHECK_CUDA(cudaLaunchCooperativeKernel(kern, grid, block, args, 0, c->stream));
  c->launches++;
  if (timed) {
    b = c->take_event();
    BZG_CHECK_CUDA(cudaEventRecord(b, c->stream));
    c->pending.push_back({name, a, b});
  }
}

// Record an externally launched (library) kernel group, e.g. CUB scans.
struct ScopedLibLaunch {
  Ctx* c; const char* name; cudaEvent_t a = nullptr; int n;
  ScopedLibLaunch(Ctx* ctx, const char* nm, int nkernels) : c(ctx), name(nm), n(nkernels) {
    if (c->timed(name)) { a = c->take_event(); BZG_CHECK_CUDA(cudaEventRecord(a, c->stream)); }
  }
  ~ScopedLibLaunch() {
    c->launches += n;
    if (a) {
      cudaEvent_t b = c->take_event();
      cudaEventRecord(b, c->stream);
      c->pending.push_back({name, a, b});
    }
  }
};

// Record fn()'s work on c->stream into an instantiated CUDA graph (stream capture, thread-local
// mode).  Every workspace must already be sized (g_capturing makes a growth an error) and no
// event may be recorded (profiling is paused).  *kernels = launches counted while capturing.
template <typename F>
cudaGraphExec_t capture_graph(Ctx* c, F&& fn, long long* kernels, cudaGraph_t* graph_out) {
  const bool prof = c->profiling;
  const long long launches0 = c->launches;
  c->profiling = false;
  g_capturing = true;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    try {
      fn();
    } catch (...) {
      cudaGraph_t tmp = nullptr;
      cudaStreamEndCapture(c->stream, &tmp);
      if (tmp) cudaGraphDestroy(tmp);
      g_capturing = false;
      c->profiling = prof;
      c->launches = launches0;
      throw;
    }
    e = cudaStreamEndCapture(c->stream, &graph);
  }
  g_capturing = false;
  c->profiling = prof;
  *kernels = c->launches - launches0;
  c->launches = launches0;
  BZG_CHECK_CUDA(e);
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  if (ei != cudaSuccess) {
    cudaGraphDestroy(graph);
    BZG_CHECK_CUDA(ei);
  }
  BZG_CHECK_CUDA(cudaGraphUpload(exec, c->stream));
  *graph_out = graph;
  return exec;
}

// run fn with c->ws switched to another workspace set (a captured plan's own buffers)
template <typename F>
void with_ws(Ctx* c, DevBuf* ws, F&& fn, Arena* arena = nullptr) {
  DevBuf* saved = c->ws;
  Arena* saved_a = c->arena;
  c->ws = ws;
  if (arena) c->arena = arena;
  try {
    fn();
  } catch (...) {
    c->ws = saved;
    c->arena = saved_a;
    throw;
  }
  c->ws = saved;
  c->arena = saved_a;
}

inline unsigned div_up(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

// ---------------------------------------------------------------- graph / mask
// Re-cut cache of a graph (cut_graph_cached): per distinct obstacle (key = its rows, bounds and
// the cut configuration, bit for bit) the three outcome bit rows of its last cut on this graph
// -- heuristic kill, QP safe, QP unsafe -- and their popcounts; a re-cut then runs the screen
// and the QPs only for obstacles it has not seen (the moved ones) and recombines the rest.
struct CutCache {
  int max_slots = 0;                       // 0: off
  long long Wb = 0;                        // words per bit row = ceil(E / 32)
  DevBuf pool;                             // max_slots x 3 x Wb uint32
  std::unordered_map<std::string, int> slot_of;
  std::vector<std::string> key_of;         // per slot ("" = free)
  std::vector<long long> stamp;            // last use (LRU)
  std::vector<long long> cnt;              // per slot: kill, qp safe, qp unsafe
  long long clock = 0;
  void clear() {
    slot_of.clear();
    for (auto& k : key_of) k.clear();
  }
};

struct Graph {
  Ctx* ctx = nullptr;
  int m = 0, gamma = 0, p = 0, n = 0;
  int64_t V = 0, E = 0;
  int64_t row_begin = 0, row_end = 0;
  std::vector<double> D;          // (p+1) x 2*gamma, host copy (kernel parameter)
  DevBuf vertices;                // V x n
  DevBuf row_ptr;                 // V+1 int64 (global row index)
  DevBuf src, dst;                // E int32
  DevBuf cost;                    // E double
  DevBuf points;                  // lazily materialised E x m x (p+1)
  bool points_ready = false;
  CutCache cut_cache;
  uint64_t version = 0;           // bumped whenever the edge set is replaced (stale queries)
  const long long* dE = nullptr;  // a captured plan's graph: the edge count on the device (E = capacity)
};

struct Mask {
  Graph* g = nullptr;
  Ctx* ctx = nullptr;  // kept here so a mask can be released after its graph (Python GC order)
  int64_t E = 0;
  int32_t n_obs = 0;
  DevBuf alive;                   // E uint8
  DevBuf prov;                    // E uint8
  int64_t counters[6] = {0, 0, 0, 0, 0, 0};
  // QP diagnostics
  int64_t n_qp = 0, n_polished = 0;
  DevBuf qp_edge, qp_obs, qp_status, qp_iters, qp_delta;
  // cached shortest-path tree (reused while (mask, v0) is unchanged: cfg4 replanning); the
  // key (the tree's v0, -1 = none) lives on the device next to the tree
  DevBuf dist, parent, tree_key;
  // cached reverse reachability to vg (relaxed snapping); its key (vg, -1 = none) on the device
  int64_t reach_vg = -1;
  DevBuf reach, reach_key;
};

// Kernel-family entry points (defined in the k_*.cu translation units).
// single_round: one round sized from Ctx::sample_est, its acceptance checked by build_pairs
void sample_states(Ctx* c, const bzg_build_desc* d, double* d_vertices, bool single_round = false,
                   const unsigned long long* pcg_dev = nullptr);
void sample_regions(Ctx* c, int n, int R, const int64_t* N, const uint64_t* pcg, const double* lo, const double* hi,
                    const int32_t* row_off, const double* A, const double* b, double eps_geo, double* d_out,
                    double* est_out = nullptr);
// a captured plan's keep-in pieces (k_build.cu): the single-round region sampler and the
// region rows of the pair test, uploaded once
struct RegionSamplePlan;
RegionSamplePlan* region_sample_plan_create(Ctx* c, int n, int R, const int64_t* N, const double* lo,
                                            const double* hi, const int32_t* row_off, const double* A,
                                            const double* b, double eps_geo, const double* est);
void region_sample_plan_enqueue(Ctx* c, RegionSamplePlan* s, const unsigned long long* d_pcg, double* d_out,
                                long long* h_acc);
void region_sample_plan_destroy(RegionSamplePlan* s);
struct RegionRowsCache;
RegionRowsCache* region_rows_cache_create(Ctx* c, const bzg_build_desc* d);
void region_rows_cache_destroy(RegionRowsCache* rc);
// th_shift moves every oracle threshold (eps-band counting); count_only != nullptr returns the
// edge count there and leaves g's CSR untouched.  Returns false (CSR untouched) when the
// preceding single-round sampler (Ctx::sample_check) accepted fewer than N states.
// A build recorded into a captured plan (bzg_planner): the oracle rows come from dF (uploaded
// once), nothing is read back mid-build, and the edge count / sampler acceptances are copied
// to h_out / h_sampled (pinned) for the plan's check after the launch.
struct BuildCapture {
  const double* dF;
  long long* h_out;
  int* h_sampled;
  const RegionRowsCache* rows = nullptr;  // keep-in rows (regions only)
};
bool build_pairs(Ctx* c, const bzg_build_desc* d, Graph* g, double th_shift = 0.0, long long* count_only = nullptr,
                 const BuildCapture* bc = nullptr);
void materialize_points(Ctx* c, Graph* g);
void set_edges(Ctx* c, Graph* g, long long E, const int* src, const int* dst, const double* cost, bool on_device);
void check_edges(Ctx* c, int n, int n_F, const double* F, const double* G, double eps, int64_t k,
                 const double* X1, const double* X2, uint8_t* out);
void cut_graph(Ctx* c, Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
               const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
               Mask* mk);
void cut_points(Ctx* c, int m, int J, long long B, const double* points, const int32_t* obs_index, int n_obs,
                const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box, const double* box_lo,
                const double* box_hi, const bzg_cut_config* cfg, int mode, int8_t* code_out, double* delta_out,
                int8_t* status_out);
double project_on_path(Ctx* c, int m, int gamma, double T, const double* D, long long L, const double* path_states,
                       double h, int spt, const double* state);
void find_path(Ctx* c, Graph* g, Mask* mk, const double* start, const double* goal, const double* tube_lo,
               const double* tube_hi, double eps, int pos_only, int require_tube, std::vector<int64_t>& path,
               double* dist);

// A search whose launches read start/goal from pinned staging (PathStage): enqueue is
// capturable; collect reads the result after the stream synchronised.
struct PathStage;
PathStage* path_stage_create(const Graph* g, const double* tube_lo, const double* tube_hi, double eps, int pos_only,
                             int require_tube);
void path_stage_set(PathStage* s, const Graph* g, const double* start, const double* goal);
void path_stage_enqueue(Ctx* c, Graph* g, Mask* mk, PathStage* s);
void path_stage_collect(Ctx* c, const Graph* g, PathStage* s, std::vector<int64_t>& path, double* dist);
void path_stage_destroy(PathStage* s);

// A find_path on a fixed (graph, mask) captured as a CUDA graph (bzg_query): start and goal go
// through pinned host memory, so a query is one graph launch and one synchronisation.
struct Query;
struct Replanner;
struct Planner;
Planner* planner_create(Ctx* c, const bzg_build_desc* d, const bzg_region_sampler* rsam, int n_obs,
                        const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box,
                        const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
                        const double* tube_lo, const double* tube_hi, double eps, int pos_only, int require_tube);
void planner_run(Planner* p, const uint64_t* pcg, const double* include, int n_obs, const int32_t* row_off,
                 const double* A, const double* b, const uint8_t* is_box, const double* box_lo,
                 const double* box_hi, const double* start, const double* goal, std::vector<int64_t>& path,
                 double* dist, int* eager_out);
void planner_destroy(Planner* p);
Ctx* planner_ctx(const Planner* p);
Graph* planner_graph(Planner* p);
const Mask* planner_mask(const Planner* p);
void planner_info(const Planner* p, int64_t info[6]);
Replanner* replanner_create(Ctx* c, Graph* g, int n_obs, const int32_t* row_off, const double* A, const double* b,
                            const uint8_t* is_box, const double* box_lo, const double* box_hi,
                            const uint8_t* dynamic, const bzg_cut_config* cfg, const double* tube_lo,
                            const double* tube_hi, double eps, int pos_only, int require_tube);
void replanner_run(Replanner* r, int n_obs, const int32_t* row_off, const double* A, const double* b,
                   const uint8_t* is_box, const double* box_lo, const double* box_hi, const double* start,
                   const double* goal, std::vector<int64_t>& path, double* dist, int* eager_out);
void replanner_destroy(Replanner* r);
Ctx* replanner_ctx(const Replanner* r);
const Mask* replanner_mask(const Replanner* r);
void replanner_info(const Replanner* r, int64_t info[4]);
Query* query_create(Ctx* c, Graph* g, Mask* mk, const double* tube_lo, const double* tube_hi, double eps,
                    int pos_only, int require_tube);
void query_run(Query* q, const double* start, const double* goal, std::vector<int64_t>& path, double* dist);
void query_destroy(Query* q);
long long query_kernels(const Query* q);
Ctx* query_ctx(const Query* q);

}  // namespace bzg
