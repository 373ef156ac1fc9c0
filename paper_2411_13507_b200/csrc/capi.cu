// extern "C" boundary of libbzg (declarations and reference citations in include/bzg.h).
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "bzg_internal.cuh"

using namespace bzg;

struct bzg_ctx : Ctx {};
struct bzg_graph : Graph {};
struct bzg_mask : Mask {};
// bzg_query is opaque here (Query is defined with the search, k_sssp.cu)
static Query* as_query(bzg_query* q) { return reinterpret_cast<Query*>(q); }
static const Query* as_query(const bzg_query* q) { return reinterpret_cast<const Query*>(q); }
static Replanner* as_rp(bzg_replanner* r) { return reinterpret_cast<Replanner*>(r); }
static Planner* as_pl(bzg_planner* p) { return reinterpret_cast<Planner*>(p); }
static const Planner* as_pl(const bzg_planner* p) { return reinterpret_cast<const Planner*>(p); }
static const Replanner* as_rp(const bzg_replanner* r) { return reinterpret_cast<const Replanner*>(r); }

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return BZG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return BZG_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BZG_EINVAL;
  }
}

void set_device(Ctx* c) { BZG_CHECK_CUDA(cudaSetDevice(c->device)); }

}  // namespace

extern "C" {

int bzg_abi_version(void) { return BZG_ABI_VERSION; }

const char* bzg_last_error(void) { return g_last_error.c_str(); }

int bzg_ctx_create(int device, void* stream, bzg_ctx** out) {
  return guarded([&] {
    BZG_REQUIRE(out, BZG_EINVAL, "null output pointer");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    BZG_REQUIRE(e == cudaSuccess && ndev > 0, BZG_ENODEV,
                std::string("no CUDA device available: ") + cudaGetErrorString(e));
    BZG_REQUIRE(device >= 0 && device < ndev, BZG_ENODEV, "device ordinal out of range");
    cudaDeviceProp prop;
    BZG_CHECK_CUDA(cudaGetDeviceProperties(&prop, device));
    BZG_REQUIRE(prop.major == 10, BZG_ENODEV,
                std::string("libbzg is built for sm_100a (B200); device is ") + prop.name);
    auto* c = new bzg_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    BZG_CHECK_CUDA(cudaSetDevice(device));
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
      c->own_stream = false;
    } else {
      BZG_CHECK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    // keep freed pool memory cached across builds (stream-ordered allocator)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
  });
}

int bzg_ctx_destroy(bzg_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    set_device(ctx);
    cudaStreamSynchronize(ctx->stream);
    ctx->flag.release();
    for (auto& w : ctx->ws_own) w.release();
    ctx->arena_own.chunks.clear();
    ctx->drain_profile();
    for (auto e : ctx->spare) cudaEventDestroy(e);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

int bzg_ctx_stream(bzg_ctx* ctx, void** stream_out) {
  return guarded([&] {
    BZG_REQUIRE(ctx && stream_out, BZG_EINVAL, "null argument");
    *stream_out = ctx->stream;
  });
}

int bzg_ctx_synchronize(bzg_ctx* ctx) {
  return guarded([&] {
    BZG_REQUIRE(ctx, BZG_EINVAL, "null context");
    set_device(ctx);
    BZG_CHECK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int bzg_ctx_set_profiling(bzg_ctx* ctx, int enabled) {
  return guarded([&] {
    BZG_REQUIRE(ctx, BZG_EINVAL, "null context");
    ctx->profiling = enabled != 0;
  });
}

int bzg_ctx_profile_only(bzg_ctx* ctx, const char* kernel) {
  return guarded([&] {
    BZG_REQUIRE(ctx, BZG_EINVAL, "null context");
    ctx->profile_only = kernel ? kernel : "";
  });
}

int bzg_ctx_stats(bzg_ctx* ctx, long long* launches, int n_cap, char* names, double* ms, long long* counts,
                  int* n_out) {
  return guarded([&] {
    BZG_REQUIRE(ctx, BZG_EINVAL, "null context");
    set_device(ctx);
    ctx->drain_profile();
    if (launches) *launches = ctx->launches;
    const int n = (int)ctx->order.size();
    if (n_out) *n_out = n;
    for (int i = 0; i < n && i < n_cap; ++i) {
      const auto& s = ctx->stats[ctx->order[i]];
      if (names) {
        std::strncpy(names + 64 * i, ctx->order[i].c_str(), 63);
        names[64 * i + 63] = 0;
      }
      if (ms) ms[i] = s.ms;
      if (counts) counts[i] = s.count;
    }
  });
}

int bzg_ctx_reset_stats(bzg_ctx* ctx) {
  return guarded([&] {
    BZG_REQUIRE(ctx, BZG_EINVAL, "null context");
    set_device(ctx);
    ctx->drain_profile();
    ctx->stats.clear();
    ctx->order.clear();
    ctx->launches = 0;
  });
}

int bzg_build_graph(bzg_ctx* ctx, const bzg_build_desc* d, bzg_graph** out) {
  bzg_graph* g = nullptr;
  int rc = guarded([&] {
    NvtxRange nvtx_range("bzg_build_graph");
    BZG_REQUIRE(ctx && d && out, BZG_EINVAL, "null argument");
    set_device(ctx);
    BZG_REQUIRE(d->m >= 1 && d->gamma >= 1, BZG_EINVAL, "require m >= 1 and gamma >= 1");
    BZG_REQUIRE(d->p == 2 * d->gamma - 1, BZG_EINVAL, "boundary-value curves require p = 2*gamma - 1");
    BZG_REQUIRE(d->N >= 2, BZG_EINVAL, "need at least two vertices");  // graph.py:143-144
    BZG_REQUIRE(d->F && d->G && d->D, BZG_EINVAL, "oracle F, G and boundary matrix D are required");
    BZG_REQUIRE(d->n_include >= 0 && (d->n_include == 0 || d->include), BZG_EINVAL, "include rows missing");
    const int n = d->m * d->gamma;
    ctx->sample_check = nullptr;
    ctx->trace("build: enter");
    g = new bzg_graph();
    g->ctx = ctx;
    g->m = d->m;
    g->gamma = d->gamma;
    g->p = d->p;
    g->n = n;
    g->V = d->N + d->n_include;
    g->row_begin = d->row_begin;
    g->row_end = d->row_end > 0 ? d->row_end : g->V;
    BZG_REQUIRE(g->row_begin >= 0 && g->row_begin <= g->row_end && g->row_end <= g->V, BZG_EINVAL,
                "row block out of range");
    BZG_REQUIRE(g->V < (1ll << 31), BZG_EUNSUPPORTED, "vertex count exceeds int32 indexing");
    g->D.assign(d->D, d->D + (size_t)(d->p + 1) * 2 * d->gamma);
    g->vertices.alloc((size_t)g->V * n * sizeof(double), ctx->stream);
    if (d->vertices) {
      BZG_CHECK_CUDA(cudaMemcpyAsync(g->vertices.ptr, d->vertices, (size_t)d->N * n * sizeof(double),
                                     cudaMemcpyHostToDevice, ctx->stream));
    } else {
      BZG_REQUIRE(d->sample_lo && d->sample_hi && d->xd_A && d->xd_b, BZG_EINVAL, "sampler inputs missing");
      sample_states(ctx, d, g->vertices.as<double>(), /*single_round=*/true);
    }
    if (d->n_include > 0)
      BZG_CHECK_CUDA(cudaMemcpyAsync(g->vertices.as<double>() + (size_t)d->N * n, d->include,
                                     (size_t)d->n_include * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->trace("build: vertices");
    if (!build_pairs(ctx, d, g)) {  // the one sampler round fell short: checked rounds, then again
      ctx->trace("build: resample");
      sample_states(ctx, d, g->vertices.as<double>());
      build_pairs(ctx, d, g);
    }
    ctx->trace("build: pairs+csr");
  });
  if (rc == BZG_OK) {
    *out = g;
  } else {
    delete g;
  }
  return rc;
}

int bzg_graph_eps_band(bzg_graph* g, const bzg_build_desc* d, double eps, int64_t counts[3]) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_graph_eps_band");
    BZG_REQUIRE(g && d && counts && d->F && d->G, BZG_EINVAL, "null argument");
    BZG_REQUIRE(eps >= 0.0, BZG_EINVAL, "eps must be non-negative");
    BZG_REQUIRE(d->m == g->m && d->gamma == g->gamma && d->N + d->n_include == g->V, BZG_EINVAL,
                "descriptor does not describe this graph");
    set_device(g->ctx);
    g->ctx->sample_check = nullptr;
    long long plus = 0, minus = 0;
    build_pairs(g->ctx, d, g, eps, &plus);
    build_pairs(g->ctx, d, g, -eps, &minus);
    counts[0] = plus - minus;
    counts[1] = plus;
    counts[2] = minus;
  });
}

int bzg_sample_states(bzg_ctx* ctx, const bzg_build_desc* d, double* out_host) {
  return guarded([&] {
    BZG_REQUIRE(ctx && d && out_host, BZG_EINVAL, "null argument");
    BZG_REQUIRE(d->m >= 1 && d->gamma >= 1 && d->N >= 0, BZG_EINVAL, "bad sampler dimensions");
    BZG_REQUIRE(d->sample_lo && d->sample_hi && d->xd_A && d->xd_b, BZG_EINVAL, "sampler inputs missing");
    set_device(ctx);
    if (d->N == 0) return;
    const int n = d->m * d->gamma;
    DevBuf out;
    out.alloc((size_t)d->N * n * sizeof(double), ctx->stream);
    sample_states(ctx, d, out.as<double>());
    BZG_CHECK_CUDA(cudaMemcpyAsync(out_host, out.ptr, (size_t)d->N * n * sizeof(double), cudaMemcpyDeviceToHost,
                                   ctx->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int bzg_sample_region_states(bzg_ctx* ctx, int32_t n, int32_t n_regions, const int64_t* N, const uint64_t* pcg,
                             const double* lo, const double* hi, const int32_t* row_off, const double* A,
                             const double* b, double eps_geo, double* out_host) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_sample_region_states");
    BZG_REQUIRE(ctx && N && pcg && lo && hi && row_off && A && b && out_host, BZG_EINVAL, "null argument");
    BZG_REQUIRE(n_regions >= 1, BZG_EINVAL, "need at least one region");
    long long total = 0;
    for (int r = 0; r < n_regions; ++r) {
      BZG_REQUIRE(N[r] >= 0, BZG_EINVAL, "negative sample count");
      BZG_REQUIRE(row_off[r + 1] > row_off[r], BZG_EINVAL, "every region needs state-set rows");
      total += N[r];
    }
    set_device(ctx);
    if (total == 0) return;
    ctx->trace("sample_regions: enter");
    DevBuf out;
    out.alloc((size_t)total * n * sizeof(double), ctx->stream);
    sample_regions(ctx, n, n_regions, N, pcg, lo, hi, row_off, A, b, eps_geo, out.as<double>());
    ctx->trace("sample_regions: done");
    BZG_CHECK_CUDA(cudaMemcpyAsync(out_host, out.ptr, (size_t)total * n * sizeof(double), cudaMemcpyDeviceToHost,
                                   ctx->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int bzg_graph_from_edges(bzg_ctx* ctx, int32_t m, int32_t gamma, int32_t p, const double* D, int64_t V,
                         const double* vertices_host, int64_t E, const int32_t* src, const int32_t* dst,
                         const double* cost, int on_device, bzg_graph** out) {
  bzg_graph* g = nullptr;
  int rc = guarded([&] {
    BZG_REQUIRE(ctx && D && vertices_host && out, BZG_EINVAL, "null argument");
    BZG_REQUIRE(m >= 1 && gamma >= 1 && p == 2 * gamma - 1, BZG_EINVAL, "boundary-value curves require p = 2*gamma - 1");
    BZG_REQUIRE(V >= 1 && V < (1ll << 31), BZG_EINVAL, "vertex count out of range");
    set_device(ctx);
    g = new bzg_graph();
    g->ctx = ctx;
    g->m = m; g->gamma = gamma; g->p = p; g->n = m * gamma;
    g->V = V;
    g->D.assign(D, D + (size_t)(p + 1) * 2 * gamma);
    g->vertices.alloc((size_t)V * g->n * sizeof(double), ctx->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(g->vertices.ptr, vertices_host, (size_t)V * g->n * sizeof(double),
                                   cudaMemcpyHostToDevice, ctx->stream));
    set_edges(ctx, g, E, src, dst, cost, on_device != 0);
  });
  if (rc == BZG_OK) *out = g; else delete g;
  return rc;
}

int bzg_graph_with_edges(const bzg_graph* like, int64_t E, const int32_t* src, const int32_t* dst,
                         const double* cost, int on_device, bzg_graph** out) {
  bzg_graph* g = nullptr;
  int rc = guarded([&] {
    BZG_REQUIRE(like && out && (E == 0 || (src && dst && cost)), BZG_EINVAL, "null argument");
    Ctx* ctx = like->ctx;
    set_device(ctx);
    g = new bzg_graph();
    g->ctx = ctx;
    g->m = like->m; g->gamma = like->gamma; g->p = like->p; g->n = like->n;
    g->V = like->V;
    g->D = like->D;
    g->vertices.alloc((size_t)g->V * g->n * sizeof(double), ctx->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(g->vertices.ptr, like->vertices.ptr, (size_t)g->V * g->n * sizeof(double),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
    set_edges(ctx, g, E, src, dst, cost, on_device != 0);
  });
  if (rc == BZG_OK) *out = g; else delete g;
  return rc;
}

int bzg_graph_set_edges(bzg_graph* g, int64_t E, const int32_t* src, const int32_t* dst, const double* cost,
                        int on_device) {
  return guarded([&] {
    BZG_REQUIRE(g && (E == 0 || (src && dst && cost)), BZG_EINVAL, "null argument");
    set_device(g->ctx);
    set_edges(g->ctx, g, E, src, dst, cost, on_device != 0);
  });
}

int bzg_graph_set_cut_cache(bzg_graph* g, int32_t max_obstacles) {
  return guarded([&] {
    BZG_REQUIRE(g && max_obstacles >= 0, BZG_EINVAL, "bad argument");
    set_device(g->ctx);
    CutCache& cc = g->cut_cache;
    cc.clear();
    cc.max_slots = max_obstacles;
    cc.Wb = 0;
    cc.key_of.clear();
    if (max_obstacles == 0) cc.pool.release();
  });
}

int bzg_graph_destroy(bzg_graph* g) {
  return guarded([&] {
    if (!g) return;
    set_device(g->ctx);
    delete g;
  });
}

int bzg_graph_info(const bzg_graph* g, int64_t* V, int64_t* E, int64_t* row_begin, int64_t* row_end) {
  return guarded([&] {
    BZG_REQUIRE(g, BZG_EINVAL, "null graph");
    if (V) *V = g->V;
    if (E) *E = g->E;
    if (row_begin) *row_begin = g->row_begin;
    if (row_end) *row_end = g->row_end;
  });
}

int bzg_graph_copy_vertices(bzg_graph* g, double* vertices) {
  return guarded([&] {
    BZG_REQUIRE(g, BZG_EINVAL, "null graph");
    set_device(g->ctx);
    if (vertices)
      BZG_CHECK_CUDA(cudaMemcpyAsync(vertices, g->vertices.ptr, (size_t)g->V * g->n * sizeof(double),
                                     cudaMemcpyDeviceToHost, g->ctx->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  });
}

int bzg_graph_copy_edges(bzg_graph* g, int64_t* edges, double* costs) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_graph_copy_edges");
    BZG_REQUIRE(g, BZG_EINVAL, "null graph");
    set_device(g->ctx);
    const long long E = g->E;
    if (edges && E > 0) {
      std::vector<int> s(E), t(E);
      BZG_CHECK_CUDA(cudaMemcpyAsync(s.data(), g->src.ptr, E * sizeof(int), cudaMemcpyDeviceToHost, g->ctx->stream));
      BZG_CHECK_CUDA(cudaMemcpyAsync(t.data(), g->dst.ptr, E * sizeof(int), cudaMemcpyDeviceToHost, g->ctx->stream));
      BZG_CHECK_CUDA(cudaStreamSynchronize(g->ctx->stream));
      for (long long e = 0; e < E; ++e) {
        edges[2 * e] = s[e];
        edges[2 * e + 1] = t[e];
      }
    }
    if (costs && E > 0)
      BZG_CHECK_CUDA(cudaMemcpyAsync(costs, g->cost.ptr, E * sizeof(double), cudaMemcpyDeviceToHost, g->ctx->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  });
}

int bzg_graph_copy_points(bzg_graph* g, double* points) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_graph_copy_points");
    BZG_REQUIRE(g, BZG_EINVAL, "null graph");
    set_device(g->ctx);
    materialize_points(g->ctx, g);
    if (points && g->E > 0)
      BZG_CHECK_CUDA(cudaMemcpyAsync(points, g->points.ptr, (size_t)g->E * g->m * (g->p + 1) * sizeof(double),
                                     cudaMemcpyDeviceToHost, g->ctx->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  });
}

int bzg_graph_copy_csr(bzg_graph* g, int64_t* row_ptr, int32_t* col) {
  return guarded([&] {
    BZG_REQUIRE(g, BZG_EINVAL, "null graph");
    set_device(g->ctx);
    if (row_ptr)
      BZG_CHECK_CUDA(cudaMemcpyAsync(row_ptr, g->row_ptr.ptr, (g->V + 1) * sizeof(long long), cudaMemcpyDeviceToHost,
                                     g->ctx->stream));
    if (col && g->E > 0)
      BZG_CHECK_CUDA(cudaMemcpyAsync(col, g->dst.ptr, g->E * sizeof(int), cudaMemcpyDeviceToHost, g->ctx->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  });
}

int bzg_graph_export_device(bzg_graph* g, int32_t* src, int32_t* dst, double* cost) {
  return guarded([&] {
    BZG_REQUIRE(g, BZG_EINVAL, "null graph");
    set_device(g->ctx);
    const long long E = g->E;
    if (E > 0) {
      if (src) BZG_CHECK_CUDA(cudaMemcpyAsync(src, g->src.ptr, E * 4, cudaMemcpyDeviceToDevice, g->ctx->stream));
      if (dst) BZG_CHECK_CUDA(cudaMemcpyAsync(dst, g->dst.ptr, E * 4, cudaMemcpyDeviceToDevice, g->ctx->stream));
      if (cost) BZG_CHECK_CUDA(cudaMemcpyAsync(cost, g->cost.ptr, E * 8, cudaMemcpyDeviceToDevice, g->ctx->stream));
    }
    BZG_CHECK_CUDA(cudaStreamSynchronize(g->ctx->stream));
  });
}

int bzg_check_edges(bzg_ctx* ctx, int32_t n, int32_t n_F, const double* F, const double* G, double eps, int64_t k,
                    const double* X1, const double* X2, uint8_t* out) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_check_edges");
    BZG_REQUIRE(ctx && F && G && (k == 0 || (X1 && X2 && out)), BZG_EINVAL, "null argument");
    set_device(ctx);
    check_edges(ctx, n, n_F, F, G, eps, k, X1, X2, out);
  });
}

int bzg_cut_graph(bzg_ctx* ctx, bzg_graph* g, int32_t n_obs, const int32_t* row_off, const double* A, const double* b,
                  const uint8_t* is_box, const double* box_lo, const double* box_hi, const bzg_cut_config* cfg,
                  bzg_mask** out) {
  bzg_mask* mk = nullptr;
  int rc = guarded([&] {
    NvtxRange nvtx_range("bzg_cut_graph");
    BZG_REQUIRE(ctx && g && cfg && out, BZG_EINVAL, "null argument");
    BZG_REQUIRE(n_obs == 0 || (row_off && A && b && is_box && box_lo && box_hi), BZG_EINVAL, "obstacle arrays missing");
    set_device(ctx);
    mk = new bzg_mask();
    cut_graph(ctx, g, n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg, mk);
  });
  if (rc == BZG_OK) *out = mk; else delete mk;
  return rc;
}

int bzg_cut_points(bzg_ctx* ctx, int32_t m, int32_t J, int64_t B, const double* points, const int32_t* obs_index,
                   int32_t n_obs, const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box,
                   const double* box_lo, const double* box_hi, const bzg_cut_config* cfg, int32_t mode, int8_t* code,
                   double* delta, int8_t* status) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_cut_points");
    BZG_REQUIRE(ctx && cfg && code && (B == 0 || (points && obs_index)), BZG_EINVAL, "null argument");
    BZG_REQUIRE(row_off && A && b && is_box && box_lo && box_hi, BZG_EINVAL, "obstacle arrays missing");
    BZG_REQUIRE(m >= 1 && m <= 3, BZG_EUNSUPPORTED, "device cut supports m in 1..3");
    set_device(ctx);
    cut_points(ctx, m, J, B, points, obs_index, n_obs, row_off, A, b, is_box, box_lo, box_hi, cfg, mode, code, delta,
               status);
  });
}

int bzg_mask_destroy(bzg_mask* mk) {
  return guarded([&] {
    if (!mk) return;
    if (mk->ctx) set_device(mk->ctx);  // not via mk->g: the graph may already be released
    delete mk;
  });
}

int bzg_mask_copy(bzg_mask* mk, uint8_t* alive, uint8_t* provenance, int64_t counters[6]) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_mask_copy");
    BZG_REQUIRE(mk && mk->g, BZG_EINVAL, "null mask");
    BZG_REQUIRE((!alive && !provenance) || mk->E == mk->g->E, BZG_EINVAL,
                "stale mask: its graph's edge set changed after the cut");
    Ctx* c = mk->g->ctx;
    set_device(c);
    if (alive && mk->E > 0) BZG_CHECK_CUDA(cudaMemcpyAsync(alive, mk->alive.ptr, mk->E, cudaMemcpyDeviceToHost, c->stream));
    if (provenance && mk->E > 0)
      BZG_CHECK_CUDA(cudaMemcpyAsync(provenance, mk->prov.ptr, mk->E, cudaMemcpyDeviceToHost, c->stream));
    if (counters)
      for (int i = 0; i < 6; ++i) counters[i] = mk->counters[i];
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bzg_mask_info(const bzg_mask* mk, int64_t* E, int64_t* n_qp) {
  return guarded([&] {
    BZG_REQUIRE(mk, BZG_EINVAL, "null mask");
    if (E) *E = mk->E;
    if (n_qp) *n_qp = mk->n_qp;
  });
}

int bzg_mask_qp_count(bzg_mask* mk, int64_t* n) {
  return guarded([&] {
    BZG_REQUIRE(mk && n, BZG_EINVAL, "null argument");
    *n = mk->n_qp;
  });
}

int bzg_mask_copy_qp(bzg_mask* mk, int64_t* edge, int32_t* obstacle, int8_t* status, int32_t* iters, double* delta) {
  return guarded([&] {
    BZG_REQUIRE(mk && mk->g, BZG_EINVAL, "null mask");
    Ctx* c = mk->g->ctx;
    set_device(c);
    const long long n = mk->n_qp;
    if (n > 0) {
      if (edge) BZG_CHECK_CUDA(cudaMemcpyAsync(edge, mk->qp_edge.ptr, n * 8, cudaMemcpyDeviceToHost, c->stream));
      if (obstacle) BZG_CHECK_CUDA(cudaMemcpyAsync(obstacle, mk->qp_obs.ptr, n * 4, cudaMemcpyDeviceToHost, c->stream));
      if (status) BZG_CHECK_CUDA(cudaMemcpyAsync(status, mk->qp_status.ptr, n, cudaMemcpyDeviceToHost, c->stream));
      if (iters) BZG_CHECK_CUDA(cudaMemcpyAsync(iters, mk->qp_iters.ptr, n * 4, cudaMemcpyDeviceToHost, c->stream));
      if (delta) BZG_CHECK_CUDA(cudaMemcpyAsync(delta, mk->qp_delta.ptr, n * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bzg_mask_from_arrays(bzg_ctx* ctx, bzg_graph* g, const uint8_t* alive, const uint8_t* provenance,
                         const int64_t counters[6], int on_device, bzg_mask** out) {
  bzg_mask* mk = nullptr;
  int rc = guarded([&] {
    BZG_REQUIRE(ctx && g && alive && out, BZG_EINVAL, "null argument");
    set_device(ctx);
    mk = new bzg_mask();
    mk->g = g;
    mk->ctx = ctx;
    mk->E = g->E;
    const auto kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    mk->alive.alloc(std::max<long long>(g->E, 1), ctx->stream);
    mk->prov.alloc(std::max<long long>(g->E, 1), ctx->stream);
    if (g->E > 0) {
      BZG_CHECK_CUDA(cudaMemcpyAsync(mk->alive.ptr, alive, g->E, kind, ctx->stream));
      if (provenance) BZG_CHECK_CUDA(cudaMemcpyAsync(mk->prov.ptr, provenance, g->E, kind, ctx->stream));
      else BZG_CHECK_CUDA(cudaMemsetAsync(mk->prov.ptr, BZG_HEURISTIC_SAFE, g->E, ctx->stream));
    }
    if (counters)
      for (int i = 0; i < 6; ++i) mk->counters[i] = counters[i];
    BZG_CHECK_CUDA(cudaStreamSynchronize(ctx->stream));
  });
  if (rc == BZG_OK) *out = mk; else delete mk;
  return rc;
}

int bzg_mask_export_device(bzg_mask* mk, uint8_t* alive, uint8_t* provenance) {
  return guarded([&] {
    BZG_REQUIRE(mk && mk->g, BZG_EINVAL, "null mask");
    BZG_REQUIRE(mk->E == mk->g->E, BZG_EINVAL, "stale mask: its graph's edge set changed after the cut");
    Ctx* c = mk->g->ctx;
    set_device(c);
    if (mk->E > 0) {
      if (alive) BZG_CHECK_CUDA(cudaMemcpyAsync(alive, mk->alive.ptr, mk->E, cudaMemcpyDeviceToDevice, c->stream));
      if (provenance) BZG_CHECK_CUDA(cudaMemcpyAsync(provenance, mk->prov.ptr, mk->E, cudaMemcpyDeviceToDevice, c->stream));
    }
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int bzg_project_on_path(bzg_ctx* ctx, int32_t m, int32_t gamma, double T, const double* D, int64_t L,
                        const double* path_states, double h, int32_t steps_per_hop, const double* state,
                        double* best_t) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_project_on_path");
    BZG_REQUIRE(ctx && D && state && best_t && (L == 0 || path_states), BZG_EINVAL, "null argument");
    set_device(ctx);
    *best_t = project_on_path(ctx, m, gamma, T, D, L, path_states, h, steps_per_hop, state);
  });
}

int bzg_find_path(bzg_ctx* ctx, bzg_graph* g, bzg_mask* mk, const double* start, const double* goal,
                  const double* tube_lo, const double* tube_hi, double eps_geo, int position_only_snap,
                  int require_tube_snap, int64_t* path_out, int64_t path_cap, int64_t* path_len, double* dist_out) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_find_path");
    BZG_REQUIRE(ctx && g && start && goal && tube_lo && tube_hi && path_len, BZG_EINVAL, "null argument");
    BZG_REQUIRE(!mk || mk->g == g, BZG_EINVAL, "mask belongs to another graph");
    BZG_REQUIRE(!mk || mk->E == g->E, BZG_EINVAL, "stale mask: its graph's edge set changed after the cut");
    set_device(ctx);
    std::vector<int64_t> path;
    double dist = 0.0;
    find_path(ctx, g, mk, start, goal, tube_lo, tube_hi, eps_geo, position_only_snap, require_tube_snap, path, &dist);
    if (path.empty()) {
      *path_len = -1;
    } else {
      *path_len = (int64_t)path.size();
      BZG_REQUIRE(path_out && path_cap >= (int64_t)path.size(), BZG_EINVAL, "path buffer too small");
      std::memcpy(path_out, path.data(), path.size() * sizeof(int64_t));
    }
    if (dist_out) *dist_out = dist;
  });
}

int bzg_query_create(bzg_ctx* ctx, bzg_graph* g, bzg_mask* mk, const double* tube_lo, const double* tube_hi,
                     double eps_geo, int position_only_snap, int require_tube_snap, bzg_query** out) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_query_create");
    BZG_REQUIRE(ctx && g && tube_lo && tube_hi && out, BZG_EINVAL, "null argument");
    BZG_REQUIRE(!mk || mk->g == g, BZG_EINVAL, "mask belongs to another graph");
    BZG_REQUIRE(!mk || mk->E == g->E, BZG_EINVAL, "stale mask: its graph's edge set changed after the cut");
    set_device(ctx);
    *out = reinterpret_cast<bzg_query*>(
        query_create(ctx, g, mk, tube_lo, tube_hi, eps_geo, position_only_snap, require_tube_snap));
  });
}

int bzg_query_run(bzg_query* q, const double* start, const double* goal, int64_t* path_out, int64_t path_cap,
                  int64_t* path_len, double* dist_out) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_query_run");
    BZG_REQUIRE(q && start && goal && path_len, BZG_EINVAL, "null argument");
    set_device(query_ctx(as_query(q)));
    std::vector<int64_t> path;
    double dist = 0.0;
    query_run(as_query(q), start, goal, path, &dist);
    if (path.empty()) {
      *path_len = -1;
    } else {
      *path_len = (int64_t)path.size();
      BZG_REQUIRE(path_out && path_cap >= (int64_t)path.size(), BZG_EINVAL, "path buffer too small");
      std::memcpy(path_out, path.data(), path.size() * sizeof(int64_t));
    }
    if (dist_out) *dist_out = dist;
  });
}

int bzg_query_kernels(const bzg_query* q, int64_t* n) {
  return guarded([&] {
    BZG_REQUIRE(q && n, BZG_EINVAL, "null argument");
    *n = query_kernels(as_query(q));
  });
}

int bzg_query_destroy(bzg_query* q) {
  return guarded([&] {
    if (!q) return;
    set_device(query_ctx(as_query(q)));
    query_destroy(as_query(q));
  });
}

int bzg_replanner_create(bzg_ctx* ctx, bzg_graph* g, int32_t n_obs, const int32_t* row_off, const double* A,
                         const double* b, const uint8_t* is_box, const double* box_lo, const double* box_hi,
                         const uint8_t* dynamic, const bzg_cut_config* cfg, const double* tube_lo, const double* tube_hi, double eps_geo,
                         int position_only_snap, int require_tube_snap, bzg_replanner** out) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_replanner_create");
    BZG_REQUIRE(ctx && g && cfg && tube_lo && tube_hi && out, BZG_EINVAL, "null argument");
    BZG_REQUIRE(row_off && A && b && is_box && box_lo && box_hi, BZG_EINVAL, "obstacle arrays missing");
    set_device(ctx);
    *out = reinterpret_cast<bzg_replanner*>(replanner_create(ctx, g, n_obs, row_off, A, b, is_box, box_lo, box_hi,
                                                             dynamic, cfg, tube_lo, tube_hi, eps_geo, position_only_snap,
                                                             require_tube_snap));
  });
}

int bzg_replanner_run(bzg_replanner* rp, int32_t n_obs, const int32_t* row_off, const double* A, const double* b,
                      const uint8_t* is_box, const double* box_lo, const double* box_hi, const double* start,
                      const double* goal, int64_t* path_out, int64_t path_cap, int64_t* path_len, double* dist_out,
                      int64_t counters[6], int32_t* eager) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_replanner_run");
    BZG_REQUIRE(rp && start && goal && path_len, BZG_EINVAL, "null argument");
    BZG_REQUIRE(row_off && A && b && is_box && box_lo && box_hi, BZG_EINVAL, "obstacle arrays missing");
    Replanner* r = as_rp(rp);
    set_device(replanner_ctx(r));
    std::vector<int64_t> path;
    double dist = 0.0;
    int eg = 0;
    replanner_run(r, n_obs, row_off, A, b, is_box, box_lo, box_hi, start, goal, path, &dist, &eg);
    if (path.empty()) {
      *path_len = -1;
    } else {
      *path_len = (int64_t)path.size();
      BZG_REQUIRE(path_out && path_cap >= (int64_t)path.size(), BZG_EINVAL, "path buffer too small");
      std::memcpy(path_out, path.data(), path.size() * sizeof(int64_t));
    }
    if (dist_out) *dist_out = dist;
    if (counters)
      for (int i = 0; i < 6; ++i) counters[i] = replanner_mask(r)->counters[i];
    if (eager) *eager = eg;
  });
}

int bzg_replanner_mask(bzg_replanner* rp, bzg_mask** out) {
  bzg_mask* mk = nullptr;
  int rc = guarded([&] {
    BZG_REQUIRE(rp && out, BZG_EINVAL, "null argument");
    const Replanner* r = as_rp(rp);
    Ctx* c = replanner_ctx(r);
    set_device(c);
    const Mask* src = replanner_mask(r);
    mk = new bzg_mask();
    mk->g = src->g;
    mk->ctx = c;
    mk->E = src->E;
    mk->n_obs = src->n_obs;
    for (int i = 0; i < 6; ++i) mk->counters[i] = src->counters[i];
    mk->alive.alloc(std::max<long long>(src->E, 1), c->stream);
    mk->prov.alloc(std::max<long long>(src->E, 1), c->stream);
    if (src->E > 0) {
      BZG_CHECK_CUDA(cudaMemcpyAsync(mk->alive.ptr, src->alive.ptr, src->E, cudaMemcpyDeviceToDevice, c->stream));
      BZG_CHECK_CUDA(cudaMemcpyAsync(mk->prov.ptr, src->prov.ptr, src->E, cudaMemcpyDeviceToDevice, c->stream));
    }
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  });
  if (rc == BZG_OK) *out = mk; else delete mk;
  return rc;
}

int bzg_replanner_info(const bzg_replanner* rp, int64_t info[4]) {
  return guarded([&] {
    BZG_REQUIRE(rp && info, BZG_EINVAL, "null argument");
    replanner_info(as_rp(rp), info);
  });
}

int bzg_replanner_destroy(bzg_replanner* rp) {
  return guarded([&] {
    if (!rp) return;
    Replanner* r = as_rp(rp);
    set_device(replanner_ctx(r));
    replanner_destroy(r);
  });
}

int bzg_planner_create(bzg_ctx* ctx, const bzg_build_desc* desc, const bzg_region_sampler* regions, int32_t n_obs,
                       const int32_t* row_off,
                       const double* A, const double* b, const uint8_t* is_box, const double* box_lo,
                       const double* box_hi, const bzg_cut_config* cfg, const double* tube_lo, const double* tube_hi,
                       double eps_geo, int position_only_snap, int require_tube_snap, bzg_planner** out) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_planner_create");
    BZG_REQUIRE(ctx && desc && cfg && tube_lo && tube_hi && out, BZG_EINVAL, "null argument");
    BZG_REQUIRE(n_obs == 0 || (row_off && A && b && is_box && box_lo && box_hi), BZG_EINVAL, "obstacle arrays missing");
    BZG_REQUIRE(desc->n_include == 0 || desc->include, BZG_EINVAL, "include rows missing");
    set_device(ctx);
    *out = reinterpret_cast<bzg_planner*>(planner_create(ctx, desc, regions, n_obs, row_off, A, b, is_box, box_lo,
                                                         box_hi, cfg, tube_lo, tube_hi, eps_geo, position_only_snap,
                                                         require_tube_snap));
  });
}

int bzg_planner_run(bzg_planner* pl, const uint64_t* pcg, const double* include, int32_t n_obs,
                    const int32_t* row_off, const double* A, const double* b, const uint8_t* is_box,
                    const double* box_lo, const double* box_hi, const double* start, const double* goal,
                    int64_t* path_out, int64_t path_cap, int64_t* path_len, double* dist_out, int64_t counters[6],
                    int64_t* num_edges, int32_t* eager) {
  return guarded([&] {
    NvtxRange nvtx_range("bzg_planner_run");
    BZG_REQUIRE(pl && pcg && start && goal && path_len, BZG_EINVAL, "null argument");
    BZG_REQUIRE(n_obs == 0 || (row_off && A && b && is_box && box_lo && box_hi), BZG_EINVAL, "obstacle arrays missing");
    Planner* p = as_pl(pl);
    set_device(planner_ctx(p));
    std::vector<int64_t> path;
    double dist = 0.0;
    int eg = 0;
    planner_run(p, pcg, include, n_obs, row_off, A, b, is_box, box_lo, box_hi, start, goal, path, &dist, &eg);
    if (path.empty()) {
      *path_len = -1;
    } else {
      *path_len = (int64_t)path.size();
      BZG_REQUIRE(path_out && path_cap >= (int64_t)path.size(), BZG_EINVAL, "path buffer too small");
      std::memcpy(path_out, path.data(), path.size() * sizeof(int64_t));
    }
    if (dist_out) *dist_out = dist;
    if (counters)
      for (int i = 0; i < 6; ++i) counters[i] = planner_mask(p)->counters[i];
    if (num_edges) *num_edges = planner_graph(p)->E;
    if (eager) *eager = eg;
  });
}

int bzg_planner_result(bzg_planner* pl, bzg_graph** g_out, bzg_mask** m_out) {
  bzg_graph* g = nullptr;
  bzg_mask* mk = nullptr;
  int rc = guarded([&] {
    BZG_REQUIRE(pl && g_out, BZG_EINVAL, "null argument");
    Planner* p = as_pl(pl);
    Ctx* c = planner_ctx(p);
    set_device(c);
    const Graph* src = planner_graph(p);
    g = new bzg_graph();
    g->ctx = c;
    g->m = src->m;
    g->gamma = src->gamma;
    g->p = src->p;
    g->n = src->n;
    g->V = src->V;
    g->D = src->D;
    g->vertices.alloc((size_t)g->V * g->n * sizeof(double), c->stream);
    BZG_CHECK_CUDA(cudaMemcpyAsync(g->vertices.ptr, src->vertices.ptr, (size_t)g->V * g->n * sizeof(double),
                                   cudaMemcpyDeviceToDevice, c->stream));
    set_edges(c, g, src->E, src->src.as<int>(), src->dst.as<int>(), src->cost.as<double>(), true);
    if (m_out) {
      const Mask* sm = planner_mask(p);
      mk = new bzg_mask();
      mk->g = g;
      mk->ctx = c;
      mk->E = g->E;
      mk->n_obs = sm->n_obs;
      for (int i = 0; i < 6; ++i) mk->counters[i] = sm->counters[i];
      mk->alive.alloc(std::max<long long>(g->E, 1), c->stream);
      mk->prov.alloc(std::max<long long>(g->E, 1), c->stream);
      if (g->E > 0) {
        BZG_CHECK_CUDA(cudaMemcpyAsync(mk->alive.ptr, sm->alive.ptr, g->E, cudaMemcpyDeviceToDevice, c->stream));
        BZG_CHECK_CUDA(cudaMemcpyAsync(mk->prov.ptr, sm->prov.ptr, g->E, cudaMemcpyDeviceToDevice, c->stream));
      }
    }
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
  });
  if (rc == BZG_OK) {
    *g_out = g;
    if (m_out) *m_out = mk;
  } else {
    delete mk;
    delete g;
  }
  return rc;
}

int bzg_planner_info(const bzg_planner* pl, int64_t info[6]) {
  return guarded([&] {
    BZG_REQUIRE(pl && info, BZG_EINVAL, "null argument");
    planner_info(as_pl(pl), info);
  });
}

int bzg_planner_destroy(bzg_planner* pl) {
  return guarded([&] {
    if (!pl) return;
    Planner* p = as_pl(pl);
    set_device(planner_ctx(p));
    planner_destroy(p);
  });
}

}  // extern "C"
