// Batched Cut-QP (dense ADMM, verdict selection, active-set polish) for one gamma: the
// k_qp_g<gamma>.cu translation units include this with BZG_QP_G defined, so the QP kernels of
// the different gammas compile in parallel.  Shared types: k_cut_types.cuh.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <string>

#include "bzg_internal.cuh"
#include "bzg_math.cuh"
#include "k_cut_types.cuh"
#include "k_qp_common.cuh"
#include "k_admm.cuh"
#include "k_admm2.cuh"
#include "k_polish.cuh"

namespace bzg {
namespace {

// Batched Cut-QP over the work list pend[0 .. n) (graph.py:320-337 / cut_qp 285-299), n =
// min(*job.d_n, job.n_inst) read on the device (job.n_inst = the buffers' capacity): ADMM,
// verdict selection, polish.  Fills job.st_out / it_out / delta_out, mk->n_polished and d_safe
// (n verdicts).  polish_mode: 0 none, 1 SOLVED, 2 SOLVED and MAX_ITER.  No host round trip.
template <int G, int M, int C>
void qp_solve_t(Ctx* c, const QpJob& job) {
  const Graph* g = job.g;
  DParams dp{};
  for (int k = 0; k < 64; ++k) dp.D[k] = job.D[k];
  const ObsRec<M, obs_cap<C>()>* d_obs = static_cast<const ObsRec<M, obs_cap<C>()>*>(job.d_obs);
  const bool canon = job.canon;
  const unsigned long long* d_pend = job.d_pend;
  const long long n_inst = job.n_inst;
  const bzg_cut_config* cfg = job.cfg;
  const int polish_mode = job.polish_mode;
  const double screen = job.screen;
  Mask* mk = job.mk;
  DevBuf& d_safe = *job.d_safe;
  auto trace = [&](const char* what) { c->trace(what); };
  constexpr int NV = 2 * G + C, MCc = C + 2 * G + 1;
  const unsigned long long* d_n = job.d_n;
  int8_t* st_out = job.st_out;
  int* it_out = job.it_out;
  double* delta_out = job.delta_out;
  DevBuf &d_x = c->ws[WS_QX], &d_zy = c->ws[WS_QZY], &d_list = c->ws[WS_QLIST], &d_next = c->ws[WS_QNEXT];
  d_x.alloc(n_inst * NV * sizeof(double), c->stream);
  d_safe.alloc(n_inst, c->stream);
  d_next.alloc(sizeof(unsigned long long), c->stream);
  d_zy.alloc(n_inst * 2 * MCc * sizeof(double), c->stream);
  d_list.alloc(n_inst * sizeof(int), c->stream);
  BZG_CHECK_CUDA(cudaMemsetAsync(d_next.ptr, 0, sizeof(unsigned long long), c->stream));
  QpParams qp{};
  qp.rho = cfg->qp_rho;
  qp.rho_eq = cfg->qp_rho * 1e3;  // equality rows (qpsolver.py:100-103, 137)
  qp.sigma = cfg->qp_sigma;
  qp.alpha = cfg->qp_alpha;
  qp.one_m_alpha = 1.0 - cfg->qp_alpha;
  qp.eps_abs = cfg->qp_eps_abs;
  qp.eps_rel = cfg->qp_eps_rel;
  qp.eps_pinf = cfg->qp_eps_pinf;
  qp.max_iter = cfg->qp_max_iter;
  static const int batch_env = std::getenv("BZG_ADMM_BATCH") ? std::atoi(std::getenv("BZG_ADMM_BATCH")) : 0;
  qp.batch = batch_env > 0 ? batch_env : kAdmmBatch;
  // persistent grid: enough resident warps to cover the SMs several times
  const long long blocks = std::min<long long>(div_up(n_inst, 128), (long long)c->num_sms * 16);
  const bool rel = cfg->qp_eps_rel != 0.0, unit = cfg->qp_rho == 1.0;
  auto admm = rel ? (unit ? k_qp_admm<G, M, C, true, true, false> : k_qp_admm<G, M, C, true, false, false>)
                  : (unit ? k_qp_admm<G, M, C, false, true, false> : k_qp_admm<G, M, C, false, false, false>);
  auto setup = k_qp_setup<G, M, C, false>;
  size_t nconst = QpConsts<G, M, C, false>::N;
  if constexpr (C == 2 * M)
    if (canon && unit && !rel) {
      admm = k_qp_admm<G, M, C, false, true, true>;
      setup = k_qp_setup<G, M, C, true>;
      nconst = QpConsts<G, M, C, true>::N;
    }
  DevBuf& d_consts = c->ws[WS_QCONST];
  d_consts.alloc(n_inst * nconst * sizeof(double), c->stream);
  trace("qp alloc");
  launch(c, "k_qp_setup", setup, dim3((unsigned)std::min<long long>(div_up(n_inst, 128), c->num_sms * 8ll)),
         dim3(128), 0, qp, dp, g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(), d_obs, d_pend, n_inst, d_n,
         d_consts.as<double>());
  // Lanes per instance: two for very short work lists (kAdmm2MaxInst), else one.
  const int lanes_env = std::getenv("BZG_ADMM_LANES") ? std::atoi(std::getenv("BZG_ADMM_LANES")) : 0;  // per call
  const bool two_ok = unit && !rel && C <= kObsRows;
  // the list length is known on the host when d_n is null, else the capacity bounds it
  const bool two = two_ok && (lanes_env == 2 || (lanes_env == 0 && n_inst <= kAdmm2MaxInst));
  if (two) {
    if constexpr (C <= kObsRows) {
      auto admm2 = k_qp_admm2<G, M, C, false>;
      if constexpr (C == 2 * M)
        if (canon) admm2 = k_qp_admm2<G, M, C, true>;
      const long long blocks2 = std::min<long long>(div_up(2 * n_inst, 128), (long long)c->num_sms * 16);
      launch(c, "k_qp_admm", admm2, dim3((unsigned)blocks2), dim3(128), 0, qp, d_consts.as<double>(), n_inst,
             d_next.as<unsigned long long>(), st_out, it_out, d_x.as<double>(), d_zy.as<double>(), d_n);
    }
  } else {
    // main pass over the work list, then resume passes over the parked tails (AdmmPass):
    // BZG_ADMM_PASSES launches, the last one without parking; BZG_ADMM_DUMP is the live-lane
    // count below which a drained warp parks its instances (default 12).  Default: one pass --
    // the parked tails are latency-bound chains that a dense relaunch does not run faster
    // (cfg2: 0.57 ms in one pass, 0.73-0.96 ms with 2-6 passes).
    const int passes = std::max(1, std::getenv("BZG_ADMM_PASSES") ? std::atoi(std::getenv("BZG_ADMM_PASSES")) : 1);
    const int dump = std::getenv("BZG_ADMM_DUMP") ? std::atoi(std::getenv("BZG_ADMM_DUMP")) : 12;
    // BZG_ADMM_BUDGET=C: the first pass parks every instance still running after C iterations
    // (the long ones then run together in the next pass)
    const int budget = std::getenv("BZG_ADMM_BUDGET") ? std::atoi(std::getenv("BZG_ADMM_BUDGET")) : 0;
    DevBuf& d_rq = c->ws[WS_QRESUME];
    d_rq.alloc((passes > 1 ? 2 * n_inst : 1) * sizeof(int) + 4 * sizeof(unsigned long long), c->stream);
    unsigned long long* qn = reinterpret_cast<unsigned long long*>(d_rq.as<char>() + (passes > 1 ? 2 * n_inst : 1) * sizeof(int));
    int* q0 = d_rq.as<int>();
    int* q1 = q0 + n_inst;
    if (passes > 1) BZG_CHECK_CUDA(cudaMemsetAsync(qn, 0, 4 * sizeof(unsigned long long), c->stream));
    for (int ps = 0; ps < passes; ++ps) {
      AdmmPass pass{};
      if (ps > 0) {
        pass.rq_in = (ps & 1) ? q0 : q1;
        pass.rq_in_n = qn + ((ps & 1) ? 0 : 1);
        BZG_CHECK_CUDA(cudaMemsetAsync(d_next.ptr, 0, sizeof(unsigned long long), c->stream));
      }
      if (ps + 1 < passes) {
        pass.rq_out = (ps & 1) ? q1 : q0;
        pass.rq_out_n = qn + ((ps & 1) ? 1 : 0);
        if (ps > 0) BZG_CHECK_CUDA(cudaMemsetAsync(pass.rq_out_n, 0, sizeof(unsigned long long), c->stream));
        pass.dump_below = budget > 0 ? 0 : dump;
        if (ps == 0) pass.park_after = budget;
      }
      launch(c, ps == 0 ? "k_qp_admm" : "k_qp_admm_tail", admm, dim3((unsigned)blocks), dim3(128), 0, qp,
             d_consts.as<double>(), n_inst, d_next.as<unsigned long long>(), st_out, it_out, d_x.as<double>(),
             d_zy.as<double>(), pass, d_n);
      if (c->trace_on && pass.rq_out_n && !g_capturing) {
        unsigned long long hq = 0;
        BZG_CHECK_CUDA(cudaMemcpyAsync(&hq, pass.rq_out_n, sizeof(hq), cudaMemcpyDeviceToHost, c->stream));
        BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
        std::fprintf(stderr, "[bzg qp] pass %d parked %llu of %lld instances\n", ps, hq, n_inst);
      }
    }
  }
  trace("admm");
  BZG_CHECK_CUDA(cudaMemsetAsync(d_next.ptr, 0, sizeof(unsigned long long), c->stream));
  launch(c, "k_qp_select", k_qp_select<G, M, C>,
         dim3((unsigned)std::min<long long>(div_up(n_inst, 256), c->num_sms * 8ll)), dim3(256), 0, n_inst, d_n,
         polish_mode, screen, cfg->eps_cut, (const int8_t*)st_out, d_x.as<double>(), delta_out, d_safe.as<uint8_t>(),
         d_list.as<int>(), d_next.as<unsigned long long>());
  static const bool polish_lu = std::getenv("BZG_POLISH_IMPL") && std::string(std::getenv("BZG_POLISH_IMPL")) == "lu";
  long long n_list = -1;  // known on the host only when it is read back (LU path, tracing)
  if ((polish_lu || c->trace_on) && !g_capturing) {
    unsigned long long* hn = static_cast<unsigned long long*>(c->host_scratch(8 * sizeof(unsigned long long))) + 7;
    BZG_CHECK_CUDA(cudaMemcpyAsync(hn, d_next.ptr, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    BZG_CHECK_CUDA(cudaStreamSynchronize(c->stream));
    n_list = (long long)*hn;
    if (c->trace_on) std::fprintf(stderr, "[bzg cut] qp instances %lld, polished %lld\n", n_inst, n_list);
  }
  mk->n_polished = n_list;
  if (polish_lu && C <= kObsRows) {  // the shared-memory core LU (kept for A/B checks)
    if constexpr (C <= kObsRows) {
      constexpr int NR = polish_dim<G, M, C>();
      const size_t psmem = (size_t)(NR * NR + NR) * kPolishThreads * sizeof(double);
      ensure_dyn_smem((const void*)k_qp_polish<G, M, C>, psmem);
      launch(c, "k_qp_polish", k_qp_polish<G, M, C>, dim3(div_up(n_list, kPolishThreads)), dim3(kPolishThreads),
             psmem, dp, g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(), d_obs, d_pend, d_list.as<int>(),
             n_list, cfg->eps_cut, d_x.as<double>(), d_zy.as<double>(), delta_out, d_safe.as<uint8_t>(), st_out);
    }
  } else {
    // persistent grid over the device-side list length (at most n_inst entries)
    const long long pblocks = std::min<long long>(div_up(n_inst, 128), (long long)c->num_sms * 8);
    launch(c, "k_qp_polish", k_qp_polish_reg<G, M, C>, dim3((unsigned)pblocks), dim3(128), 0, dp,
           g->vertices.as<double>(), g->src.as<int>(), g->dst.as<int>(), d_obs, d_pend, d_list.as<int>(),
           d_next.as<unsigned long long>(), cfg->eps_cut, d_x.as<double>(), d_zy.as<double>(), delta_out,
           d_safe.as<uint8_t>(), st_out);
  }
  trace("select+polish");
}


}  // namespace

#define BZG_QP_ENTRY_(g) qp_solve_g##g
#define BZG_QP_ENTRY(g) BZG_QP_ENTRY_(g)
void BZG_QP_ENTRY(BZG_QP_G)(Ctx* c, int M, int C, const QpJob& job) {
  constexpr int G = BZG_QP_G;
  if (M == 1 && C == 2) return qp_solve_t<G, 1, 2>(c, job);
  if (M == 1 && C == kObsRows) return qp_solve_t<G, 1, kObsRows>(c, job);
  if (M == 2 && C == 4) return qp_solve_t<G, 2, 4>(c, job);
  if (M == 2 && C == kObsRows) return qp_solve_t<G, 2, kObsRows>(c, job);
  if (M == 3 && C == 6) return qp_solve_t<G, 3, 6>(c, job);
  if (M == 3 && C == kObsRows) return qp_solve_t<G, 3, kObsRows>(c, job);
  if (M == 1 && C == kObsRowsBig) return qp_solve_t<G, 1, kObsRowsBig>(c, job);
  if (M == 2 && C == kObsRowsBig) return qp_solve_t<G, 2, kObsRowsBig>(c, job);
  if (M == 3 && C == kObsRowsBig) return qp_solve_t<G, 3, kObsRowsBig>(c, job);
  throw Error(BZG_EUNSUPPORTED, "Cut-QP: unsupported (m, obstacle rows)");
}

}  // namespace bzg
