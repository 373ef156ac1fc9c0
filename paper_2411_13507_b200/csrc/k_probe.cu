// Diagnostic microbenchmarks used for the roofline denominators (not a reference entry
// point): sustained FP64 DFMA / DADD issue rate of the device, measured with CUDA events.
#include <algorithm>

#include "bzg_internal.cuh"

namespace bzg {
namespace {

template <bool kFma>
__global__ void k_probe_fp64(int iters, double seed, double* out) {
  BZG_PDL_ENTRY();
  // 8 independent dependency chains per thread keep the FP64 pipe saturated
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double m = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (kFma) {
        a0 = __fma_rn(a0, m, c); a1 = __fma_rn(a1, m, c); a2 = __fma_rn(a2, m, c); a3 = __fma_rn(a3, m, c);
        a4 = __fma_rn(a4, m, c); a5 = __fma_rn(a5, m, c); a6 = __fma_rn(a6, m, c); a7 = __fma_rn(a7, m, c);
      } else {
        a0 = __dadd_rn(a0, c); a1 = __dadd_rn(a1, c); a2 = __dadd_rn(a2, c); a3 = __dadd_rn(a3, c);
        a4 = __dadd_rn(a4, c); a5 = __dadd_rn(a5, c); a6 = __dadd_rn(a6, c); a7 = __dadd_rn(a7, c);
      }
    }
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

}  // namespace
}  // namespace bzg

extern "C" int bzg_probe_fp64(bzg_ctx* ctx, int use_fma, double* instr_per_s) {
  using namespace bzg;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  try {
    BZG_REQUIRE(c && instr_per_s, BZG_EINVAL, "null argument");
    BZG_CHECK_CUDA(cudaSetDevice(c->device));
    DevBuf out;
    out.alloc(8, c->stream);
    const int blocks = c->num_sms * 8, threads = 256, iters = 2048;
    cudaEvent_t a, b;
    BZG_CHECK_CUDA(cudaEventCreate(&a));
    BZG_CHECK_CUDA(cudaEventCreate(&b));
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
      BZG_CHECK_CUDA(cudaEventRecord(a, c->stream));
      if (use_fma) k_probe_fp64<true><<<blocks, threads, 0, c->stream>>>(iters, 1.0, out.as<double>());
      else k_probe_fp64<false><<<blocks, threads, 0, c->stream>>>(iters, 1.0, out.as<double>());
      BZG_CHECK_CUDA(cudaGetLastError());
      BZG_CHECK_CUDA(cudaEventRecord(b, c->stream));
      BZG_CHECK_CUDA(cudaEventSynchronize(b));
      float ms = 0.f;
      BZG_CHECK_CUDA(cudaEventElapsedTime(&ms, a, b));
      const double instr = (double)blocks * threads * iters * 16 * 8;
      if (rep > 0) best = std::max(best, instr / (ms * 1e-3));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *instr_per_s = best;
    return BZG_OK;
  } catch (const Error& e) {
    return e.code;
  }
}
