// Does FP64 MMA (mma.sync m8n8k4 f64) run on a pipe separate from DFMA on this GPU?
// Time: (a) DFMA-only loop, (b) DMMA-only loop, (c) both interleaved.  If (c) ~ max(a, b), they
// overlap; if (c) ~ a + b, they share the FP64 pipe.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b, const double (&c)[2]) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d[0]), "=d"(d[1]) : "d"(a), "d"(b), "d"(c[0]), "d"(c[1]));
}

template <int MODE>
__global__ void k(double* out, int n) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  double acc[4][2] = {{1, 2}, {3, 4}, {5, 6}, {7, 8}};
  const double a = 1.0000001, b = 0.9999999;
  for (int it = 0; it < n; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __fma_rn(x[i], a, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double d[2];
        dmma(d, a + r, b, acc[r]);
        acc[r][0] = d[0];
        acc[r][1] = d[1];
      }
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  for (int r = 0; r < 4; ++r) s += acc[r][0] + acc[r][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
float run(double* out, int n) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 4, 256>>>(out, n);
  cudaEventRecord(e0);
  k<MODE><<<148 * 4, 256>>>(out, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out; cudaMalloc(&out, 148 * 4 * 256 * sizeof(double));
  const int n = 4096;
  float a = run<0>(out, n), b = run<1>(out, n), c = run<2>(out, n);
  const double dfma = 148.0 * 4 * 256 * n * 32.0;   // DFMA instructions (per thread)
  const double dmma = 148.0 * 4 * 8 * n * 4.0;      // DMMA ops (per warp)
  printf("DFMA only %.3f ms (%.3e DFMA/s)\nDMMA only %.3f ms (%.3e DMMA/s, %.2f TFLOP/s)\nboth %.3f ms\n", a, dfma / a * 1e3,
         b, dmma / b * 1e3, dmma * 512 / b * 1e-9, c);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
