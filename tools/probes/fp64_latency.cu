// Dependent-chain latency of FP64 ops on the current GPU (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = __fma_rn(x, b, a);
      if (OP == 1) x = __dadd_rn(x, b);
      if (OP == 2) x = __dmul_rn(x, b);
      if (OP == 3) x = (x < b) ? x : b * 0.5;   // DSETP + select chain
      if (OP == 4) x = fabs(x) <= b ? x + 1.0 : x - 1.0;
      if (OP == 5) x = __shfl_xor_sync(0xffffffffu, x, 1);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
void run(const char* name) {
  double* d; long long* c; cudaMalloc(&d, 1024 * 8); cudaMalloc(&c, 8);
  const int n = 4096;
  chain<OP><<<1, 32>>>(d, c, 1.0000001, 0.9999999, n);
  chain<OP><<<1, 32>>>(d, c, 1.0000001, 0.9999999, n);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.2f cycles/op\n", name, (double)h / (n * 16.0));
}

int main() {
  run<0>("DFMA dependent");
  run<1>("DADD dependent");
  run<2>("DMUL dependent");
  run<3>("DSETP+select dependent");
  run<4>("fabs/cmp/DADD dependent");
  run<5>("SHFL.xor (double) dependent");
  return 0;
}
