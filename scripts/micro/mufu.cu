// Microbenchmark: throughput of DFMA vs MUFU.RCP64H (+refinement) vs F2F path on one GPU.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp64h(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r;
}
template <int MODE>
__global__ void k(int iters, double a, double* out) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = 1.0 + threadIdx.x * 1e-6 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) x[j] = fma(x[j], a, 1e-9);
      if (MODE == 1) x[j] = rcp64h(x[j]) + 1e-9;          // MUFU + DADD
      if (MODE == 2) { float f = __fdividef(1.0f, (float)x[j]); x[j] = (double)f + 1e-9; }
    }
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1.234) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int blocks = 148 * 8, threads = 256, iters = 2048;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"DFMA", "MUFU.RCP64H+DADD", "F2F+RCP32+F2F+DADD"};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 1) k<1><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 2) k<2><<<blocks, threads>>>(iters, 0.9999, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double ops = 8.0 * iters * blocks * threads;
    printf("%-22s %8.3f ms  %8.1f Gop/s  (%.2f lane-ops/clk/SM at 1.9GHz)\n", names[mode], best,
           ops / best / 1e6, ops / (best * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
