// Microbenchmark: cost of the near-field reciprocal seed inside a DFMA stream.
// Each iteration per thread: 8 independent chains x 3 DFMA (24 DFMA), plus
// MODE 1: one MUFU.RCP64H (rcp.approx.ftz.f64) seed,
// MODE 2: one fp32 seed (F2F.F32.F64, MUFU.RCP, F2F.F64.F32),
// MODE 3: two MUFU.RCP64H (each seed result summed into one DADD chain).
// The extra time over MODE 0, in DFMA-slot equivalents, is what the seed
// costs the fp64 pipe of the P2P pair update.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float rcp32(float x) {
  float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r;
}
__device__ __forceinline__ double rcp64h(double x) {
  double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r;
}
template <int MODE>
__global__ void __launch_bounds__(256) k(int iters, double a, double* out) {
  double x[8], y = 1.5 + threadIdx.x * 1e-7;
  for (int j = 0; j < 8; ++j) x[j] = 1.0 + threadIdx.x * 1e-6 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, 1e-9);
    if (MODE == 1) y += rcp64h(x[0]);
    if (MODE == 2) y += (double)rcp32((float)x[0]);
    if (MODE == 3) { y += rcp64h(x[0]); y += rcp64h(x[3]); }
  }
  double s = y; for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1.234) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[4] = {"24 DFMA", "24 DFMA + RCP64H", "24 DFMA + fp32 seed", "24 DFMA + 2 RCP64H"};
  float t[4];
  for (int mode = 0; mode < 4; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 1) k<1><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 2) k<2><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 3) k<3><<<blocks, threads>>>(iters, 0.9999, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    t[mode] = best;
    printf("%-22s %8.3f ms  extra = %5.2f DFMA-slot equivalents per iteration\n", names[mode], best,
           24.0 * (best - t[0]) / t[0]);
  }
  return 0;
}
