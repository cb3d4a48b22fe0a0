// Microbenchmark: fp64 tensor (mma.sync m8n8k4 f64 -> DMMA.8x8x4) vs DFMA vs
// SHFL throughput on one GPU (the M2L/M2M contraction choice).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma scripts/micro/dmma.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void k(int iters, double a, double* out) {
  double x[8], y[8];
  for (int j = 0; j < 8; ++j) { x[j] = 1.0 + threadIdx.x * 1e-6 + j; y[j] = 0.5 * j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) x[j] = fma(x[j], a, 1e-9);
      if (MODE == 1) dmma(x[j], y[j], a, 1e-3);
      if (MODE == 2) x[j] += __shfl_xor_sync(0xffffffffu, x[j], 1 + (j & 15));
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j] + y[j];
  if (s == 1.234) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int blocks = 148 * 8, threads = 256, iters = 1024;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"DFMA (2 flop/lane)", "DMMA.8x8x4 (512 flop/warp)",
                          "SHFL.BFLY f64 (2 SHFL + DADD)"};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 1) k<1><<<blocks, threads>>>(iters, 0.9999, d);
      if (mode == 2) k<2><<<blocks, threads>>>(iters, 0.9999, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double warp_ops = 8.0 * iters * blocks * (threads / 32);
    const double flop = mode == 0 ? warp_ops * 64 : mode == 1 ? warp_ops * 512 : 0;
    printf("%-32s %8.3f ms  %8.2f warp-instr/clk/SM  %8.2f TFLOP/s\n", names[mode], best,
           warp_ops / (best * 1e-3) / 148 / 1.965e9, flop / (best * 1e-3) / 1e12);
  }
  return 0;
}
