// Accuracy of the P2P reciprocal with ONE Newton step on the MUFU seed
// (p2p.cu p2p_rcp, DDM_P2P_RCP2=1) and with the cubic refinement (fast_rcp):
// max relative error against the correctly rounded 1/x over 2^24 values of
// x = |w|^2 spanning 1e-12 .. 1e12 (log-uniform), plus the seed alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rcp_probe scripts/micro/rcp_probe.cu
#include <cstdio>
#include <cmath>
__device__ double seed(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ double rcp1(double x) { const double r = seed(x); return fma(r, fma(-x, r, 1.0), r); }
__device__ double rcp3(double x) { const double r = seed(x); const double e = fma(-x, r, 1.0); return fma(r, fma(e, e, e), r); }
__device__ unsigned long long hash(unsigned long long v) {
  v ^= v >> 33; v *= 0xff51afd7ed558ccdULL; v ^= v >> 33; v *= 0xc4ceb9fe1a85ec53ULL; v ^= v >> 33; return v;
}
__device__ double atomicMaxD(double* a, double v) {
  unsigned long long* p = (unsigned long long*)a; unsigned long long old = *p, as;
  do { as = old; if (__longlong_as_double(as) >= v) break; old = atomicCAS(p, as, __double_as_longlong(v)); } while (old != as);
  return __longlong_as_double(old);
}
__global__ void k(double* err) {
  const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const double u = (hash(i) >> 11) * (1.0 / 9007199254740992.0);
  const double x = pow(10.0, -12.0 + 24.0 * u);
  const double ex = 1.0 / x;
  atomicMaxD(err + 0, fabs(seed(x) - ex) / ex);
  atomicMaxD(err + 1, fabs(rcp1(x) - ex) / ex);
  atomicMaxD(err + 2, fabs(rcp3(x) - ex) / ex);
}
int main() {
  double* d; cudaMalloc(&d, 3 * sizeof(double)); cudaMemset(d, 0, 3 * sizeof(double));
  k<<<1 << 16, 256>>>(d);
  double h[3]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("max rel error: seed %.3e  one Newton %.3e  cubic %.3e  (2^-53 = %.3e)\n", h[0], h[1], h[2], ldexp(1.0, -53));
  return 0;
}
