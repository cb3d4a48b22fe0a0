// Host cost of device allocations (cudaMalloc vs pool cudaMallocAsync) by size
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
int main() {
  cudaFree(0);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t keep = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  const size_t MB = 1 << 20;
  size_t sizes[] = {24 * MB, 384 * MB, 384 * MB, 384 * MB, 768 * MB, 1536 * MB, 3072 * MB, 384 * MB};
  for (int mode = 0; mode < 2; ++mode)
    for (size_t sz : sizes) {
      void* p = nullptr;
      auto t0 = std::chrono::steady_clock::now();
      if (mode == 0) cudaMalloc(&p, sz); else cudaMallocAsync(&p, sz, s);
      cudaStreamSynchronize(s);
      auto t1 = std::chrono::steady_clock::now();
      cudaMemsetAsync(p, 0, sz, s);
      cudaStreamSynchronize(s);
      auto t2 = std::chrono::steady_clock::now();
      size_t fr, tot;
      cudaMemGetInfo(&fr, &tot);
      auto t3 = std::chrono::steady_clock::now();
      printf("%s %6zu MB alloc %8.3f ms  first memset %8.3f ms  memgetinfo %.3f ms\n",
             mode ? "async " : "malloc", sz / MB,
             std::chrono::duration<double, std::milli>(t1 - t0).count(),
             std::chrono::duration<double, std::milli>(t2 - t1).count(),
             std::chrono::duration<double, std::milli>(t3 - t2).count());
    }
  return 0;
}
