// Device exclusive prefix sums (tree build / list compaction / work items).
#include "ddm_internal.cuh"

namespace ddm {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

template <class T>
__device__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Exclusive scan of one tile per block; block total to sums[blockIdx.x].
template <class T>
__global__ void scan_tile_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t n,
                                 T* __restrict__ sums) {
  __shared__ T warp_tot[kScanThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T run = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    v[k] = (i < n) ? in[i] : T(0);
    run += v[k];
  }
  T incl = warp_incl_scan(run);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    T t = warp_tot[lane];
    T s = warp_incl_scan(t);
    warp_tot[lane] = s - t;
  }
  __syncthreads();
  T excl = incl - run + warp_tot[w];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < n) out[i] = excl;
    excl += v[k];
  }
  if (threadIdx.x == kScanThreads - 1 && sums) sums[blockIdx.x] = excl;
}

template <class T>
__global__ void add_block_offsets(T* __restrict__ out, int64_t n, const T* __restrict__ offs) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  const T o = offs[blockIdx.x];
  for (int k = threadIdx.x; k < kScanTile; k += blockDim.x) {
    const int64_t i = base + k;
    if (i < n) out[i] += o;
  }
}

template <class T>
__global__ void scan_total_kernel(const T* in, const T* out, int64_t n, T* tot) {
  *tot = out[n - 1] + in[n - 1];
}

template <class T>
int scan_rec(ddm_ctx_s* ctx, const T* in, T* out, int64_t n, cudaStream_t s) {
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb == 1) {
    scan_tile_kernel<T><<<1, kScanThreads, 0, s>>>(in, out, n, (T*)nullptr);
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }
  T* sums = nullptr;
  T* sums_scan = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&sums, nb * sizeof(T), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&sums_scan, nb * sizeof(T), s));
  int rc = DDM_OK;
  scan_tile_kernel<T><<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, n, sums);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) rc = cuda_error(ctx, e, "scan_tile_kernel");
  if (!rc) rc = scan_rec<T>(ctx, sums, sums_scan, nb, s);
  if (!rc) {
    add_block_offsets<T><<<(unsigned)nb, 256, 0, s>>>(out, n, sums_scan);
    e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_error(ctx, e, "add_block_offsets");
  }
  cudaFreeAsync(sums, s);
  cudaFreeAsync(sums_scan, s);
  return rc;
}

template <class T>
int scan_top(ddm_ctx_s* ctx, const T* in, T* out, int64_t n, T* total_host, cudaStream_t s) {
  if (n <= 0) {
    if (total_host) *total_host = 0;
    return DDM_OK;
  }
  int rc = scan_rec<T>(ctx, in, out, n, s);
  if (rc) return rc;
  if (total_host) {
    T* d = reinterpret_cast<T*>(ctx->d_scalar);
    scan_total_kernel<T><<<1, 1, 0, s>>>(in, out, n, d);
    DDM_CUDA(ctx, cudaGetLastError());
    DDM_CUDA(ctx, cudaMemcpyAsync(total_host, d, sizeof(T), cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
  }
  return DDM_OK;
}

}  // namespace

int exclusive_scan_i32(ddm_ctx_s* ctx, const int* in, int* out, int n, int* total_host,
                       cudaStream_t s) {
  return scan_top<int>(ctx, in, out, n, total_host, s);
}

int exclusive_scan_i64(ddm_ctx_s* ctx, const int64_t* in, int64_t* out, int n,
                       int64_t* total_host, cudaStream_t s) {
  return scan_top<long long>(ctx, reinterpret_cast<const long long*>(in),
                             reinterpret_cast<long long*>(out), n,
                             reinterpret_cast<long long*>(total_host), s);
}

}  // namespace ddm
