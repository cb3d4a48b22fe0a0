// GMRES with the FMM operator (DESIGN.md §4.1 row a12, §4.7; "a modified
// version of GMRES with FMM for matrix-vector multiplication"; reading R11):
// restarted GMRES, Arnoldi by classical Gram-Schmidt with selective
// reorthogonalisation (a second CGS pass when the first cancelled more than
// half of ||w||^2: Daniel-Gragg-Kaufman-Stewart criterion),
// Givens rotations, relative residual ||b - A x|| / ||b|| <= tol.
//
// Vectors live in Morton-sorted order; each rank keeps its owned rows
// [own_el_lo, own_el_hi) of every Krylov vector.  Per iteration: one all-gather
// of the new basis vector (multi-GPU only), the matvec, one batched dot pass
// (one all-reduce of k+1 partial dots) and two norms, plus a second dot pass
// when reorthogonalisation is needed.  The small Hessenberg
// least-squares problem is solved on the host.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kcommon.cuh"

namespace {
// Programmatic dependent launch inside the captured Arnoldi step (DESIGN.md
// §4.7h): the CGS and finish kernels are launched with programmatic stream
// serialisation, trigger their dependents at entry and wait for their
// predecessor before touching anything (no-ops without the attribute).
__device__ __forceinline__ void step_pdl() {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// launch with programmatic stream serialisation (DDM_GMRES_PDL=0: plain)
template <typename... KArgs, typename... Args>
cudaError_t launch_step(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t shm,
                        cudaStream_t s, Args... args) {
  static const bool on = [] {
    const char* e = getenv("DDM_GMRES_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = shm;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
}  // namespace

namespace ddm {
namespace {

constexpr int kDotThreads = 256;

// part[i * nb + b] = sum over chunk b of V[i * ld + j] * w[j]; the last
// block of vector i to finish (atomic ticket) sums the nb partials in a fixed
// order into out[i] (deterministic, no second launch) and resets the ticket.
__device__ __forceinline__ double fixed_order_sum(const double* part, int nb) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[b];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// kd != nullptr (captured Arnoldi step): the step index k
// is read from device memory, nvec = k + 1 and out += (pass ? k + 1 : 0);
// vectors i = blockIdx.y, blockIdx.y + gridDim.y, ...
__global__ void __launch_bounds__(kDotThreads)
multi_dot(const double* __restrict__ V, int64_t ld, const double* __restrict__ w, int64_t len,
          int nb, double* __restrict__ part, unsigned* __restrict__ ticket,
          double* __restrict__ out, const int* __restrict__ kd, int pass, int dgks = 0) {
  const int b = blockIdx.x;
  int nvec = gridDim.y;
  if (kd) {
    const int k = *kd;
    nvec = k + 1;
    if (dgks && pass == 1 && out[2 * (k + 1) + 2] == 0.0) {   // DGKS: no second pass
      if (b == 0 && threadIdx.x == 0)
        for (int i = blockIdx.y; i < nvec; i += gridDim.y) out[k + 1 + i] = 0.0;
      return;
    }
    out += pass ? k + 1 : 0;
  }
  const int64_t chunk = (len + nb - 1) / nb;
  const int64_t j0 = b * chunk, j1 = min(len, j0 + chunk);
  __shared__ double sh[kDotThreads / 32];
  __shared__ bool last;
  for (int i = blockIdx.y; i < nvec; i += gridDim.y) {
    const double* v = V + (int64_t)i * ld;
    double acc = 0.0;
    for (int64_t j = j0 + threadIdx.x; j < j1; j += kDotThreads) acc = fma(v[j], w[j], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int k = 0; k < kDotThreads / 32; ++k) s += sh[k];
      part[(int64_t)i * nb + b] = s;
      __threadfence();
      last = atomicAdd(ticket + i, 1u) == (unsigned)(nb - 1);
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {
      __threadfence();
      const double s = fixed_order_sum(part + (int64_t)i * nb, nb);
      if (threadIdx.x == 0) {
        out[i] = s;
        ticket[i] = 0u;
      }
    }
    __syncthreads();
  }
}

// w[j] += sign * sum_i V[i * ld + j] c[i] (and optionally ||w||^2 of the
// result).  Block = 64 rows x 4 vector groups: thread (j, q) sums the vectors
// i = q, q + 4, ... with four accumulators (loads of four vectors in flight),
// the four group partials are added in a fixed order, so every row's sum has
// the same order whatever the row range (deterministic, rank independent).
// With kd (captured step): nvec = *kd + 1, c += pass ? k + 1 : 0, and the
// norm goes to out[2 (k+1) + 1].
// DDM_V_KEEP=1: the CGS passes read the Krylov basis with an L2 evict_last
// cache policy (createpolicy + ld.L2::cache_hint), so the basis stays in L2
// across the operator apply, whose streamed data (the poroelastic near-field
// cache, the preconditioner blocks) is read evict-first
#ifndef DDM_V_KEEP
#define DDM_V_KEEP 1
#endif
__device__ __forceinline__ uint64_t v_policy() {
  uint64_t pol = 0;
#if DDM_V_KEEP
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ double v_ld(const double* a, uint64_t pol) {
#if DDM_V_KEEP
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldg(a);
#endif
}

constexpr int kAxRows = 64, kAxGroups = 4;
#ifndef DDM_AX_UNROLL
#define DDM_AX_UNROLL 4
#endif
constexpr int kAxU = DDM_AX_UNROLL;   // loads in flight per thread (multiple of 4)

// DGKS (captured step, kd != nullptr, dgks > 0): pass 0 also sums ||w||^2
// before the update into out[2 (k+1)] and sets out[2 (k+1) + 2] = 1 when the
// update cancelled more than a fraction dgks of ||w||^2 (a second CGS pass is
// needed); pass 1 returns at once when out[2 (k+1) + 2] == 0.
template <bool NORM>
__global__ void __launch_bounds__(kAxRows * kAxGroups)
cgs_axpy(const double* __restrict__ V, int64_t ld, int nvec, const double* __restrict__ c,
         double sign, double* __restrict__ w, int64_t len, double* __restrict__ part,
         unsigned* __restrict__ ticket, double* __restrict__ out, const int* __restrict__ kd,
         int pass, double dgks = 0.0) {
  step_pdl();
  extern __shared__ double sc[];
  __shared__ double red[kAxGroups][kAxRows];
  __shared__ double wsum[kAxRows / 32 > 0 ? kAxRows / 32 : 1];
  __shared__ double wsum0[kAxRows / 32 > 0 ? kAxRows / 32 : 1];
  __shared__ bool last;
  double* dflag = nullptr;
  if (kd) {
    const int k = *kd;
    nvec = k + 1;
    c += pass ? k + 1 : 0;
    if (NORM) {
      dflag = out + 2 * (k + 1) + 2;
      out += 2 * (k + 1) + 1;
      if (dgks > 0.0 && pass == 1 && *dflag == 0.0) return;   // no second pass needed
    }
  }
  const bool track0 = NORM && dgks > 0.0 && pass == 0 && kd;
  const uint64_t pol = v_policy();
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) sc[i] = c[i];
  __syncthreads();
  const int r = threadIdx.x % kAxRows, q = threadIdx.x / kAxRows;
  const int64_t j = blockIdx.x * (int64_t)kAxRows + r;
  double acc = 0.0;
  if (j < len) {
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    const double* v = V + j;
    int i = q;
    for (; i + (kAxU - 1) * kAxGroups < nvec; i += kAxU * kAxGroups) {
      double t[kAxU];
#pragma unroll
      for (int u = 0; u < kAxU; ++u) t[u] = v_ld(v + (int64_t)(i + u * kAxGroups) * ld, pol);
#pragma unroll
      for (int u = 0; u < kAxU; ++u) a[u & 3] = fma(t[u], sc[i + u * kAxGroups], a[u & 3]);
    }
    for (int u = 0; i < nvec; i += kAxGroups, ++u) a[u & 3] = fma(v_ld(v + (int64_t)i * ld, pol), sc[i], a[u & 3]);
    acc = (a[0] + a[1]) + (a[2] + a[3]);
  }
  red[q][r] = acc;
  __syncthreads();
  double nrm = 0.0, nrm0 = 0.0;
  if (q == 0 && j < len) {
    const double tot = ((red[0][r] + red[1][r]) + (red[2][r] + red[3][r]));
    const double w0 = w[j];
    const double wn = fma(sign, tot, w0);
    w[j] = wn;
    nrm = wn * wn;
    nrm0 = w0 * w0;
  }
  if (!NORM) return;
  if (q == 0) {   // warps 0, 1: the block's rows
    for (int o = 16; o; o >>= 1) {
      nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      nrm0 += __shfl_xor_sync(0xffffffffu, nrm0, o);
    }
    if ((threadIdx.x & 31) == 0) {
      wsum[threadIdx.x >> 5] = nrm;
      wsum0[threadIdx.x >> 5] = nrm0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, t0 = 0.0;
    for (int k2 = 0; k2 < kAxRows / 32; ++k2) {
      t += wsum[k2];
      t0 += wsum0[k2];
    }
    part[blockIdx.x] = t;
    if (track0) part[gridDim.x + blockIdx.x] = t0;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    const double t = fixed_order_sum(part, gridDim.x);
    const double t0 = track0 ? fixed_order_sum(part + gridDim.x, gridDim.x) : 0.0;
    if (threadIdx.x == 0) {
      out[0] = t;
      if (track0) {
        out[-1] = t0;
        *dflag = (t < dgks * t0) ? 1.0 : 0.0;
      }
      ticket[0] = 0u;
    }
  }
}

// Row-blocked CGS passes of the captured Arnoldi step:
// a CTA of 512 threads owns 512 consecutive rows (thread = row) and ALL k+1
// basis vectors, so w is read once per pass and -- in the fused kernel -- the
// first pass's update w -= V c and the second pass's dots V^T w share one
// sweep over the CTA's rows of V (the dots re-read the rows from L2).
// Dots: groups of 8 vectors with 32 loads in flight per thread, a warp
// reduce-scatter (9 shuffles for 8 sums), the 32 warps' sums added in warp
// order into one partial per (vector, CTA); the last CTA (ticket) sums each
// vector's <= 128 partials in CTA order.  Deterministic.
#ifndef DDM_ROW_T
#define DDM_ROW_T 512
#endif
#ifndef DDM_ROW_UPD
#define DDM_ROW_UPD 16   // 0: the update loop of cgs_rows<1> as 2 chains x unroll 8; U > 0: U loads at once
#endif
constexpr int kRowT = DDM_ROW_T, kRowsCta = kRowT, kRowMaxCta = kRowT >= 512 ? 128 : 256,
              kRowChunk = 256;

// 8 per-lane values -> lane l holds the warp sum of value
// v = 4 ((l >> 4) & 1) + 2 ((l >> 3) & 1) + ((l >> 2) & 1)
__device__ __forceinline__ double warp_rs8(const double (&a)[8], int lane) {
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double b[4], c[2];
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const double send = h16 ? a[v] : a[v + 4];
    b[v] = (h16 ? a[v + 4] : a[v]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const double send = h8 ? b[v] : b[v + 2];
    c[v] = (h8 ? b[v + 2] : b[v]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const double send = h4 ? c[0] : c[1];
  double d = (h4 ? c[1] : c[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
  d += __shfl_xor_sync(0xffffffffu, d, 2);
  d += __shfl_xor_sync(0xffffffffu, d, 1);
  return d;
}

// MODE 0: out = V^T w (pass 0 dots -> dh[0 .. k]).
// MODE 1: w -= V c with c = dh[0 .. k], then out = V^T w -> dh[k+1 .. 2k+1].
// (The second update + norm stays on cgs_axpy: a row-blocked version measured
// slower, config 3 39.2 -> 41.0 ms.)
template <int MODE, int RT = kRowT>
__global__ void __launch_bounds__(RT)
cgs_rows(const double* __restrict__ V, int64_t ld, int64_t len, double* __restrict__ w,
         const int* __restrict__ kd, double* __restrict__ dh, double* __restrict__ part,
         unsigned* __restrict__ ticket) {
  step_pdl();
  __shared__ double red[RT / 32][kRowChunk];   // per-warp sums of a chunk of vectors
  __shared__ bool last;
  const int k = *kd, nvec = k + 1, nb = gridDim.x;
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
  const uint64_t pol = v_policy();
  const int64_t j = (int64_t)blockIdx.x * RT + t;
  const bool ok = j < len;
  const double* Vj = V + (ok ? j : 0);
  double wr;
  if constexpr (MODE > 0) {
    const double* sc = dh;   // pass-0 coefficients (broadcast loads)
    double a0 = 0.0, a1 = 0.0;
    int i = 0;
#if DDM_ROW_UPD > 0
    {
      double a2 = 0.0, a3 = 0.0;
      for (; i + DDM_ROW_UPD <= nvec; i += DDM_ROW_UPD) {
        double tv[DDM_ROW_UPD];
        const double* vp = Vj + (int64_t)i * ld;
#pragma unroll
        for (int u = 0; u < DDM_ROW_UPD; ++u) {
          tv[u] = v_ld(vp, pol);
          vp += ld;
        }
#pragma unroll
        for (int u = 0; u < DDM_ROW_UPD; u += 4) {
          a0 = fma(tv[u], __ldg(sc + i + u), a0);
          a1 = fma(tv[u + 1], __ldg(sc + i + u + 1), a1);
          a2 = fma(tv[u + 2], __ldg(sc + i + u + 2), a2);
          a3 = fma(tv[u + 3], __ldg(sc + i + u + 3), a3);
        }
      }
      a0 += a2;
      a1 += a3;
    }
#endif
#pragma unroll 8
    for (; i + 1 < nvec; i += 2) {
      a0 = fma(v_ld(Vj + (int64_t)i * ld, pol), __ldg(sc + i), a0);
      a1 = fma(v_ld(Vj + (int64_t)(i + 1) * ld, pol), __ldg(sc + i + 1), a1);
    }
    if (i < nvec) a0 = fma(v_ld(Vj + (int64_t)i * ld, pol), __ldg(sc + i), a0);
    wr = 0.0;
    if (ok) {
      wr = w[j] - (a0 + a1);
      w[j] = wr;
    }
  } else {
    wr = ok ? w[j] : 0.0;
  }
  if (!ok) wr = 0.0;
  double* out = dh + (MODE == 1 ? nvec : 0);
  const int vsel = 4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1);
  for (int c0 = 0; c0 < nvec; c0 += kRowChunk) {   // chunks of vectors (one for k < 256)
    const int c1 = min(nvec, c0 + kRowChunk);
    // groups of 8 vectors, four groups' loads in flight at once
    for (int g0 = c0; g0 < c1; g0 += 32) {
      double a[4][8];
      if (g0 + 32 <= c1) {   // full group: a running pointer, no bounds checks
        const double* vp = Vj + (int64_t)g0 * ld;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            a[q][v] = v_ld(vp, pol);
            vp += ld;
          }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int i = g0 + 8 * q + v;
            a[q][v] = i < c1 ? v_ld(Vj + (int64_t)i * ld, pol) : 0.0;
          }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int v = 0; v < 8; ++v) a[q][v] *= wr;
        const double d = warp_rs8(a[q], lane);
        const int i = g0 + 8 * q + vsel;
        if ((lane & 3) == 0 && i < c1) red[wp][i - c0] = d;
      }
    }
    __syncthreads();
    for (int i = c0 + t; i < c1; i += RT) {
      double sum = 0.0;
#pragma unroll
      for (int q = 0; q < RT / 32; ++q) sum += red[q][i - c0];
      part[(int64_t)i * nb + blockIdx.x] = sum;
    }
    __syncthreads();
  }
  if (t == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == (unsigned)(nb - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    // warp wp: vectors wp + NW r; lane: CTAs lane + 32 q (4 vectors' loads
    // in flight at once)
    constexpr int NW = RT / 32, Q = (RT >= 512 ? 128 : 256) / 32;
    for (int r0 = 0; wp + NW * r0 < nvec; r0 += 4) {
      double v[4][Q];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int i = wp + NW * (r0 + r), b = lane + 32 * q;
          v[r][q] = (i < nvec && b < nb) ? __ldcg(part + (int64_t)i * nb + b) : 0.0;
        }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double sum = v[r][0];
#pragma unroll
        for (int q = 1; q < Q; ++q) sum += v[r][q];
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const int i = wp + NW * (r0 + r);
        if (lane == 0 && i < nvec) out[i] = sum;
      }
    }
    if (t == 0) *ticket = 0u;
  }
}

__global__ void sub_scale(const double* __restrict__ b, const double* __restrict__ w,
                          double* __restrict__ r, int64_t len) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < len) r[j] = b[j] - w[j];
}

__global__ void scale_copy(const double* __restrict__ src, double a, double* __restrict__ dst,
                           int64_t len) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < len) dst[j] = a * src[j];
}

__global__ void gather_sorted(int64_t n, int ncomp, const int* __restrict__ perm,
                              const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm[i];
  for (int c = 0; c < ncomp; ++c) out[i * ncomp + c] = in[(int64_t)j * ncomp + c];
}

__global__ void scatter_to_user(int64_t n, int ncomp, const int* __restrict__ perm,
                                const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm[i];
  for (int c = 0; c < ncomp; ++c) out[(int64_t)j * ncomp + c] = in[i * ncomp + c];
}

// in place: blk[e] <- inverse(blk[e]) (ncomp x ncomp, row major); a singular
// block (|det| <= 1e-300 scale) becomes the identity
__global__ void invert_blocks(int64_t n, int ncomp, double* __restrict__ blk) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n) return;
  double* A = blk + e * ncomp * ncomp;
  if (ncomp == 2) {
    const double a = A[0], b = A[1], c = A[2], d = A[3];
    const double det = a * d - b * c;
    if (!(fabs(det) > 0.0) || !isfinite(det)) {
      A[0] = 1.0; A[1] = 0.0; A[2] = 0.0; A[3] = 1.0;
      return;
    }
    A[0] = d / det; A[1] = -b / det; A[2] = -c / det; A[3] = a / det;
    return;
  }
  double m[9], r[9];
  for (int k = 0; k < 9; ++k) m[k] = A[k];
  r[0] = m[4] * m[8] - m[5] * m[7];
  r[1] = m[2] * m[7] - m[1] * m[8];
  r[2] = m[1] * m[5] - m[2] * m[4];
  r[3] = m[5] * m[6] - m[3] * m[8];
  r[4] = m[0] * m[8] - m[2] * m[6];
  r[5] = m[2] * m[3] - m[0] * m[5];
  r[6] = m[3] * m[7] - m[4] * m[6];
  r[7] = m[1] * m[6] - m[0] * m[7];
  r[8] = m[0] * m[4] - m[1] * m[3];
  const double det = m[0] * r[0] + m[1] * r[3] + m[2] * r[6];
  if (!(fabs(det) > 0.0) || !isfinite(det)) {
    for (int k = 0; k < 9; ++k) A[k] = (k % 4 == 0) ? 1.0 : 0.0;
    return;
  }
  for (int k = 0; k < 9; ++k) A[k] = r[k] / det;
}

// out[e] (+)= blk[e] in[e] over elements [e0, e1) (vectors in sorted order)
__global__ void block_apply(int64_t e0, int64_t e1, int ncomp, const double* __restrict__ blk,
                            const double* __restrict__ in, double* __restrict__ out, int add) {
  const int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= e1) return;
  const double* A = blk + e * ncomp * ncomp;
  double v[3], o[3];
  for (int c = 0; c < ncomp; ++c) v[c] = in[e * ncomp + c];
  for (int r = 0; r < ncomp; ++r) {
    double acc = 0.0;
    for (int c = 0; c < ncomp; ++c) acc = fma(A[r * ncomp + c], v[c], acc);
    o[r] = acc;
  }
  for (int r = 0; r < ncomp; ++r) out[e * ncomp + r] = add ? out[e * ncomp + r] + o[r] : o[r];
}

// In place: the chunk's dense block (row-major, d = ncomp * count) becomes
// its inverse, stored column-major (coalesced rows in chunk_apply).  Rows are
// equilibrated first (the poroelastic rows mix tractions and pressures of
// very different scale), then Gauss-Jordan with partial pivoting in shared
// memory: A^-1 = (R A)^-1 R.  A singular block becomes the identity.
__global__ void __launch_bounds__(256)
chunk_invert(const int2* __restrict__ chunks, const int64_t* __restrict__ off, int ncomp,
             double* __restrict__ blk) {
  extern __shared__ double sm[];
  const int d = ncomp * chunks[blockIdx.x].y;
  double* A = sm;
  double* rs = A + d * d;
  double* colk = rs + d;
  __shared__ int piv[kPcChunk * 3];
  __shared__ int singular;
  double* B = blk + off[blockIdx.x];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int f = tid; f < d * d; f += nt) A[f] = B[f];
  if (tid == 0) singular = 0;
  __syncthreads();
  for (int r = tid; r < d; r += nt) {
    double mx = 0.0;
    for (int j = 0; j < d; ++j) mx = fmax(mx, fabs(A[r * d + j]));
    const double sc = mx > 0.0 ? 1.0 / mx : 1.0;
    rs[r] = sc;
    for (int j = 0; j < d; ++j) A[r * d + j] *= sc;
  }
  __syncthreads();
  for (int k = 0; k < d; ++k) {
    if (tid < 32) {   // pivot: argmax_{i >= k} |A[i][k]| (lowest index on ties)
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < d; i += 32) {
        const double v = fabs(A[i * d + k]);
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) {
        piv[k] = bi;
        if (!(best > 0.0)) singular = 1;
      }
    }
    __syncthreads();
    if (singular) break;
    const int p = piv[k];
    if (p != k)
      for (int j = tid; j < d; j += nt) {
        const double t = A[k * d + j];
        A[k * d + j] = A[p * d + j];
        A[p * d + j] = t;
      }
    __syncthreads();
    const double ip = 1.0 / A[k * d + k];
    for (int i = tid; i < d; i += nt) colk[i] = A[i * d + k];
    __syncthreads();
    for (int j = tid; j < d; j += nt) A[k * d + j] = (j == k ? 1.0 : A[k * d + j]) * ip;
    __syncthreads();
    for (int f = tid; f < d * d; f += nt) {
      const int i = f / d, j = f % d;
      if (i == k) continue;
      A[f] = (j == k ? 0.0 : A[f]) - colk[i] * A[k * d + j];
    }
    __syncthreads();
  }
  if (singular) {
    const int ld = d + (d & 1);
    for (int f = tid; f < ld * d; f += nt) B[f] = (f / ld == f % ld) ? 1.0 : 0.0;
    return;
  }
  for (int k = d - 1; k >= 0; --k) {   // undo the row interchanges as column swaps
    const int p = piv[k];
    if (p != k)
      for (int i = tid; i < d; i += nt) {
        const double t = A[i * d + k];
        A[i * d + k] = A[i * d + p];
        A[i * d + p] = t;
      }
    __syncthreads();
  }
  // (R A)^-1 R: column c scaled by rs[c]; stored column-major with the even
  // leading dimension ld = d + (d & 1) (16-byte aligned columns for the
  // double2 loads of chunk_mv; the padding row is 0)
  const int ld = d + (d & 1);
  for (int f = tid; f < ld * d; f += nt) {
    const int c = f / ld, r = f % ld;
    B[f] = r < d ? A[r * d + c] * rs[c] : 0.0;
  }
}

// y (+)= blockdiag(inv) x over the chunks [q0, q0 + gridDim.x) (sorted order).
// CTA per chunk; the d columns are split over G = blockDim / d thread groups
// (thread (r, g) sums columns c = g, g + G, ... of row r with eight
// accumulators: coalesced over r, eight loads in flight), partials summed over
// the groups in a fixed order.
constexpr int kApplyThreads = 256;

// DDM_PC_STREAM=1: the inverse blocks are read with the streaming (evict-first)
// cache hint, so the once-per-step 46 MB (config 3) does not push the Krylov
// basis out of L2
#ifndef DDM_PC_STREAM
#define DDM_PC_STREAM 1
#endif
__device__ __forceinline__ double2 pc_ld(const double2* p) {
#if DDM_PC_STREAM
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

// y_rows (+)= Ai xs for one chunk (d rows, column-major inverse with even
// leading dimension ld): thread (row pair rp, column group g) accumulates
// double2 rows (2 rp, 2 rp + 1) over the columns c = g, g + G, ... with four
// 16-byte loads in flight; the G group partials are summed in a fixed order.
__device__ __forceinline__ void chunk_mv(const double* __restrict__ Ai, int d,
                                         const double* xs, double2* part,
                                         double* __restrict__ y, int add) {
  const int ld = d + (d & 1), RP = ld >> 1;
  const int G = max(1, (int)blockDim.x / RP);
  const int rp = threadIdx.x % RP, g = threadIdx.x / RP;
  if (g < G) {
    const double2* A2 = reinterpret_cast<const double2*>(Ai);
    double2 a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) a[u] = make_double2(0.0, 0.0);
    int c = g;
    for (; c + 3 * G < d; c += 4 * G) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = pc_ld(A2 + (size_t)(c + u * G) * RP + rp);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double xv = xs[c + u * G];
        a[u].x = fma(v[u].x, xv, a[u].x);
        a[u].y = fma(v[u].y, xv, a[u].y);
      }
    }
    for (int u = 0; c < d; c += G, ++u) {
      const double2 v = pc_ld(A2 + (size_t)c * RP + rp);
      const double xv = xs[c];
      a[u & 3].x = fma(v.x, xv, a[u & 3].x);
      a[u & 3].y = fma(v.y, xv, a[u & 3].y);
    }
    part[threadIdx.x] = make_double2((a[0].x + a[1].x) + (a[2].x + a[3].x),
                                     (a[0].y + a[1].y) + (a[2].y + a[3].y));
  }
  __syncthreads();
  if (threadIdx.x < RP) {
    double2 v = make_double2(0.0, 0.0);
    for (int gg = 0; gg < G; ++gg) {
      const double2 q = part[gg * RP + threadIdx.x];
      v.x += q.x;
      v.y += q.y;
    }
    const int r0 = 2 * threadIdx.x;
    y[r0] = add ? y[r0] + v.x : v.x;
    if (r0 + 1 < d) y[r0 + 1] = add ? y[r0 + 1] + v.y : v.y;
  }
}

__global__ void __launch_bounds__(kApplyThreads)
chunk_apply(const int2* __restrict__ chunks, const int64_t* __restrict__ off, int q0, int ncomp,
            const double* __restrict__ inv, const double* __restrict__ x, double* __restrict__ y,
            int add) {
  __shared__ double xs[kPcChunk * 3];
  __shared__ double2 part[kApplyThreads];
  const int q = q0 + blockIdx.x;
  const int2 ch = chunks[q];
  const int d = ncomp * ch.y;
  const int64_t b0 = (int64_t)ch.x * ncomp;
  for (int t = threadIdx.x; t < d; t += blockDim.x) xs[t] = x[b0 + t];
  __syncthreads();
  if (d == 0) return;
  chunk_mv(inv + off[q], d, xs, part, y + b0, add);
}

// The Givens part of an Arnoldi step (block 0 of finish_scale*, all its
// threads): column k of H = h1 + h2 with the previous rotations applied, a
// new rotation zeroing h(k+1,k) = hn, the rotated rhs and the residual
// estimate.  The rotations and the column are staged in shared memory in
// chunks of 256 by the whole block (the serial recurrence of thread 0 used to
// wait on a global load per rotation: ~35 us at k = 180 on config 3).
__device__ void givens_block(int k, double hn, double a, bool broke, const double* __restrict__ dh,
                             double* __restrict__ Hp, double* __restrict__ cs,
                             double* __restrict__ sn, double* __restrict__ g,
                             double* __restrict__ est, double* __restrict__ scal,
                             int* __restrict__ flag) {
  __shared__ double sc[256], ss[256], sy[256];
  double* col = Hp + (size_t)k * (k + 3) / 2;
  double x = 0.0;
  if (threadIdx.x == 0 && !broke) x = dh[0] + dh[k + 1];
  for (int i0 = 0; i0 < k && !broke; i0 += 256) {
    const int n = min(256, k - i0);
    __syncthreads();
    if ((int)threadIdx.x < n) {
      const int i = i0 + threadIdx.x;
      sc[threadIdx.x] = cs[i];
      ss[threadIdx.x] = sn[i];
      sy[threadIdx.x] = dh[i + 1] + dh[k + 2 + i];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int u = 0; u < n; ++u) {
        const double c = sc[u], sv = ss[u], y = sy[u];
        col[i0 + u] = c * x + sv * y;
        x = -sv * x + c * y;
      }
  }
  if (threadIdx.x != 0) return;
  if (broke) {
    est[k] = est[k > 0 ? k - 1 : 0];
    scal[0] = 0.0;
    return;
  }
  const double den = hypot(x, hn);
  cs[k] = x / den;
  sn[k] = hn / den;
  col[k] = den;
  col[k + 1] = 0.0;
  g[k + 1] = -sn[k] * g[k];
  g[k] = cs[k] * g[k];
  est[k] = fabs(g[k + 1]);
  scal[0] = a;
  if (!(hn > 0.0)) flag[0] = k + 1;
}

// One Arnoldi step's small work on the device (batched GMRES, no host round
// trip per step), fused with the normalisation of the next basis vector.
// dh = [h1 (k+1) | h2 (k+1) | -- | ||w||^2] of the CGS2 passes.  Block 0,
// thread 0: column k of the packed Hessenberg Hp(i, k) = Hp[k (k+3)/2 + i]
// becomes h1 + h2 with h(k+1,k) = ||w||, the previous Givens rotations are
// applied, a new one zeroes h(k+1,k), and the rotated rhs g gives the
// residual estimate est[k] = |g[k+1]|; a breakdown (h(k+1,k) = 0) sets
// flag[0] = k + 1 and makes later steps no-ops.  All blocks: dst = w / h(k+1,k)
// (0 after a breakdown).
__global__ void finish_scale(int k, const double* __restrict__ dh, double* __restrict__ Hp,
                             double* __restrict__ cs, double* __restrict__ sn,
                             double* __restrict__ g, double* __restrict__ est,
                             double* __restrict__ scal, int* __restrict__ flag,
                             const double* __restrict__ w, double* __restrict__ dst, int64_t len) {
  const bool broke = flag[0] != 0;
  const double hn = sqrt(dh[2 * (k + 1) + 1]);
  const double a = (!broke && hn > 0.0) ? 1.0 / hn : 0.0;
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < len) dst[j] = a * w[j];
  if (blockIdx.x == 0) givens_block(k, hn, a, broke, dh, Hp, cs, sn, g, est, scal, flag);
}

// finish_scale fused with the leaf-block preconditioner of the next step
// (single rank, leaf blocks covering every row): CTA per chunk q scales its
// rows of the next basis vector (dst = w / h(k+1,k)) and applies the chunk's
// inverse block to them (uf = M^-1 dst), so the next operator apply skips a
// separate preconditioner launch.  CTA 0, thread 0 also does the Givens step
// (as finish_scale).
// kd != nullptr (captured step): k = *kd, dst = V + (k + 1) nloc, and the
// last CTA to finish (ticket) advances *kd for the next step.
__global__ void __launch_bounds__(kApplyThreads)
finish_scale_pc(int k, const double* __restrict__ dh, double* __restrict__ Hp,
                double* __restrict__ cs, double* __restrict__ sn, double* __restrict__ g,
                double* __restrict__ est, double* __restrict__ scal, int* __restrict__ flag,
                const double* __restrict__ w, double* __restrict__ dst,
                const int2* __restrict__ chunks, const int64_t* __restrict__ off, int ncomp,
                const double* __restrict__ inv, double* __restrict__ uf, int* __restrict__ kd,
                int64_t nloc, unsigned* __restrict__ kd_ticket) {
  step_pdl();
  __shared__ double xs[kPcChunk * 3];
  __shared__ double2 part[kApplyThreads];
  if (kd) {
    k = *kd;
    dst += (int64_t)(k + 1) * nloc;
  }
  const bool broke = flag[0] != 0;
  const double hn = sqrt(dh[2 * (k + 1) + 1]);
  const double a = (!broke && hn > 0.0) ? 1.0 / hn : 0.0;
  const int2 ch = chunks[blockIdx.x];
  const int d = ncomp * ch.y;
  const int64_t b0 = (int64_t)ch.x * ncomp;
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    const double v = a * w[b0 + t];
    dst[b0 + t] = v;
    xs[t] = v;
  }
  __syncthreads();
  if (d > 0) chunk_mv(inv + off[blockIdx.x], d, xs, part, uf + b0, 0);
  if (blockIdx.x == 0) givens_block(k, hn, a, broke, dh, Hp, cs, sn, g, est, scal, flag);
  if (kd) {   // every CTA has read k: the last one advances it
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(kd_ticket, 1u) == gridDim.x - 1) {
        *kd = k + 1;
        *kd_ticket = 0u;
      }
    }
  }
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

struct Gm {
  ddm_ctx_s* ctx;
  ddm_tree_s* t;
  cudaStream_t s;
  int ncomp;
  int64_t nloc, lo;       // owned rows (in doubles) and first owned double
  double* part;           // partial dots
  int64_t part_cap;
  double* dh;             // device h buffer

  int nb() const { return (int)std::max<int64_t>(1, std::min<int64_t>(256, nloc / 2048)); }

  // dots of V[0..nvec) (leading dim ld) with w over the owned rows -> dh[off..off+nvec)
  unsigned* ticket;      // [>= nvec] zeroed tickets of the fused dot reductions
  unsigned* ticket_norm; // zeroed ticket of axpy_norm

  int dots(const double* V, int64_t ld, int nvec, const double* w, int off) {
    const int b = nb();
    if ((int64_t)nvec * b > part_cap) return set_error(ctx, DDM_ERR_ARG, "gmres part buffer");
    dim3 grid(b, nvec);
    multi_dot<<<grid, kDotThreads, 0, s>>>(V, ld, w, nloc, b, part, ticket, dh + off, nullptr, 0);
    DDM_CUDA(ctx, cudaGetLastError());
    return allreduce_sum(ctx, dh + off, nvec, s);
  }
  // w += sign V c, then dh[off] = ||w||^2 (owned rows, summed over ranks)
  int axpy_norm(const double* V, int64_t ld, int nvec, const double* c, double sign, double* w,
                int off) {
    const unsigned g = nblk(nloc, kAxRows);
    if ((int64_t)g > part_cap) return set_error(ctx, DDM_ERR_ARG, "gmres part buffer");
    cgs_axpy<true><<<g, kAxRows * kAxGroups, nvec * sizeof(double), s>>>(
        V, ld, nvec, c, sign, w, nloc, part, ticket_norm, dh + off, nullptr, 0);
    DDM_CUDA(ctx, cudaGetLastError());
    return allreduce_sum(ctx, dh + off, 1, s);
  }
  // one Arnoldi step with the step index in device memory (captured once,
  // replayed for every step of a cycle): CGS2 over V[0..k] and w, then
  // finish_scale_pc writes V[k+1], M^-1 V[k+1] and advances *kd
  int cgs2_k(const double* V, int m, double* w, const int* kd, double dgks_eta2) {
    const int b = nb();
    const int gy = std::min(m + 1, 64);
    if ((int64_t)(m + 1) * b > part_cap) return set_error(ctx, DDM_ERR_ARG, "gmres part buffer");
    const unsigned ga = nblk(nloc, kAxRows);
    if ((int64_t)ga > part_cap) return set_error(ctx, DDM_ERR_ARG, "gmres part buffer");
    const size_t shc = (size_t)(m + 1) * sizeof(double);
    // classical Gram-Schmidt with a DGKS-selective second pass decided on
    // the device (eta^2 = dgks_eta2: the second pass runs only when the
    // first cancelled most of ||w||^2); dgks_eta2 = 0 keeps plain CGS2
    const int use_dgks = dgks_eta2 > 0.0 ? 1 : 0;
    static const int rows_env = [] {
      const char* e = getenv("DDM_GMRES_ROWS");
      return e ? atoi(e) : 1;
    }();
    // rows per CTA: 512, or 256 / 128 on smaller systems (>= 32 CTAs)
    static const int rowt_env = [] {
      const char* e = getenv("DDM_GMRES_ROWT");
      return e ? atoi(e) : 0;
    }();
    int rt = rowt_env > 0 ? rowt_env
             : nloc >= 32 * 512 ? 512 : nloc >= 32 * 256 ? 256 : 128;
    if (rt != 128 && rt != 256) rt = 512;
    const int nbr = (int)((nloc + rt - 1) / rt);
    const int rmax = rt >= 512 ? 128 : 256;
    // (small systems keep the vector-parallel kernels: a few row CTAs cannot
    // keep enough loads in flight)
    if (rows_env && !use_dgks && nbr >= (rt == 512 ? 32 : 24) && nbr <= rmax &&
        (int64_t)(m + 1) * nbr <= part_cap) {
      // row-blocked: dots, fused (update + second-pass dots), update + norm
      if (getenv("DDM_GMRES_TRACE")) fprintf(stderr, "[gmres] row-blocked CGS2, %d CTAs, m %d\n", nbr, m);
      {
        const int64_t ln = nloc;
        cudaError_t e0;
        if (rows_env == 2) {
          multi_dot<<<dim3(b, gy), kDotThreads, 0, s>>>(V, nloc, w, nloc, b, part, ticket, dh, kd, 0);
          e0 = cudaGetLastError();
        } else
          e0 = rt == 512 ? launch_step(cgs_rows<0, 512>, nbr, 512, 0, s, V, ln, ln, w, kd, dh, part, ticket)
               : rt == 256 ? launch_step(cgs_rows<0, 256>, nbr, 256, 0, s, V, ln, ln, w, kd, dh, part, ticket)
                           : launch_step(cgs_rows<0, 128>, nbr, 128, 0, s, V, ln, ln, w, kd, dh, part, ticket);
        DDM_CUDA(ctx, e0);
        DDM_CUDA(ctx, rt == 512 ? launch_step(cgs_rows<1, 512>, nbr, 512, 0, s, V, ln, ln, w, kd, dh, part, ticket)
                      : rt == 256 ? launch_step(cgs_rows<1, 256>, nbr, 256, 0, s, V, ln, ln, w, kd, dh, part, ticket)
                                  : launch_step(cgs_rows<1, 128>, nbr, 128, 0, s, V, ln, ln, w, kd, dh, part, ticket));
        DDM_CUDA(ctx, launch_step(cgs_axpy<true>, ga, kAxRows * kAxGroups, shc, s, V, ln, 0,
                                  (const double*)dh, -1.0, w, ln, part, ticket_norm, dh, kd, 1, 0.0));
      }
      DDM_CUDA(ctx, cudaGetLastError());
      return DDM_OK;
    }
    multi_dot<<<dim3(b, gy), kDotThreads, 0, s>>>(V, nloc, w, nloc, b, part, ticket, dh, kd, 0);
    if (use_dgks)
      cgs_axpy<true><<<ga, kAxRows * kAxGroups, shc, s>>>(V, nloc, 0, dh, -1.0, w, nloc, part,
                                                         ticket_norm, dh, kd, 0, dgks_eta2);
    else
      cgs_axpy<false><<<ga, kAxRows * kAxGroups, shc, s>>>(V, nloc, 0, dh, -1.0, w, nloc, nullptr,
                                                          nullptr, nullptr, kd, 0);
    multi_dot<<<dim3(b, gy), kDotThreads, 0, s>>>(V, nloc, w, nloc, b, part, ticket, dh, kd, 1,
                                                  use_dgks);
#ifdef DDM_EXP_DOT2   // timing experiment: the second-pass dots twice
    multi_dot<<<dim3(b, gy), kDotThreads, 0, s>>>(V, nloc, w, nloc, b, part, ticket, dh, kd, 1,
                                                  use_dgks);
#endif
    cgs_axpy<true><<<ga, kAxRows * kAxGroups, shc, s>>>(V, nloc, 0, dh, -1.0, w, nloc, part,
                                                       ticket_norm, dh, kd, 1, dgks_eta2);
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }
  int axpy(const double* V, int64_t ld, int nvec, const double* c, double sign, double* w) {
    const unsigned g = nblk(nloc, kAxRows);
    cgs_axpy<false><<<g, kAxRows * kAxGroups, nvec * sizeof(double), s>>>(
        V, ld, nvec, c, sign, w, nloc, nullptr, nullptr, nullptr, nullptr, 0);
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }
};

}  // namespace

// Chunks of the leaf-block preconditioner: each leaf's sorted element range
// split into ceil(count / kPcChunk) near-equal consecutive chunks; block
// offsets for ncomp components.  Owned chunks: [pc_q_lo, pc_q_hi).
static int pc_build_chunks(ddm_ctx_s* ctx, ddm_tree_s* t, int ncomp, cudaStream_t s) {
  if (t->pc_chunks && t->pc_off_ncomp == ncomp) return DDM_OK;
  std::vector<int> leaves(t->nleaves), start(t->ncells), count(t->ncells);
  DDM_CUDA(ctx, cudaMemcpyAsync(leaves.data(), t->leaves, t->nleaves * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(start.data(), t->c_start, t->ncells * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(count.data(), t->c_count, t->ncells * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  std::vector<std::pair<int, int>> lr;
  for (int c : leaves) lr.push_back({start[c], count[c]});
  std::sort(lr.begin(), lr.end());
  std::vector<int2> ch;
  std::vector<int64_t> off;
  int64_t tot = 0;
  t->pc_q_lo = -1;
  t->pc_q_hi = 0;
  for (const auto& l : lr) {
    const int nc = (l.second + kPcChunk - 1) / kPcChunk;
    for (int q = 0; q < nc; ++q) {
      const int a = l.first + (int)((int64_t)l.second * q / nc);
      const int b = l.first + (int)((int64_t)l.second * (q + 1) / nc);
      if (a >= t->own_el_lo && a < t->own_el_hi) {
        if (t->pc_q_lo < 0) t->pc_q_lo = (int)ch.size();
        t->pc_q_hi = (int)ch.size() + 1;
      }
      ch.push_back(make_int2(a, b - a));
      off.push_back(tot);
      const int64_t d = ncomp * (b - a);
      tot += (d + (d & 1)) * d;   // inverse stored with an even leading dimension (chunk_mv)
    }
  }
  if (t->pc_q_lo < 0) t->pc_q_lo = t->pc_q_hi = 0;
  if (t->pc_chunks) cudaFree(t->pc_chunks);
  if (t->pc_off) cudaFree(t->pc_off);
  if (t->pcl) cudaFree(t->pcl);
  t->pc_chunks = nullptr;
  t->pc_off = nullptr;
  t->pcl = nullptr;
  int rc;
  if ((rc = dalloc(ctx, &t->pc_chunks, ch.size())) || (rc = dalloc(ctx, &t->pc_off, off.size())) ||
      (rc = dalloc(ctx, &t->pcl, (size_t)tot)))
    return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->pc_chunks, ch.data(), ch.size() * sizeof(int2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->pc_off, off.data(), off.size() * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  t->pc_nchunks = (int)ch.size();
  t->pc_off_ncomp = ncomp;
  t->pcl_n = tot;
  std::memset(t->pcl_key, 0, sizeof(t->pcl_key));
  return DDM_OK;
}

// leaf-block inverses for this material / dt (cached on the tree)
static int pc_leaf_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                          cudaStream_t s) {
  const int ncomp = mat->kind == 1 ? 3 : 2;
  int rc = pc_build_chunks(ctx, t, ncomp, s);
  if (rc) return rc;
  const double key[8] = {(double)mat->kind, mat->G, mat->nu, mat->nu_u, mat->alpha, mat->kappa,
                         mat->kind == 1 ? dt : 0.0, 2.0};
  if (std::memcmp(key, t->pcl_key, sizeof(key)) == 0) return DDM_OK;
  if (mat->kind == 1) {
    if (!(dt > 0)) return set_error(ctx, DDM_ERR_ARG, "poroelastic GMRES needs dt > 0");
    rc = launch_poro_chunk_blocks(ctx, t, poro_params(mat, dt), t->pc_nchunks, t->pc_chunks,
                                  t->pc_off, t->pcl, s);
  } else {
    rc = launch_elastic_chunk_blocks(ctx, t, mat->G / (4.0 * M_PI * (1.0 - mat->nu)),
                                     t->pc_nchunks, t->pc_chunks, t->pc_off, t->pcl, s);
  }
  if (rc) return rc;
  const int dmax = ncomp * kPcChunk;
  const size_t shm = ((size_t)dmax * dmax + 2 * dmax) * sizeof(double);
  DDM_CUDA(ctx, cudaFuncSetAttribute(chunk_invert, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)shm));
  chunk_invert<<<t->pc_nchunks, 256, shm, s>>>(t->pc_chunks, t->pc_off, ncomp, t->pcl);
  DDM_CUDA(ctx, cudaGetLastError());
  std::memcpy(t->pcl_key, key, sizeof(key));
  return DDM_OK;
}

int precond_apply(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt, int kind,
                  const double* x_sorted, double* y_sorted, cudaStream_t s) {
  const int ncomp = mat->kind == 1 ? 3 : 2;
  int rc;
  if (kind == 1) {
    const double key[8] = {(double)mat->kind, mat->G, mat->nu, mat->nu_u, mat->alpha, mat->kappa,
                           mat->kind == 1 ? dt : 0.0, 1.0};
    if (!t->pc || std::memcmp(key, t->pc_key, sizeof(key)) != 0) {
      if (!t->pc && (rc = dalloc(ctx, &t->pc, (size_t)t->n * 9))) return rc;
      rc = mat->kind == 1
               ? launch_poro_self_blocks(ctx, t, poro_params(mat, dt), t->pc, s)
               : launch_elastic_self_blocks(ctx, t, mat->G / (4.0 * M_PI * (1.0 - mat->nu)), t->pc, s);
      if (rc) return rc;
      invert_blocks<<<nblk(t->n, 256), 256, 0, s>>>(t->n, ncomp, t->pc);
      DDM_CUDA(ctx, cudaGetLastError());
      std::memcpy(t->pc_key, key, sizeof(key));
    }
    block_apply<<<nblk(t->n, 256), 256, 0, s>>>(0, t->n, ncomp, t->pc, x_sorted, y_sorted, 0);
  } else {
    if ((rc = pc_leaf_blocks(ctx, t, mat, dt, s))) return rc;
    chunk_apply<<<t->pc_nchunks, kApplyThreads, 0, s>>>(t->pc_chunks, t->pc_off, 0, ncomp, t->pcl, x_sorted,
                                              y_sorted, 0);
  }
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// y = M^-1 x in user order (ddm_precond_apply)
int precond_apply_user(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                       int kind, const double* x_user, double* y_user, cudaStream_t s) {
  const int ncomp = mat->kind == 1 ? 3 : 2;
  const int64_t n = t->n;
  double *xs = nullptr, *ys = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&xs, (size_t)n * ncomp * sizeof(double), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&ys, (size_t)n * ncomp * sizeof(double), s));
  gather_sorted<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, x_user, xs);
  int rc = precond_apply(ctx, t, mat, dt, kind, xs, ys, s);
  if (!rc) {
    scatter_to_user<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, ys, y_user);
    rc = cuda_error_if(ctx, cudaGetLastError(), "scatter_to_user");
  }
  cudaFreeAsync(xs, s);
  cudaFreeAsync(ys, s);
  if (!rc) rc = cuda_error_if(ctx, cudaStreamSynchronize(s), "precond_apply");
  return rc;
}

int gmres_solve(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                const double* b_user, double* x_user, double tol, int restart, int max_iter,
                int mode, int* iters_out, double* rel_out, cudaStream_t s) {
  const int ncomp = mat->kind == 1 ? 3 : 2;
  const bool use_pc = !(mode & DDM_GMRES_NO_PRECOND);
  const bool pc_point = (mode & DDM_GMRES_PC_POINT) != 0;
  mode &= ~(DDM_GMRES_NO_PRECOND | DDM_GMRES_PC_POINT);
  const int64_t n = t->n;
  const int64_t nfull = n * ncomp;
  const int64_t lo = t->own_el_lo * ncomp;
  const int64_t nloc = (t->own_el_hi - t->own_el_lo) * ncomp;
  const int m = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)restart,
                                                               (int64_t)std::max(max_iter, 1), nfull}));
  int rc;
  // workspace: Krylov basis (owned rows), full vectors, partials
  if (t->krylov_m < m + 1 || t->krylov_dof != nloc) {
    if (t->krylov) cudaFree(t->krylov);
    t->krylov = nullptr;
    if ((rc = dalloc(ctx, &t->krylov, (size_t)(m + 1) * std::max<int64_t>(nloc, 1)))) return rc;
    t->krylov_m = m + 1;
    t->krylov_dof = nloc;
  }
  if (!t->gm_w) {
    // gm_w: 6 full vectors (b, x, v, w, u, trial x); gm_tmp: h buffer
    if ((rc = dalloc(ctx, &t->gm_w, (size_t)6 * 3 * n))) return rc;
  }
  if (use_pc && mat->kind == 1 && !(dt > 0))
    return set_error(ctx, DDM_ERR_ARG, "poroelastic GMRES needs dt > 0");
  const int64_t part_need = std::max<int64_t>((int64_t)(m + 2) * std::max<int64_t>(256, nloc / 128 + 1),
                                              2 * (nloc / 64 + 2));
  if (t->gm_part_n < part_need) {
    if (t->gm_part) cudaFree(t->gm_part);
    if ((rc = dalloc(ctx, &t->gm_part, part_need))) return rc;
    t->gm_part_n = part_need;
    if (t->gm_tmp) cudaFree(t->gm_tmp);
    if ((rc = dalloc(ctx, &t->gm_tmp, (size_t)3 * (m + 2)))) return rc;
  }
  double* bs = t->gm_w;
  double* xs = t->gm_w + nfull;
  double* vf = t->gm_w + 2 * nfull;
  double* wf = t->gm_w + 3 * nfull;
  double* uf = t->gm_w + 4 * nfull;   // preconditioned operand M^-1 v (full) / update V y
  double* xt = t->gm_w + 5 * nfull;   // trial iterate (true-residual check)
  double* V = t->krylov;
  if (t->gm_ticket_n < m + 4) {
    if (t->gm_ticket) cudaFree(t->gm_ticket);
    t->gm_ticket = nullptr;
    t->gm_ticket_n = 0;
    DDM_CUDA(ctx, cudaMalloc((void**)&t->gm_ticket, (size_t)(m + 4) * sizeof(unsigned)));
    DDM_CUDA(ctx, cudaMemsetAsync(t->gm_ticket, 0, (size_t)(m + 4) * sizeof(unsigned), s));
    t->gm_ticket_n = m + 4;
  }
  Gm g{ctx, t, s, ncomp, nloc, lo, t->gm_part, t->gm_part_n, t->gm_tmp, t->gm_ticket,
       t->gm_ticket + m + 3};
  // DDM_GMRES_SYNC=1: the host takes every Arnoldi step's decisions (Givens,
  // DGKS reorthogonalisation); default: batched device-side steps
  static const bool sync_mode = [] {
    const char* e = getenv("DDM_GMRES_SYNC");
    return e && e[0] == '1';
  }();
  static const int batch = [] {
    const char* e = getenv("DDM_GMRES_BATCH");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  const size_t hp_n = (size_t)(m + 1) * (m + 4) / 2;
  const int dev_need = (int)std::min<size_t>(hp_n + 4 * (size_t)m + 8, (size_t)INT32_MAX);
  if (!sync_mode && t->gm_dev_m < dev_need) {
    if (t->gm_dev) cudaFree(t->gm_dev);
    t->gm_dev = nullptr;
    t->gm_dev_m = 0;
    if ((rc = dalloc(ctx, &t->gm_dev, (size_t)dev_need))) return rc;
    t->gm_dev_m = dev_need;
  }
  double* Hd = t->gm_dev;
  double* csd = Hd + hp_n;
  double* snd = csd + m;
  double* gd = snd + m;
  double* estd = gd + m + 1;
  double* scald = estd + m;
  int* flagd = reinterpret_cast<int*>(scald + 2);

  // GMRES applies the operator many times at one elapsed time: build the
  // poroelastic near-field cache up front instead of on the
  // second matvec
  if (mat->kind == 1 && (mode & 0xff) == DDM_FMM && dt > 0) {
    if ((rc = fmm_workspace(ctx, t, s))) return rc;
    const PoroParams P = poro_params(mat, dt);
    for (int k = 0; k < 2; ++k)
      if ((rc = poro_near_cache_update(ctx, t, P, s))) return rc;
  }
  gather_sorted<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, b_user, bs);
  gather_sorted<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, x_user, xs);
  DDM_CUDA(ctx, cudaGetLastError());

  // operator: A M^-1 (right preconditioning) or A
  auto apply = [&](const double* vfull) -> int {
    if (!use_pc) return fmm_matvec(ctx, t, mat, dt, vfull, true, nullptr, wf, mode, s);
    int rc2 = precond_apply(ctx, t, mat, dt, pc_point ? 1 : 2, vfull, uf, s);
    if (rc2) return rc2;
    return fmm_matvec(ctx, t, mat, dt, uf, true, nullptr, wf, mode, s);
  };
  // r = b - A x uses A itself (x is in the unpreconditioned space)
  auto apply_plain = [&](const double* vfull) -> int {
    return fmm_matvec(ctx, t, mat, dt, vfull, true, nullptr, wf, mode, s);
  };
  std::vector<double> hh(2 * (m + 1) + 1);
  auto fetch = [&](int cnt) -> int {
    DDM_CUDA(ctx, cudaMemcpyAsync(hh.data(), g.dh, cnt * sizeof(double), cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    return DDM_OK;
  };

  if ((rc = g.dots(bs + lo, 0, 1, bs + lo, 0)) || (rc = fetch(1))) return rc;
  const double bnorm = std::sqrt(hh[0]);
  if (bnorm == 0.0) {
    DDM_CUDA(ctx, cudaMemsetAsync(x_user, 0, nfull * sizeof(double), s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    if (iters_out) *iters_out = 0;
    if (rel_out) *rel_out = 0.0;
    return DDM_OK;
  }
  int iters = 0;
  bool converged = false;
  // Hessenberg matrix, packed by columns: H(i, k) = Hp[k (k + 3) / 2 + i], i <= k + 1.
  // Column k is touched only at step k (contiguous, grows with the basis):
  // a dense (m+1) x m row-major array made every step walk k rows m apart,
  // which costs TLB misses proportional to the restart length, not to k.
  std::vector<double> Hp, cs(m), sn(m), gv(m + 1), y(m);
  auto H = [&Hp](int i, int k) -> double& { return Hp[(size_t)k * (k + 3) / 2 + i]; };
  double rel = 0.0;
  static const bool trace = [] {
    const char* e = getenv("DDM_GMRES_TRACE");
    return e && e[0] == '1';
  }();
  auto now_ms = [] {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t_start = now_ms();
  // DDM_GMRES_CGS2=1: reorthogonalise every step (plain CGS2)
  static const bool always_cgs2 = [] {
    const char* e = getenv("DDM_GMRES_CGS2");
    return e && e[0] == '1';
  }();
  int n_reorth = 0;
  static const double eta2 = [] {
    const char* e = getenv("DDM_GMRES_ETA2");
    return e ? atof(e) : 0.5;
  }();
  bool accepted = false;
  // dst (full) = x + M^-1 V y (or x + V y), y = H^-1 g over the first kd
  // columns (upper triangular, by columns; gv itself is left intact)
  std::vector<double> gtmp(m + 1);
  auto form_x = [&](int kd, double* dst) -> int {
    for (int i = 0; i < kd; ++i) gtmp[i] = gv[i];
    for (int j = kd - 1; j >= 0; --j) {
      y[j] = gtmp[j] / H(j, j);
      for (int i = 0; i < j; ++i) gtmp[i] -= H(i, j) * y[j];
    }
    DDM_CUDA(ctx, cudaMemcpyAsync(g.dh, y.data(), kd * sizeof(double), cudaMemcpyHostToDevice, s));
    if (dst != xs)
      DDM_CUDA(ctx, cudaMemcpyAsync(dst, xs, nfull * sizeof(double), cudaMemcpyDeviceToDevice, s));
    int rc2;
    if (use_pc) {
      DDM_CUDA(ctx, cudaMemsetAsync(uf + lo, 0, nloc * sizeof(double), s));
      if ((rc2 = g.axpy(V, nloc, kd, g.dh, 1.0, uf + lo))) return rc2;
      if (pc_point) {
        block_apply<<<nblk(t->own_el_hi - t->own_el_lo, 256), 256, 0, s>>>(
            t->own_el_lo, t->own_el_hi, ncomp, t->pc, uf, dst, 1);
      } else if (t->pc_q_hi > t->pc_q_lo) {
        chunk_apply<<<t->pc_q_hi - t->pc_q_lo, kApplyThreads, 0, s>>>(t->pc_chunks, t->pc_off, t->pc_q_lo,
                                                            ncomp, t->pcl, uf, dst, 1);
      }
      DDM_CUDA(ctx, cudaGetLastError());
    } else if ((rc2 = g.axpy(V, nloc, kd, g.dh, 1.0, dst + lo))) {
      return rc2;
    }
    if (ctx->exchange && (rc2 = allgather_sorted(ctx, t, dst, ncomp, s))) return rc2;
    DDM_CUDA(ctx, cudaStreamSynchronize(s));   // y (host) must stay alive until the copy ran
    return DDM_OK;
  };
  for (;;) {
    // r = b - A x
    if ((rc = apply_plain(xs))) return rc;
    sub_scale<<<nblk(nloc, 256), 256, 0, s>>>(bs + lo, wf + lo, V, nloc);
    DDM_CUDA(ctx, cudaGetLastError());
    if ((rc = g.dots(V, 0, 1, V, 0)) || (rc = fetch(1))) return rc;
    const double beta = std::sqrt(hh[0]);
    rel = beta / bnorm;
    if (trace)
      fprintf(stderr, "[gmres] iters %d true rel %.3e at %.1f ms, %d reorthogonalised\n", iters,
              rel, now_ms() - t_start, n_reorth);
    if (beta <= tol * bnorm) { converged = true; break; }
    if (iters >= max_iter) break;
    scale_copy<<<nblk(nloc, 256), 256, 0, s>>>(V, 1.0 / beta, V, nloc);
    DDM_CUDA(ctx, cudaGetLastError());
    std::fill(gv.begin(), gv.end(), 0.0);
    double inner = tol;   // estimate target (relative), tightened when the true residual lags
    gv[0] = beta;
    int kdone = 0;
    if (!sync_mode) {
      // the leaf-block preconditioner of the next step fused into the step's
      // normalisation (one rank, leaf blocks built by the first apply)
      bool uf_ready = false;
      const bool fuse_pc_env = [] {
        const char* e = getenv("DDM_GMRES_FUSE_PC");
        return !(e && e[0] == '0');
      }();
      bool fuse_pc = false;
      // batched: the Arnoldi steps queue back to back on the stream; the
      // host reads the residual estimates every `batch` steps and picks the
      // first step that met the target (later steps of the batch are
      // discarded work, not counted as iterations)
      const int it0 = iters;
      std::vector<double> g0(m + 1, 0.0);
      g0[0] = beta;
      DDM_CUDA(ctx, cudaMemcpyAsync(gd, g0.data(), (m + 1) * sizeof(double), cudaMemcpyHostToDevice, s));
      DDM_CUDA(ctx, cudaMemsetAsync(flagd, 0, sizeof(int), s));
      // residual estimates and breakdown flag read back into pinned host memory
      if (t->gm_pin_n < batch + 2) {
        if (t->gm_pin) cudaFreeHost(t->gm_pin);
        t->gm_pin = nullptr;
        t->gm_pin_n = 0;
        DDM_CUDA(ctx, cudaMallocHost((void**)&t->gm_pin, (size_t)(batch + 2) * sizeof(double)));
        t->gm_pin_n = batch + 2;
      }
      double* hest = t->gm_pin;
      int* hflagp = reinterpret_cast<int*>(t->gm_pin + batch);
      int kb = 0;
      bool stop = false;
      // captured Arnoldi step: from step 1 on, one CUDA
      // graph per step -- operator apply on M^-1 V_k, CGS2 and the fused
      // normalisation + preconditioner -- with k in device memory, so the
      // same graph serves every step (one rank, leaf blocks; DDM_GMRES_GRAPH=0
      // launches the kernels one by one)
      static const bool graph_env = [] {
        const char* e = getenv("DDM_GMRES_GRAPH");
        return !(e && e[0] == '0');
      }();
      int* kdd = reinterpret_cast<int*>(scald + 3);
      unsigned* kd_tick = t->gm_ticket + m + 2;
      bool graph_on = false;
      auto get_step_graph = [&]() -> int {
        const uintptr_t key[12] = {(uintptr_t)V, (uintptr_t)wf, (uintptr_t)uf, (uintptr_t)nloc,
                                   (uintptr_t)m, (uintptr_t)mode, (uintptr_t)t->pcl,
                                   (uintptr_t)mat->kind, 0, 0, 0, 0};
        uintptr_t kk[12];
        std::memcpy(kk, key, sizeof(kk));
        double dd[2] = {dt, mat->G * 1e-9 + mat->nu + mat->nu_u + mat->alpha + mat->kappa * 1e12};
        std::memcpy(&kk[8], &dd[0], sizeof(double));
        std::memcpy(&kk[9], &dd[1], sizeof(double));
        kk[10] = (uintptr_t)Hd;
        kk[11] = (uintptr_t)g.dh;
        if (t->gm_exec && std::memcmp(kk, t->gm_key, sizeof(kk)) == 0) return DDM_OK;
        if (t->gm_exec) cudaGraphExecDestroy(t->gm_exec);
        t->gm_exec = nullptr;
        const cudaStream_t sc = ctx->s_cap;
        cudaGraph_t graph = nullptr;
        DDM_CUDA(ctx, cudaStreamBeginCapture(sc, cudaStreamCaptureModeThreadLocal));
        Gm gc = g;
        gc.s = sc;
        int rc2 = fmm_matvec(ctx, t, mat, dt, uf, true, nullptr, wf, mode, sc);
        // DDM_GMRES_DGKS=1: the second CGS pass only when DGKS asks for it
        // (measured: config 3 44.0 vs 42.1 ms with plain CGS2 -- the first
        // pass cancels most of ||w||^2 in most steps), default plain CGS2
        static const double dgks_eta2 = [] {
          const char* e = getenv("DDM_GMRES_DGKS");
          return (e && e[0] == '1') ? 0.5 : 0.0;
        }();
        if (!rc2) rc2 = gc.cgs2_k(V, m, wf + lo, kdd, dgks_eta2);
        if (!rc2)
          rc2 = cuda_error_if(ctx, launch_step(finish_scale_pc, (unsigned)t->pc_nchunks, kApplyThreads,
                                              0, sc, 0, (const double*)g.dh, Hd, csd, snd, gd, estd,
                                              scald, flagd, (const double*)(wf + lo), V,
                                              (const int2*)t->pc_chunks, (const int64_t*)t->pc_off,
                                              ncomp, (const double*)t->pcl, uf, kdd, (int64_t)nloc,
                                              kd_tick),
                              "finish_scale_pc");
        const cudaError_t ce = cudaStreamEndCapture(sc, &graph);
        if (rc2) {
          if (graph) cudaGraphDestroy(graph);
          return rc2;
        }
        if (ce != cudaSuccess) return cuda_error(ctx, ce, "cudaStreamEndCapture (gmres step)");
        const cudaError_t ie =
            cudaGraphInstantiateWithFlags(&t->gm_exec, graph, cudaGraphInstantiateFlagUseNodePriority);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) {
          t->gm_exec = nullptr;
          return cuda_error(ctx, ie, "cudaGraphInstantiate (gmres step)");
        }
        std::memcpy(t->gm_key, kk, sizeof(kk));
        return DDM_OK;
      };
      // H and g of the first kd steps from the device (for form_x)
      auto fetch_state = [&](int kd) -> int {
        const size_t hn_ = (size_t)kd * (kd + 3) / 2;
        if (Hp.size() < hn_) Hp.resize(hn_);
        DDM_CUDA(ctx, cudaMemcpyAsync(Hp.data(), Hd, hn_ * sizeof(double), cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaMemcpyAsync(gv.data(), gd, (kd + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaStreamSynchronize(s));
        return DDM_OK;
      };
      for (int k = 0; k < m && iters < max_iter; ++k) {
        const double* vk = V + (int64_t)k * nloc;
        const double* vin = vk;
        if (graph_on) {
          if (!uf_ready) {   // uf served as scratch of a true-residual check
            if ((rc = precond_apply(ctx, t, mat, dt, 2, vk, uf, s))) return rc;
            set_int_kernel<<<1, 1, 0, s>>>(kdd, k);
            DDM_CUDA(ctx, cudaGetLastError());
          }
          DDM_CUDA(ctx, cudaGraphLaunch(t->gm_exec, s));
          uf_ready = true;
          ++iters;
          kdone = k + 1;
          if (k + 1 - kb < batch && k + 1 < m && iters < max_iter) continue;
        } else {
        if (ctx->exchange) {
          DDM_CUDA(ctx, cudaMemcpyAsync(vf + lo, vk, nloc * sizeof(double), cudaMemcpyDeviceToDevice, s));
          if ((rc = allgather_sorted(ctx, t, vf, ncomp, s))) return rc;
          vin = vf;
        }
        if (uf_ready) {   // M^-1 V_k came with the previous step's finish_scale_pc
          if ((rc = fmm_matvec(ctx, t, mat, dt, uf, true, nullptr, wf, mode, s))) return rc;
          uf_ready = false;
        } else if ((rc = apply(vin))) {
          return rc;
        }
        if (k == 0)   // the first apply built the leaf blocks for this material / dt
          fuse_pc = fuse_pc_env && use_pc && !pc_point && !ctx->exchange && t->pc_nchunks > 0;
        double* w = wf + lo;
        // CGS2 (two classical Gram-Schmidt passes, no host decision)
        const int o_w1 = 2 * (k + 1) + 1;
        if ((rc = g.dots(V, nloc, k + 1, w, 0))) return rc;
        if ((rc = g.axpy(V, nloc, k + 1, g.dh, -1.0, w))) return rc;
        if ((rc = g.dots(V, nloc, k + 1, w, k + 1))) return rc;
        if ((rc = g.axpy_norm(V, nloc, k + 1, g.dh + k + 1, -1.0, w, o_w1))) return rc;
        if (fuse_pc) {
          finish_scale_pc<<<t->pc_nchunks, kApplyThreads, 0, s>>>(
              k, g.dh, Hd, csd, snd, gd, estd, scald, flagd, w, V + (int64_t)(k + 1) * nloc,
              t->pc_chunks, t->pc_off, ncomp, t->pcl, uf, nullptr, 0, nullptr);
          uf_ready = true;   // uf = M^-1 V_{k+1} for the next step's operator apply
        } else {
          finish_scale<<<nblk(nloc, 256), 256, 0, s>>>(k, g.dh, Hd, csd, snd, gd, estd, scald,
                                                       flagd, w, V + (int64_t)(k + 1) * nloc, nloc);
        }
        DDM_CUDA(ctx, cudaGetLastError());
        ++iters;
        kdone = k + 1;
        if (k == 0 && fuse_pc && graph_env && ctx->world == 1 && !ctx->exchange && !ctx->profiling &&
            ctx->s_cap && m > 1) {
          if ((rc = get_step_graph())) return rc;
          set_int_kernel<<<1, 1, 0, s>>>(kdd, 1);
          DDM_CUDA(ctx, cudaGetLastError());
          graph_on = true;
        }
        if (k + 1 - kb < batch && k + 1 < m && iters < max_iter) continue;
        }
        DDM_CUDA(ctx, cudaMemcpyAsync(hest, estd + kb, (k + 1 - kb) * sizeof(double),
                                      cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaMemcpyAsync(hflagp, flagd, sizeof(int), cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaStreamSynchronize(s));
        const int hflag = *hflagp;
        for (int kk = kb; kk <= k; ++kk) {
          const bool brk = hflag && kk + 1 >= hflag;   // h(kk+1, kk) = 0
          const bool est_ok = hest[kk - kb] <= inner * bnorm;
          if (!est_ok && !brk) continue;
          const int it_kk = it0 + kk + 1;
          if (est_ok && !brk && kk + 1 < m && it_kk < max_iter) {
            // the estimate says converged: check the true residual without
            // ending the cycle (as in the synchronous path); uf is reused as
            // scratch, so the next step applies the preconditioner itself
            uf_ready = false;
            if ((rc = fetch_state(kk + 1)) || (rc = form_x(kk + 1, xt))) return rc;
            if ((rc = apply_plain(xt))) return rc;
            sub_scale<<<nblk(nloc, 256), 256, 0, s>>>(bs + lo, wf + lo, uf + lo, nloc);
            DDM_CUDA(ctx, cudaGetLastError());
            if ((rc = g.dots(uf + lo, 0, 1, uf + lo, 0)) || (rc = fetch(1))) return rc;
            const double tr = std::sqrt(hh[0]);
            if (trace)
              fprintf(stderr, "[gmres] iters %d estimate %.3e true %.3e\n", it_kk,
                      hest[kk - kb] / bnorm, tr / bnorm);
            if (tr <= tol * bnorm) {
              DDM_CUDA(ctx, cudaMemcpyAsync(xs, xt, nfull * sizeof(double), cudaMemcpyDeviceToDevice, s));
              rel = tr / bnorm;
              converged = accepted = true;
              iters = it_kk;
              break;
            }
            inner = std::min(inner, hest[kk - kb] / bnorm) * 0.5 * (tol * bnorm / tr);
            continue;
          }
          // end of the cycle at step kk (estimate met at the cycle's end or
          // max_iter, or breakdown): restart from x + M^-1 V y
          kdone = kk + 1;
          iters = it_kk;
          stop = true;
          break;
        }
        kb = k + 1;
        if (accepted || stop) break;
      }
      if (!accepted && (rc = fetch_state(kdone))) return rc;
    } else
    for (int k = 0; k < m; ++k) {
      const double* vk = V + (int64_t)k * nloc;
      const double* vin = vk;
      if (ctx->exchange) {
        DDM_CUDA(ctx, cudaMemcpyAsync(vf + lo, vk, nloc * sizeof(double), cudaMemcpyDeviceToDevice, s));
        if ((rc = allgather_sorted(ctx, t, vf, ncomp, s))) return rc;
        vin = vf;
      }
      if ((rc = apply(vin))) return rc;
      double* w = wf + lo;
      // classical Gram-Schmidt with selective reorthogonalisation (DGKS,
      // eta = 1/sqrt(2)): one pass h = V^T w, w -= V h; a second pass only
      // when it cancelled most of w (||w'|| < eta ||w||), where a single
      // pass loses orthogonality.  dh layout: [h1 (k+1) | h2 (k+1) | ||w||^2 | ||w'||^2]
      const int o_w0 = 2 * (k + 1), o_w1 = o_w0 + 1;
      if ((rc = g.dots(V, nloc, k + 1, w, 0))) return rc;
      if ((rc = g.dots(w, 0, 1, w, o_w0))) return rc;
      if ((rc = g.axpy(V, nloc, k + 1, g.dh, -1.0, w))) return rc;
      if ((rc = g.dots(w, 0, 1, w, o_w1))) return rc;
      if ((rc = fetch(o_w1 + 1))) return rc;
      bool reorth = !(hh[o_w1] >= eta2 * hh[o_w0]) || always_cgs2;
      if (reorth) {
        if ((rc = g.dots(V, nloc, k + 1, w, k + 1))) return rc;
        if ((rc = g.axpy(V, nloc, k + 1, g.dh + k + 1, -1.0, w))) return rc;
        if ((rc = g.dots(w, 0, 1, w, o_w1))) return rc;
        if ((rc = fetch(o_w1 + 1))) return rc;
        ++n_reorth;
      }
      const double hn = std::sqrt(hh[o_w1]);
      if (Hp.size() < (size_t)(k + 1) * (k + 4) / 2) Hp.resize((size_t)(k + 1) * (k + 4) / 2);
      for (int i = 0; i <= k; ++i) H(i, k) = hh[i] + (reorth ? hh[k + 1 + i] : 0.0);
      H(k + 1, k) = hn;
      if (hn > 0.0) {
        scale_copy<<<nblk(nloc, 256), 256, 0, s>>>(w, 1.0 / hn, V + (int64_t)(k + 1) * nloc, nloc);
        DDM_CUDA(ctx, cudaGetLastError());
      }
      for (int i = 0; i < k; ++i) {
        const double a = H(i, k), bb = H(i + 1, k);
        H(i, k) = cs[i] * a + sn[i] * bb;
        H(i + 1, k) = -sn[i] * a + cs[i] * bb;
      }
      const double a = H(k, k), bb = H(k + 1, k);
      const double den = std::hypot(a, bb);
      cs[k] = a / den;
      sn[k] = bb / den;
      H(k, k) = den;
      H(k + 1, k) = 0.0;
      gv[k + 1] = -sn[k] * gv[k];
      gv[k] = cs[k] * gv[k];
      ++iters;
      kdone = k + 1;
      const bool est_ok = std::fabs(gv[k + 1]) <= inner * bnorm;
      if (est_ok && kdone < m && iters < max_iter && hn != 0.0) {
        // the estimate says converged: check the true residual of the
        // iterate without ending the cycle.  Near the operator's accuracy
        // floor the two differ; a restart here would rebuild the Krylov
        // space from one vector and crawl (one step per cycle).
        if ((rc = form_x(kdone, xt))) return rc;
        if ((rc = apply_plain(xt))) return rc;
        sub_scale<<<nblk(nloc, 256), 256, 0, s>>>(bs + lo, wf + lo, uf + lo, nloc);
        DDM_CUDA(ctx, cudaGetLastError());
        if ((rc = g.dots(uf + lo, 0, 1, uf + lo, 0)) || (rc = fetch(1))) return rc;
        const double tr = std::sqrt(hh[0]);
        if (trace)
          fprintf(stderr, "[gmres] iters %d estimate %.3e true %.3e\n", iters,
                  std::fabs(gv[k + 1]) / bnorm, tr / bnorm);
        if (tr <= tol * bnorm) {
          DDM_CUDA(ctx, cudaMemcpyAsync(xs, xt, nfull * sizeof(double), cudaMemcpyDeviceToDevice, s));
          rel = tr / bnorm;
          converged = accepted = true;
          break;
        }
        inner = std::min(inner, std::fabs(gv[k + 1]) / bnorm) * 0.5 * (tol * bnorm / tr);
        continue;
      }
      if (est_ok || iters >= max_iter || hn == 0.0) break;
    }
    if (accepted) break;
    if ((rc = form_x(kdone, xs))) return rc;
  }
  if (ctx->exchange && (rc = allgather_sorted(ctx, t, xs, ncomp, s))) return rc;
  scatter_to_user<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, xs, x_user);
  DDM_CUDA(ctx, cudaGetLastError());
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  if (iters_out) *iters_out = iters;
  if (rel_out) *rel_out = rel;
  if (!converged)
    return set_error(ctx, DDM_ERR_NOCONV, "GMRES reached max_iter before tol");
  return DDM_OK;
}

}  // namespace ddm
