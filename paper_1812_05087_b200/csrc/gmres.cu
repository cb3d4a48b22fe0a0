// GMRES with the FMM operator (DESIGN.md §4.1 row a12, §4.7; "a modified
// version of GMRES with FMM for matrix-vector multiplication"; reading R11):
// restarted GMRES, Arnoldi by classical Gram-Schmidt applied twice (CGS2),
// Givens rotations, relative residual ||b - A x|| / ||b|| <= tol.
//
// Vectors live in Morton-sorted order; each rank keeps its owned rows
// [own_el_lo, own_el_hi) of every Krylov vector.  Per iteration: one all-gather
// of the new basis vector (multi-GPU only), the matvec, two batched dot passes
// (each one all-reduce of k+1 partial dots) and one norm.  The small Hessenberg
// least-squares problem is solved on the host.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "kcommon.cuh"

namespace ddm {
namespace {

constexpr int kDotThreads = 256;

// part[i * nb + b] = sum over chunk b of V[i * ld + j] * w[j]
__global__ void __launch_bounds__(kDotThreads)
multi_dot(const double* __restrict__ V, int64_t ld, const double* __restrict__ w, int64_t len,
          int nb, double* __restrict__ part) {
  const int i = blockIdx.y, b = blockIdx.x;
  const int64_t chunk = (len + nb - 1) / nb;
  const int64_t j0 = b * chunk, j1 = min(len, j0 + chunk);
  const double* v = V + (int64_t)i * ld;
  double acc = 0.0;
  for (int64_t j = j0 + threadIdx.x; j < j1; j += kDotThreads) acc = fma(v[j], w[j], acc);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double sh[kDotThreads / 32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < kDotThreads / 32; ++k) s += sh[k];
    part[(int64_t)i * nb + b] = s;
  }
}

// out[i] = sum_b part[i * nb + b] in a fixed order (deterministic)
__global__ void reduce_parts(const double* __restrict__ part, int nvec, int nb,
                             double* __restrict__ out) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= nvec) return;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += part[(int64_t)i * nb + b];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[i] = s;
}

// w[j] += sign * sum_i V[i * ld + j] c[i]: eight independent accumulators
// per thread (eight loads of the basis in flight), summed in a fixed order
__global__ void multi_axpy(const double* __restrict__ V, int64_t ld, int nvec,
                           const double* __restrict__ c, double sign, double* __restrict__ w,
                           int64_t len) {
  extern __shared__ double sc[];
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) sc[i] = c[i];
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < len;
       j += (int64_t)gridDim.x * blockDim.x) {
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    const double* v = V + j;
    int i = 0;
    for (; i + 8 <= nvec; i += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = fma(__ldg(v + (int64_t)(i + q) * ld), sc[i + q], a[q]);
    }
    for (int q = 0; i < nvec; ++i, ++q) a[q] = fma(__ldg(v + (int64_t)i * ld), sc[i], a[q]);
    const double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    w[j] = fma(sign, acc, w[j]);
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
  int dots(const double* V, int64_t ld, int nvec, const double* w, int off) {
    const int b = nb();
    if ((int64_t)nvec * b > part_cap) return set_error(ctx, DDM_ERR_ARG, "gmres part buffer");
    dim3 grid(b, nvec);
    multi_dot<<<grid, kDotThreads, 0, s>>>(V, ld, w, nloc, b, part);
    DDM_CUDA(ctx, cudaGetLastError());
    reduce_parts<<<nblk(nvec, 8), 256, 0, s>>>(part, nvec, b, dh + off);
    DDM_CUDA(ctx, cudaGetLastError());
    return allreduce_sum(ctx, dh + off, nvec, s);
  }
  int axpy(const double* V, int64_t ld, int nvec, const double* c, double sign, double* w) {
    const unsigned g = std::min(nblk(nloc, 256), 148u * 8);
    multi_axpy<<<g, 256, nvec * sizeof(double), s>>>(V, ld, nvec, c, sign, w, nloc);
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }
};

}  // namespace

int gmres_solve(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                const double* b_user, double* x_user, double tol, int restart, int max_iter,
                int mode, int* iters_out, double* rel_out, cudaStream_t s) {
  const int ncomp = mat->kind == 1 ? 3 : 2;
  const bool use_pc = !(mode & DDM_GMRES_NO_PRECOND);
  mode &= ~DDM_GMRES_NO_PRECOND;
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
    // gm_w: 5 full vectors (b, x, v, w, u); gm_tmp: h buffer
    if ((rc = dalloc(ctx, &t->gm_w, (size_t)5 * 3 * n))) return rc;
  }
  if (use_pc) {
    // block-Jacobi: inverse self blocks for this material and elapsed time
    const double key[8] = {(double)mat->kind, mat->G, mat->nu, mat->nu_u, mat->alpha, mat->kappa,
                           mat->kind == 1 ? dt : 0.0, 1.0};
    if (!t->pc || std::memcmp(key, t->pc_key, sizeof(key)) != 0) {
      if (!t->pc && (rc = dalloc(ctx, &t->pc, (size_t)n * 9))) return rc;
      if (mat->kind == 1) {
        if (!(dt > 0)) return set_error(ctx, DDM_ERR_ARG, "poroelastic GMRES needs dt > 0");
        rc = launch_poro_self_blocks(ctx, t, poro_params(mat, dt), t->pc, s);
      } else {
        rc = launch_elastic_self_blocks(ctx, t, mat->G / (4.0 * M_PI * (1.0 - mat->nu)), t->pc, s);
      }
      if (rc) return rc;
      invert_blocks<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->pc);
      DDM_CUDA(ctx, cudaGetLastError());
      std::memcpy(t->pc_key, key, sizeof(key));
    }
  }
  const int64_t part_need = (int64_t)(m + 2) * 256;
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
  double* V = t->krylov;
  Gm g{ctx, t, s, ncomp, nloc, lo, t->gm_part, t->gm_part_n, t->gm_tmp};

  gather_sorted<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, b_user, bs);
  gather_sorted<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, t->perm, x_user, xs);
  DDM_CUDA(ctx, cudaGetLastError());

  // operator: A M^-1 (right preconditioning) or A
  auto apply = [&](const double* vfull) -> int {
    if (!use_pc) return fmm_matvec(ctx, t, mat, dt, vfull, true, nullptr, wf, mode, s);
    block_apply<<<nblk(n, 256), 256, 0, s>>>(0, n, ncomp, t->pc, vfull, uf, 0);
    DDM_CUDA(ctx, cudaGetLastError());
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
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gv(m + 1), y(m);
  double rel = 0.0;
  for (;;) {
    // r = b - A x
    if ((rc = apply_plain(xs))) return rc;
    sub_scale<<<nblk(nloc, 256), 256, 0, s>>>(bs + lo, wf + lo, V, nloc);
    DDM_CUDA(ctx, cudaGetLastError());
    if ((rc = g.dots(V, 0, 1, V, 0)) || (rc = fetch(1))) return rc;
    const double beta = std::sqrt(hh[0]);
    rel = beta / bnorm;
    if (beta <= tol * bnorm) { converged = true; break; }
    if (iters >= max_iter) break;
    scale_copy<<<nblk(nloc, 256), 256, 0, s>>>(V, 1.0 / beta, V, nloc);
    DDM_CUDA(ctx, cudaGetLastError());
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int kdone = 0;
    for (int k = 0; k < m; ++k) {
      const double* vk = V + (int64_t)k * nloc;
      const double* vin = vk;
      if (ctx->world > 1) {
        DDM_CUDA(ctx, cudaMemcpyAsync(vf + lo, vk, nloc * sizeof(double), cudaMemcpyDeviceToDevice, s));
        if ((rc = allgather_sorted(ctx, t, vf, ncomp, s))) return rc;
        vin = vf;
      }
      if ((rc = apply(vin))) return rc;
      double* w = wf + lo;
      // CGS2: two classical Gram-Schmidt passes
      if ((rc = g.dots(V, nloc, k + 1, w, 0))) return rc;
      if ((rc = g.axpy(V, nloc, k + 1, g.dh, -1.0, w))) return rc;
      if ((rc = g.dots(V, nloc, k + 1, w, k + 1))) return rc;
      if ((rc = g.axpy(V, nloc, k + 1, g.dh + k + 1, -1.0, w))) return rc;
      if ((rc = g.dots(w, 0, 1, w, 2 * (k + 1)))) return rc;
      if ((rc = fetch(2 * (k + 1) + 1))) return rc;
      const double hn = std::sqrt(hh[2 * (k + 1)]);
      for (int i = 0; i <= k; ++i) H[(size_t)i * m + k] = hh[i] + hh[k + 1 + i];
      H[(size_t)(k + 1) * m + k] = hn;
      if (hn > 0.0) {
        scale_copy<<<nblk(nloc, 256), 256, 0, s>>>(w, 1.0 / hn, V + (int64_t)(k + 1) * nloc, nloc);
        DDM_CUDA(ctx, cudaGetLastError());
      }
      for (int i = 0; i < k; ++i) {
        const double a = H[(size_t)i * m + k], bb = H[(size_t)(i + 1) * m + k];
        H[(size_t)i * m + k] = cs[i] * a + sn[i] * bb;
        H[(size_t)(i + 1) * m + k] = -sn[i] * a + cs[i] * bb;
      }
      const double a = H[(size_t)k * m + k], bb = H[(size_t)(k + 1) * m + k];
      const double den = std::hypot(a, bb);
      cs[k] = a / den;
      sn[k] = bb / den;
      H[(size_t)k * m + k] = den;
      H[(size_t)(k + 1) * m + k] = 0.0;
      gv[k + 1] = -sn[k] * gv[k];
      gv[k] = cs[k] * gv[k];
      ++iters;
      kdone = k + 1;
      if (std::fabs(gv[k + 1]) <= tol * bnorm || iters >= max_iter || hn == 0.0) break;
    }
    // y = H^-1 g (upper triangular), x += V y
    for (int i = kdone - 1; i >= 0; --i) {
      double acc = gv[i];
      for (int j = i + 1; j < kdone; ++j) acc -= H[(size_t)i * m + j] * y[j];
      y[i] = acc / H[(size_t)i * m + i];
    }
    DDM_CUDA(ctx, cudaMemcpyAsync(g.dh, y.data(), kdone * sizeof(double), cudaMemcpyHostToDevice, s));
    if (use_pc) {   // x += M^-1 (V y)
      DDM_CUDA(ctx, cudaMemsetAsync(uf + lo, 0, nloc * sizeof(double), s));
      if ((rc = g.axpy(V, nloc, kdone, g.dh, 1.0, uf + lo))) return rc;
      block_apply<<<nblk(t->own_el_hi - t->own_el_lo, 256), 256, 0, s>>>(
          t->own_el_lo, t->own_el_hi, ncomp, t->pc, uf, xs, 1);
      DDM_CUDA(ctx, cudaGetLastError());
    } else if ((rc = g.axpy(V, nloc, kdone, g.dh, 1.0, xs + lo))) {
      return rc;
    }
    if (ctx->world > 1 && (rc = allgather_sorted(ctx, t, xs, ncomp, s))) return rc;
    DDM_CUDA(ctx, cudaStreamSynchronize(s));   // y (host) must stay alive until the copy ran
  }
  if (ctx->world > 1 && (rc = allgather_sorted(ctx, t, xs, ncomp, s))) return rc;
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
