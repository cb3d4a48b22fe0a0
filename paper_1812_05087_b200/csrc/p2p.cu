// Near field (a10) and direct evaluation of the elastic constant-DD kernel
// (rows a5-prep and a10).  The exact element influence is
// evaluated in Kolosov–Muskhelishvili form: "the direct
// multiplication ... is used for points that are not well-separated"
// (P:536-538), "P2P term, to account for the self and neighbor interactions"
// (P:868-877).
#include "kcommon.cuh"

namespace ddm {
namespace {

// Per element (sorted order), from the DDs (D_s, D_n) and geometry:
//   e = e^{i beta}, B = (D_s + i D_n) e, r = conj(e)^2, Bh = B/2,
//   Q' = Q - 2 B r = -(r B + conj B), P1 = Bh (r - 1), P2 = i Bh (r + 1)
//   src = {z1, z2, P1, P2, Bh, Q'}  (12 doubles, kSrcStride)
__global__ void prep_sources(int64_t n, int ncomp, const int* __restrict__ perm,
                             const double* __restrict__ D, const double* __restrict__ ex,
                             const double* __restrict__ ey, const double* __restrict__ ea,
                             const double* __restrict__ ec, const double* __restrict__ es,
                             double* __restrict__ src, double* __restrict__ dsort) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm ? perm[i] : (int)i;
  const double ds = D[(int64_t)j * ncomp + 0];
  const double dn = D[(int64_t)j * ncomp + 1];
  if (dsort) {   // D gathered into sorted order for the upward pass
    dsort[i * ncomp + 0] = ds;
    dsort[i * ncomp + 1] = dn;
  }
  const double c = ec[i], s = es[i], a = ea[i];
  const double2 B = make_double2(ds * c - dn * s, ds * s + dn * c);
  const double2 r = make_double2(c * c - s * s, -2.0 * c * s);
  const double2 rB = cmul(r, B);
  const double2 Qp = make_double2(-(rB.x + B.x), -(rB.y - B.y));
  const double2 Bh = make_double2(0.5 * B.x, 0.5 * B.y);
  const double2 P1 = cmul(Bh, make_double2(r.x - 1.0, r.y));
  const double2 T2 = cmul(Bh, make_double2(r.x + 1.0, r.y));
  double2* o = reinterpret_cast<double2*>(src + i * kSrcStride);
  o[0] = make_double2(ex[i] - a * c, ey[i] - a * s);
  o[1] = make_double2(ex[i] + a * c, ey[i] + a * s);
  o[2] = P1;
  o[3] = make_double2(-T2.y, T2.x);    // P2 = i Bh (r + 1)
  o[4] = Bh;
  o[5] = Qp;
}

// Contribution of source element (z1, z2, P1, P2, Bh, Q') to the target at z:
//   r1 = 1/(z - z1), r2 = 1/(z - z2), I2 = r2 - r1, I3 = I2 (r1 + r2)/2
//   Phi           += i G C B I2                 -> phi += Im(Bh I2)
//   zb Phi' + Psi += i G C I2 [Q' + B (r D - conj D)(r1 + r2)/2],  D = z - zc
// with Bh (r D2 - conj D2) = dx P1 + dy P2 for D2 = 2 D = dx + i dy.
// 36 fp64-pipe instructions + 1 MUFU.RCP64H; r1, r2 share one reciprocal.
struct P2PAcc {
  double phi = 0.0;
  double2 psi = make_double2(0.0, 0.0);
};

__device__ __forceinline__ void pair_update(P2PAcc& acc, double zx, double zy, const double* sp) {
  const double w1x = zx - sp[0], w1y = zy - sp[1];
  const double w2x = zx - sp[2], w2y = zy - sp[3];
  const double n1 = fma(w1x, w1x, w1y * w1y);
  const double n2 = fma(w2x, w2x, w2y * w2y);
  const double inv = fast_rcp(n1 * n2);
  const double i1 = n2 * inv, i2 = n1 * inv;
  const double r1x = w1x * i1, r1y = -w1y * i1;        // r1 = conj(w1)/|w1|^2
  const double I2x = fma(w2x, i2, -r1x), I2y = fma(-w2y, i2, -r1y);   // r2 - r1
  const double Sx = fma(w2x, i2, r1x), Sy = fma(-w2y, i2, r1y);       // r2 + r1
  const double dx = w1x + w2x, dy = w1y + w2y;   // 2 (z - zc)
  const double BXx = fma(dx, sp[4], dy * sp[6]);
  const double BXy = fma(dx, sp[5], dy * sp[7]);
  const double Vx = fma(BXx, Sx, fma(-BXy, Sy, sp[10]));
  const double Vy = fma(BXx, Sy, fma(BXy, Sx, sp[11]));
  acc.psi.x = fma(I2x, Vx, fma(-I2y, Vy, acc.psi.x));
  acc.psi.y = fma(I2x, Vy, fma(I2y, Vx, acc.psi.y));
  acc.phi = fma(sp[8], I2y, fma(sp[9], I2x, acc.phi));
}

// traction (sigma_s, sigma_n) at a target with direction (ct, st):
//   T = sigma_n + i sigma_s = 2 Re Phi + e^{2 i bt} (zb Phi' + Psi)
__device__ __forceinline__ double2 acc_to_traction(const P2PAcc& a, double gc, double ct, double st) {
  // Phi = i G C * 2 * sum Bh I2  ->  2 Re Phi = -4 G C phi
  const double2 W = make_double2(-gc * a.psi.y, gc * a.psi.x);   // i G C psi
  const double2 e2 = make_double2(ct * ct - st * st, 2.0 * ct * st);
  const double2 T = cmul(e2, W);
  return make_double2(T.y, T.x - 4.0 * gc * a.phi);            // (sigma_s, sigma_n)
}

// One warp per work item (leaf k, group of nt <= kTgtGroup targets, interval
// of the leaf's concatenated source ranges).  Each lane owns kTPL targets
// (independent chains sharing every source load); the tp = ceil(nt/kTPL)
// lane-target slots are replicated over S = 32 / tp source slices: lane l
// takes slot l % tp and the sources j = l / tp (mod S).  Source records are
// read through L1 (the tp lanes of a slice broadcast one record).  The S slice
// partials are summed in a fixed order (deterministic results).
constexpr int kP2PWarps = 4;
#ifndef DDM_P2P_MINB
#define DDM_P2P_MINB 6
#endif
#ifndef DDM_TPL
#define DDM_TPL 2
#endif
constexpr int kTPL = DDM_TPL;   // targets per lane (independent chains sharing each source load)

__global__ void __launch_bounds__(kP2PWarps * 32, DDM_P2P_MINB)
p2p_kernel(int nown, const int* __restrict__ order, const int4* __restrict__ items,
           const int* __restrict__ u_off, const int* __restrict__ u_lo,
           const int* __restrict__ u_hi, const int* __restrict__ leaves,
           const int* __restrict__ c_start, const int* __restrict__ c_count,
           const double* __restrict__ src, const double* __restrict__ ex,
           const double* __restrict__ ey, const double* __restrict__ ec,
           const double* __restrict__ es, double gc, double2* __restrict__ part) {
  __shared__ double red[kP2PWarps][3][32 * kTPL];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int oi = blockIdx.x * kP2PWarps + w; oi < nown; oi += gridDim.x * kP2PWarps) {
    const int it = order[oi];
    const int4 item = items[it];
    const int k = item.x;
    const int c = leaves[k];
    const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
    const int tp = (nt + kTPL - 1) / kTPL;
    const int S = 32 / tp;
    const int tl = lane % tp, slice = lane / tp;
    const bool active = slice < S;
    double zx[kTPL], zy[kTPL];
    P2PAcc acc[kTPL];
#pragma unroll
    for (int q = 0; q < kTPL; ++q) {
      const int ti = item.y + min(tl * kTPL + q, nt - 1);
      zx[q] = ex[ti];
      zy[q] = ey[ti];
    }
    if (active) {
      int pos = 0;   // position in the concatenated range space
      for (int r = u_off[k], rend = u_off[k + 1]; r < rend && pos < item.w; ++r) {
        const int lo = u_lo[r], len = u_hi[r] - lo;
        const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
        const double* base = src + (int64_t)lo * kSrcStride;
#pragma unroll 2
        for (int j = b + slice; j < e; j += S) {
          double sp[kSrcStride];
          const double2* g = reinterpret_cast<const double2*>(base + (int64_t)j * kSrcStride);
#pragma unroll
          for (int f = 0; f < kSrcStride / 2; ++f) {
            const double2 v = __ldg(g + f);
            sp[2 * f] = v.x;
            sp[2 * f + 1] = v.y;
          }
#pragma unroll
          for (int q = 0; q < kTPL; ++q) pair_update(acc[q], zx[q], zy[q], sp);
        }
        pos += len;
      }
    }
    // slot of (target t, slice s) = t + s * tp * kTPL
#pragma unroll
    for (int q = 0; q < kTPL; ++q) {
      const int sl = tl * kTPL + q + slice * tp * kTPL;
      if (active) {
        red[w][0][sl] = acc[q].phi;
        red[w][1][sl] = acc[q].psi.x;
        red[w][2][sl] = acc[q].psi.y;
      }
    }
    __syncwarp();
    if (lane < kTgtGroup) {
      double2 T = make_double2(0.0, 0.0);
      if (lane < nt) {
        P2PAcc tot;
        for (int s2 = 0; s2 < S; ++s2) {
          const int sl = lane + s2 * tp * kTPL;
          tot.phi += red[w][0][sl];
          tot.psi.x += red[w][1][sl];
          tot.psi.y += red[w][2][sl];
        }
        const int ti = item.y + lane;
        T = acc_to_traction(tot, gc, ec[ti], es[ti]);
      }
      part[(int64_t)it * kTgtGroup + lane] = T;
    }
    __syncwarp();
  }
}

// All pairs (mode DDM_DIRECT): thread per target, sources tiled through smem.
constexpr int kDirThreads = 128;

__global__ void __launch_bounds__(kDirThreads)
direct_kernel(int64_t n, int64_t t_lo, int64_t t_hi, int ncomp, const double* __restrict__ src,
              const double* __restrict__ ex, const double* __restrict__ ey,
              const double* __restrict__ ec, const double* __restrict__ es, double gc,
              const int* __restrict__ perm, double* __restrict__ y_user,
              double* __restrict__ y_sorted) {
  __shared__ double ssrc[kDirThreads * kSrcStride];
  const int64_t ti = t_lo + blockIdx.x * (int64_t)kDirThreads + threadIdx.x;
  const bool tvalid = ti < t_hi;
  double zx = 0.0, zy = 0.0;
  if (tvalid) { zx = ex[ti]; zy = ey[ti]; }
  P2PAcc acc;
  for (int64_t j0 = 0; j0 < n; j0 += kDirThreads) {
    const int nb = (int)min((int64_t)kDirThreads, n - j0);
    __syncthreads();
    for (int f = threadIdx.x; f < nb * kSrcStride / 2; f += kDirThreads)
      reinterpret_cast<double2*>(ssrc)[f] =
          reinterpret_cast<const double2*>(src + j0 * kSrcStride)[f];
    __syncthreads();
    for (int j = 0; j < nb; ++j) pair_update(acc, zx, zy, ssrc + j * kSrcStride);
  }
  if (!tvalid) return;
  const double2 T = acc_to_traction(acc, gc, ec[ti], es[ti]);
  if (y_sorted) {
    y_sorted[ti * ncomp] = T.x;
    y_sorted[ti * ncomp + 1] = T.y;
  }
  if (y_user) {
    const int j = perm[ti];
    y_user[(int64_t)j * ncomp] = T.x;
    y_user[(int64_t)j * ncomp + 1] = T.y;
  }
}

}  // namespace

int launch_prep_sources(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D,
                        int ncomp, cudaStream_t s) {
  prep_sources<<<nblk(t->n, 256), 256, 0, s>>>(t->n, ncomp, perm_in, D, t->ex, t->ey, t->ea,
                                                 t->ec, t->es, t->src,
                                                 perm_in ? t->d_sorted : nullptr);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_p2p(ddm_ctx_s* ctx, ddm_tree_s* t, int item_lo, int item_hi, double gc,
               cudaStream_t s) {
  if (item_hi <= item_lo) return DDM_OK;
  // short-lived blocks (4 items each): slots free up continuously, so the
  // high-priority far-field kernels interleave with the near field
  const unsigned nb = nblk(item_hi - item_lo, kP2PWarps);
  p2p_kernel<<<nb, kP2PWarps * 32, 0, s>>>(item_hi - item_lo, t->p2p_order, t->items, t->u_off,
                                           t->u_lo,
                                           t->u_hi, t->leaves, t->c_start, t->c_count, t->src,
                                           t->ex, t->ey, t->ec, t->es, gc, t->part);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_direct(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, int ncomp, double gc,
                  double* y_user, double* y_sorted, cudaStream_t s) {
  if (hi <= lo) return DDM_OK;
  direct_kernel<<<nblk(hi - lo, kDirThreads), kDirThreads, 0, s>>>(
      t->n, lo, hi, ncomp, t->src, t->ex, t->ey, t->ec, t->es, gc, t->perm, y_user, y_sorted);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

namespace {
// Self blocks of the elastic influence (block-Jacobi preconditioner of
// GMRES): blk[i][r][c] = traction component r (s, n) at element i's centre
// from a unit DD component c (s, n) on element i (sorted order).
__global__ void elastic_self_blocks(int64_t n, const double* __restrict__ ex,
                                    const double* __restrict__ ey, const double* __restrict__ ea,
                                    const double* __restrict__ ec, const double* __restrict__ es,
                                    double gc, double* __restrict__ blk) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double c = ec[i], s = es[i], a = ea[i];
  const double2 r = make_double2(c * c - s * s, -2.0 * c * s);
  for (int col = 0; col < 2; ++col) {
    const double ds = col == 0 ? 1.0 : 0.0, dn = col == 1 ? 1.0 : 0.0;
    const double2 B = make_double2(ds * c - dn * s, ds * s + dn * c);
    const double2 rB = cmul(r, B);
    const double2 Bh = make_double2(0.5 * B.x, 0.5 * B.y);
    const double2 P1 = cmul(Bh, make_double2(r.x - 1.0, r.y));
    const double2 T2 = cmul(Bh, make_double2(r.x + 1.0, r.y));
    double sp[kSrcStride] = {ex[i] - a * c, ey[i] - a * s, ex[i] + a * c, ey[i] + a * s,
                             P1.x, P1.y, -T2.y, T2.x, Bh.x, Bh.y, -(rB.x + B.x), -(rB.y - B.y)};
    P2PAcc acc;
    pair_update(acc, ex[i], ey[i], sp);
    const double2 T = acc_to_traction(acc, gc, c, s);
    blk[i * 4 + 0 * 2 + col] = T.x;
    blk[i * 4 + 1 * 2 + col] = T.y;
  }
}
// dense diagonal blocks of the leaf-block Jacobi preconditioner (gmres.cu):
// CTA per chunk; entry (2 i + r, 2 j + c) = traction component r at element
// e0+i from a unit DD component c on element e0+j (the exact pair kernel)
__global__ void elastic_chunk_blocks(const int2* __restrict__ chunks,
                                     const int64_t* __restrict__ off, const double* __restrict__ ex,
                                     const double* __restrict__ ey, const double* __restrict__ ea,
                                     const double* __restrict__ ec, const double* __restrict__ es,
                                     double gc, double* __restrict__ blk) {
  const int2 ch = chunks[blockIdx.x];
  const int e0 = ch.x, ne = ch.y, d = 2 * ne;
  double* Bk = blk + off[blockIdx.x];
  for (int idx = threadIdx.x; idx < ne * ne * 2; idx += blockDim.x) {
    const int col = idx % 2, pr = idx / 2, i = e0 + pr / ne, j = e0 + pr % ne;
    const double c = ec[j], s = es[j], a = ea[j];
    const double2 r = make_double2(c * c - s * s, -2.0 * c * s);
    const double ds = col == 0 ? 1.0 : 0.0, dn = col == 1 ? 1.0 : 0.0;
    const double2 B = make_double2(ds * c - dn * s, ds * s + dn * c);
    const double2 rB = cmul(r, B);
    const double2 Bh = make_double2(0.5 * B.x, 0.5 * B.y);
    const double2 P1 = cmul(Bh, make_double2(r.x - 1.0, r.y));
    const double2 T2 = cmul(Bh, make_double2(r.x + 1.0, r.y));
    const double sp[kSrcStride] = {ex[j] - a * c, ey[j] - a * s, ex[j] + a * c, ey[j] + a * s,
                                   P1.x, P1.y, -T2.y, T2.x, Bh.x, Bh.y, -(rB.x + B.x),
                                   -(rB.y - B.y)};
    P2PAcc acc;
    pair_update(acc, ex[i], ey[i], sp);
    const double2 T = acc_to_traction(acc, gc, ec[i], es[i]);
    const int r0 = 2 * (i - e0), c0 = 2 * (j - e0) + col;
    Bk[(size_t)r0 * d + c0] = T.x;
    Bk[(size_t)(r0 + 1) * d + c0] = T.y;
  }
}
}  // namespace

int launch_elastic_chunk_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, double gc, int nchunks,
                                const int2* chunks, const int64_t* off, double* blk,
                                cudaStream_t s) {
  if (nchunks <= 0) return DDM_OK;
  elastic_chunk_blocks<<<nchunks, 128, 0, s>>>(chunks, off, t->ex, t->ey, t->ea, t->ec, t->es,
                                               gc, blk);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_elastic_self_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, double gc, double* blk,
                               cudaStream_t s) {
  elastic_self_blocks<<<nblk(t->n, 128), 128, 0, s>>>(t->n, t->ex, t->ey, t->ea, t->ec, t->es,
                                                      gc, blk);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

}  // namespace ddm
