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
//   e = e^{i beta}, B = (D_s + i D_n) e, r = conj(e)^2, Q' = Q - 2 B r = -(r B + conj B)
//   src = {z1, z2, r, B/2, Q'}  (10 doubles)
__global__ void prep_sources(int64_t n, int ncomp, const int* __restrict__ perm,
                             const double* __restrict__ D, const double* __restrict__ ex,
                             const double* __restrict__ ey, const double* __restrict__ ea,
                             const double* __restrict__ ec, const double* __restrict__ es,
                             double* __restrict__ src) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm ? perm[i] : (int)i;
  const double ds = D[(int64_t)j * ncomp + 0];
  const double dn = D[(int64_t)j * ncomp + 1];
  const double c = ec[i], s = es[i], a = ea[i];
  const double2 B = make_double2(ds * c - dn * s, ds * s + dn * c);
  const double2 r = make_double2(c * c - s * s, -2.0 * c * s);
  const double2 rB = cmul(r, B);
  const double2 Qp = make_double2(-(rB.x + B.x), -(rB.y - B.y));
  double2* o = reinterpret_cast<double2*>(src + i * 10);
  o[0] = make_double2(ex[i] - a * c, ey[i] - a * s);
  o[1] = make_double2(ex[i] + a * c, ey[i] + a * s);
  o[2] = r;
  o[3] = make_double2(0.5 * B.x, 0.5 * B.y);
  o[4] = Qp;
}

// Contribution of source element (z1, z2, r, Bh, Q') to the target at z:
//   r1 = 1/(z - z1), r2 = 1/(z - z2), I2 = r2 - r1, I3 = I2 (r1 + r2)/2
//   Phi           += i G C B I2                 -> phi += Im(Bh I2)
//   zb Phi' + Psi += i G C I2 [Q' + B (r D - conj D)(r1 + r2)/2],  D = z - zc
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
  const double2 r1 = make_double2(w1x * i1, -w1y * i1);
  const double2 r2 = make_double2(w2x * i2, -w2y * i2);
  const double2 I2 = csub(r2, r1);
  const double2 S = cadd(r1, r2);
  const double dx = w1x + w2x, dy = w1y + w2y;   // 2 (z - zc)
  // X = r * D2 - conj(D2)
  const double2 X = make_double2(fma(sp[4], dx, fma(-sp[5], dy, -dx)),
                                 fma(sp[4], dy, fma(sp[5], dx, dy)));
  const double2 BX = cmul(make_double2(sp[6], sp[7]), X);   // (B/2) X = B (r D - conj D)
  double2 V = make_double2(sp[8], sp[9]);
  cmac(V, BX, S);
  cmac(acc.psi, I2, V);
  acc.phi = fma(sp[6], I2.y, fma(sp[7], I2.x, acc.phi));
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
// of the leaf's concatenated source ranges).  The 32 lanes are split into
// S = 32 / nt source slices: lane l evaluates target l % nt against the
// sources j = l / nt (mod S) of each 32-source batch staged in shared memory;
// the S slice partials are summed in a fixed order (deterministic).
constexpr int kP2PWarps = 4;
#ifndef DDM_P2P_MINB
#define DDM_P2P_MINB 8   // >= 8 resident blocks per SM (measured best: 1.18 -> 1.06 ms)
#endif

__global__ void __launch_bounds__(kP2PWarps * 32, DDM_P2P_MINB)
p2p_kernel(int item_lo, int item_hi, const int4* __restrict__ items,
           const int* __restrict__ u_off, const int* __restrict__ u_lo,
           const int* __restrict__ u_hi, const int* __restrict__ leaves,
           const int* __restrict__ c_start, const int* __restrict__ c_count,
           const double* __restrict__ src, const double* __restrict__ ex,
           const double* __restrict__ ey, const double* __restrict__ ec,
           const double* __restrict__ es, double gc, double2* __restrict__ part) {
  __shared__ double sh[kP2PWarps][32 * 10];
  __shared__ double red[kP2PWarps][3][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ssrc = sh[w];
  for (int it = item_lo + blockIdx.x * kP2PWarps + w; it < item_hi;
       it += gridDim.x * kP2PWarps) {
    const int4 item = items[it];
    const int k = item.x;
    const int c = leaves[k];
    const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
    const int S = 32 / nt;
    const int tl = lane % nt, slice = lane / nt;
    const bool active = slice < S;
    const int ti = item.y + tl;
    const double zx = ex[ti], zy = ey[ti];
    P2PAcc acc;
    // cursor into the leaf's concatenated source ranges
    int r = u_off[k];
    const int rend = u_off[k + 1];
    int roff = item.z;
    while (r < rend && roff >= u_hi[r] - u_lo[r]) { roff -= u_hi[r] - u_lo[r]; ++r; }
    for (int t = item.z; t < item.w; t += 32) {
      const int nb = min(32, item.w - t);
      if (lane < nb) {
        int rr = r, q = roff + lane;
        while (q >= u_hi[rr] - u_lo[rr]) { q -= u_hi[rr] - u_lo[rr]; ++rr; }
        const double2* g = reinterpret_cast<const double2*>(src + (int64_t)(u_lo[rr] + q) * 10);
        double2* d = reinterpret_cast<double2*>(ssrc + lane * 10);
#pragma unroll
        for (int f = 0; f < 5; ++f) d[f] = g[f];
      }
      __syncwarp();
      if (active) {
#pragma unroll 4
        for (int j = slice; j < nb; j += S) pair_update(acc, zx, zy, ssrc + j * 10);
      }
      __syncwarp();
      roff += nb;
      while (r < rend && roff >= u_hi[r] - u_lo[r]) { roff -= u_hi[r] - u_lo[r]; ++r; }
    }
    red[w][0][lane] = acc.phi;
    red[w][1][lane] = acc.psi.x;
    red[w][2][lane] = acc.psi.y;
    __syncwarp();
    if (lane < kTgtGroup) {
      double2 T = make_double2(0.0, 0.0);
      if (lane < nt) {
        P2PAcc tot;
        for (int s2 = 0; s2 < S; ++s2) {
          tot.phi += red[w][0][lane + s2 * nt];
          tot.psi.x += red[w][1][lane + s2 * nt];
          tot.psi.y += red[w][2][lane + s2 * nt];
        }
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
  __shared__ double ssrc[kDirThreads * 10];
  const int64_t ti = t_lo + blockIdx.x * (int64_t)kDirThreads + threadIdx.x;
  const bool tvalid = ti < t_hi;
  double zx = 0.0, zy = 0.0;
  if (tvalid) { zx = ex[ti]; zy = ey[ti]; }
  P2PAcc acc;
  for (int64_t j0 = 0; j0 < n; j0 += kDirThreads) {
    const int nb = (int)min((int64_t)kDirThreads, n - j0);
    __syncthreads();
    for (int f = threadIdx.x; f < nb * 5; f += kDirThreads)
      reinterpret_cast<double2*>(ssrc)[f] = reinterpret_cast<const double2*>(src + j0 * 10)[f];
    __syncthreads();
    for (int j = 0; j < nb; ++j) pair_update(acc, zx, zy, ssrc + j * 10);
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
                                                 t->ec, t->es, t->src);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_p2p(ddm_ctx_s* ctx, ddm_tree_s* t, int item_lo, int item_hi, double gc,
               cudaStream_t s) {
  if (item_hi <= item_lo) return DDM_OK;
  // short-lived blocks (4 items each): slots free up continuously, so the
  // high-priority far-field kernels interleave with the near field
  const unsigned nb = nblk(item_hi - item_lo, kP2PWarps);
  p2p_kernel<<<nb, kP2PWarps * 32, 0, s>>>(item_lo, item_hi, t->items, t->u_off, t->u_lo,
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

}  // namespace ddm
