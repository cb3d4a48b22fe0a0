// FMM matvec for the elastic constant-DD kernel.
//
// PAPER.md §3.2: upward pass (P2M "P2L" Eq.(p2l), M2M Eq.(m2m)),
// downward pass (M2L over interaction lists Eq.(m2l), L2L Eq.(l2l)), final
// L2P + P2P for self and neighbour cells.  The paper's Chebyshev
// interpolation (bbFMM) is replaced by complex-variable (Kolosov–Muskhelishvili)
// expansions of the constant-element influence: every cell
// carries two Laurent / Taylor series, Phi and Psi~ = Psi + conj(z_c) Phi'.
//
// Normalised storage (cell side s, centre z0):
//   multipole  Phi(z) = sum_{n=1..p} a_n ((z - z0)/s)^(-n)      (slot n-1)
//   local      Phi(z) = sum_{m=0..p-1} l_m ((z - z0)/s)^m       (slot m)
// and likewise for Psi~.  The factor i G C, C = 1/(4 pi (1 - nu)), is applied
// once, at evaluation.
#include <cmath>
#include <vector>

#include "ddm_internal.cuh"

namespace ddm {
namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc += a * b
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// 1/x for x > 0 normal: MUFU.RCP64H seed + cubic Newton refinement (error ~e^3)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

struct CellGeom {
  double x_min, y_min, W;
  __device__ __forceinline__ double side(int lev) const { return ldexp(W, -lev); }
  __device__ __forceinline__ double2 centre(int lev, int ix, int iy) const {
    const double s = ldexp(W, -lev);
    return make_double2(x_min + (ix + 0.5) * s, y_min + (iy + 0.5) * s);
  }
};

// ------------------------------------------------------------ source prep
// Per element (sorted order), from the DDs (D_s, D_n) and geometry:
//   e = e^{i beta}, B = (D_s + i D_n) e, r = conj(e)^2, Q' = Q - 2 B r = -(r B + conj B)
//   src = {z1, z2, r, B/2, Q'}  (10 doubles)     [P2P]
__global__ void prep_sources(int64_t n, int ncomp, const int* __restrict__ perm,
                             const double* __restrict__ D, const double* __restrict__ ex,
                             const double* __restrict__ ey, const double* __restrict__ ea,
                             const double* __restrict__ ec, const double* __restrict__ es,
                             double* __restrict__ src, double* __restrict__ d_sorted) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm ? perm[i] : (int)i;
  const double ds = D[(int64_t)j * ncomp + 0];
  const double dn = D[(int64_t)j * ncomp + 1];
  if (d_sorted) {
    d_sorted[i * ncomp + 0] = ds;
    d_sorted[i * ncomp + 1] = dn;
  }
  const double c = ec[i], s = es[i], a = ea[i];
  const double2 B = make_double2(ds * c - dn * s, ds * s + dn * c);
  const double2 r = make_double2(c * c - s * s, -2.0 * c * s);
  const double2 rB = cmul(r, B);
  const double2 Qp = make_double2(-(rB.x + B.x), -(rB.y - B.y));
  double* o = src + i * 10;
  o[0] = ex[i] - a * c;
  o[1] = ey[i] - a * s;
  o[2] = ex[i] + a * c;
  o[3] = ey[i] + a * s;
  o[4] = r.x;
  o[5] = r.y;
  o[6] = 0.5 * B.x;
  o[7] = 0.5 * B.y;
  o[8] = Qp.x;
  o[9] = Qp.y;
}

// ------------------------------------------------------------ pair kernel
// Contribution of source element (z1, z2, r, Bh, Q') to the target at z
// (App. A.2 of SURVEY.md):
//   r1 = 1/(z - z1), r2 = 1/(z - z2), I2 = r2 - r1, I3 = I2 (r1 + r2)/2
//   Phi       += i G C B I2                 -> accPhi += Im(Bh I2)
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

// traction (sigma_s, sigma_n) from the accumulators at a target with
// direction (ct, st):  T = sigma_n + i sigma_s = 2 Re Phi + e^{2 i bt} (zb Phi' + Psi)
__device__ __forceinline__ double2 acc_to_traction(const P2PAcc& a, double gc, double ct, double st) {
  // Phi = i G C * 2 * sum Bh I2  ->  2 Re Phi = -4 G C accPhi
  const double2 W = make_double2(-gc * a.psi.y, gc * a.psi.x);   // i G C psi
  const double2 e2 = make_double2(ct * ct - st * st, 2.0 * ct * st);
  const double2 T = cmul(e2, W);
  return make_double2(T.y, T.x - 4.0 * gc * a.phi);            // (sigma_s, sigma_n)
}

// ------------------------------------------------------------ P2P (near field)
constexpr int kP2PWarps = 4;

__global__ void __launch_bounds__(kP2PWarps * 32)
p2p_kernel(int item_lo, int item_hi, const int4* __restrict__ items,
           const int* __restrict__ u_off, const int* __restrict__ u_lo,
           const int* __restrict__ u_hi, const int* __restrict__ leaves,
           const int* __restrict__ c_start, const int* __restrict__ c_count,
           const double* __restrict__ src, const double* __restrict__ ex,
           const double* __restrict__ ey, const double* __restrict__ ec,
           const double* __restrict__ es, double gc, double2* __restrict__ part) {
  __shared__ double sh[kP2PWarps][32 * 10];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ssrc = sh[w];
  for (int it = item_lo + blockIdx.x * kP2PWarps + w; it < item_hi;
       it += gridDim.x * kP2PWarps) {
    const int4 item = items[it];
    const int k = item.x;
    const int c = leaves[k];
    const int tend = c_start[c] + c_count[c];
    const int ti = item.y + lane;
    const bool tvalid = ti < tend;
    double zx = 0.0, zy = 0.0;
    if (tvalid) { zx = ex[ti]; zy = ey[ti]; }
    P2PAcc acc;
    // cursor into the leaf's concatenated source ranges
    int r = u_off[k];
    const int rend = u_off[k + 1];
    int roff = item.z;
    while (r < rend && roff >= u_hi[r] - u_lo[r]) { roff -= u_hi[r] - u_lo[r]; ++r; }
    for (int t = item.z; t < item.w; t += 32) {
      const int nb = min(32, item.w - t);
      // lane-local source of this batch
      if (lane < nb) {
        int rr = r, q = roff + lane;
        while (q >= u_hi[rr] - u_lo[rr]) { q -= u_hi[rr] - u_lo[rr]; ++rr; }
        const double2* g = reinterpret_cast<const double2*>(src + (int64_t)(u_lo[rr] + q) * 10);
        double2* d = reinterpret_cast<double2*>(ssrc + lane * 10);
#pragma unroll
        for (int f = 0; f < 5; ++f) d[f] = g[f];
      }
      __syncwarp();
      for (int j = 0; j < nb; ++j) pair_update(acc, zx, zy, ssrc + j * 10);
      __syncwarp();
      roff += nb;
      while (r < rend && roff >= u_hi[r] - u_lo[r]) { roff -= u_hi[r] - u_lo[r]; ++r; }
    }
    double2 T = make_double2(0.0, 0.0);
    if (tvalid) T = acc_to_traction(acc, gc, ec[ti], es[ti]);
    part[(int64_t)it * 32 + lane] = T;
  }
}

// ------------------------------------------------------------ direct (all pairs)
constexpr int kDirThreads = 128;

__global__ void __launch_bounds__(kDirThreads)
direct_kernel(int64_t n, int64_t t_lo, int64_t t_hi, const double* __restrict__ src,
              const double* __restrict__ ex, const double* __restrict__ ey,
              const double* __restrict__ ec, const double* __restrict__ es, double gc,
              double2* __restrict__ out) {
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
  if (tvalid) out[ti] = acc_to_traction(acc, gc, ec[ti], es[ti]);
}

// ------------------------------------------------------------ P2M (a5)
// warp per leaf; lane = element of the round, then lane = coefficient.
// alpha_n = (B/s) P_{n-1};  gamma_n = (1/s)[Q P_{n-1} + B((n-1) A P_{n-2} + (n-2) r P_{n-1})]
// with zeta_{1,2} = (z_{1,2} - z0)/s, P_m = zeta2^m - zeta1^m,
// A = conj(zc - z0)/s - r (zc - z0)/s.
constexpr int kP2MWarps = 4;

__global__ void __launch_bounds__(kP2MWarps * 32)
p2m_kernel(int nleaves, const int* __restrict__ leaves, const int* __restrict__ c_level,
           const int* __restrict__ c_ix, const int* __restrict__ c_iy,
           const int* __restrict__ c_start, const int* __restrict__ c_count, CellGeom cg,
           int p, const int* __restrict__ perm, const double* __restrict__ D, int ncomp,
           const double* __restrict__ ex, const double* __restrict__ ey,
           const double* __restrict__ ea, const double* __restrict__ ec,
           const double* __restrict__ es, double2* __restrict__ mpole) {
  extern __shared__ double2 p2m_sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int stride = (p + 1) | 1;                 // odd row stride in double2 units
  double2* buf = p2m_sh + (size_t)w * 32 * stride * 2;   // [32][stride] x {alpha, gamma}
  for (int k = blockIdx.x * kP2MWarps + w; k < nleaves; k += gridDim.x * kP2MWarps) {
    const int c = leaves[k];
    const int lev = c_level[c];
    const double s = cg.side(lev);
    const double is = 1.0 / s;
    const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
    const int e0 = c_start[c], ne = c_count[c];
    double2 acc_a[2], acc_g[2];
    acc_a[0] = acc_a[1] = acc_g[0] = acc_g[1] = make_double2(0.0, 0.0);
    for (int r0 = 0; r0 < ne; r0 += 32) {
      const int i = e0 + r0 + lane;
      const bool valid = r0 + lane < ne;
      double2 B = make_double2(0, 0), Q = B, rr = B, A = B, z1 = B, z2 = B;
      if (valid) {
        const int j = perm ? perm[i] : i;
        const double ds = D[(int64_t)j * ncomp], dn = D[(int64_t)j * ncomp + 1];
        const double cb = ec[i], sb = es[i], a = ea[i];
        B = make_double2(ds * cb - dn * sb, ds * sb + dn * cb);
        rr = make_double2(cb * cb - sb * sb, -2.0 * cb * sb);
        Q = csub(cmul(rr, B), cconj(B));
        const double2 d = make_double2((ex[i] - z0.x) * is, (ey[i] - z0.y) * is);
        A = csub(cconj(d), cmul(rr, d));
        z1 = make_double2(d.x - a * cb * is, d.y - a * sb * is);
        z2 = make_double2(d.x + a * cb * is, d.y + a * sb * is);
        B = cscale(B, is);
        Q = cscale(Q, is);
      }
      // powers: pw = zeta^m, P_m = pw2 - pw1 ; start m = 0 (P_0 = 0)
      double2 pw1 = make_double2(1.0, 0.0), pw2 = pw1;
      double2 Pm1 = make_double2(0.0, 0.0);   // P_{n-2}
      double2 Pm = make_double2(0.0, 0.0);    // P_{n-1}
      for (int n = 1; n <= p; ++n) {
        // P_{n-1}: for n = 1 it is P_0 = 0; then advance powers
        if (n >= 2) {
          pw1 = cmul(pw1, z1);
          pw2 = cmul(pw2, z2);
          Pm1 = Pm;
          Pm = csub(pw2, pw1);
        }
        const double2 alpha = cmul(B, Pm);
        double2 gam = cmul(Q, Pm);
        double2 t = cscale(cmul(A, Pm1), (double)(n - 1));
        cmac(t, cscale(rr, (double)(n - 2)), Pm);
        cmac(gam, B, t);
        buf[lane * stride * 2 + (n - 1)] = alpha;
        buf[lane * stride * 2 + stride + (n - 1)] = gam;
      }
      __syncwarp();
      // lane = coefficient index: sum the rows in element order
      for (int cc = 0; cc < 2; ++cc) {
        const int n = lane + 32 * cc;
        if (n < p) {
          double2 sa = acc_a[cc], sg = acc_g[cc];
          const int rows = min(32, ne - r0);
          for (int e = 0; e < rows; ++e) {
            sa = cadd(sa, buf[e * stride * 2 + n]);
            sg = cadd(sg, buf[e * stride * 2 + stride + n]);
          }
          acc_a[cc] = sa;
          acc_g[cc] = sg;
        }
      }
      __syncwarp();
    }
    double2* out = mpole + (size_t)c * 2 * p;
    for (int cc = 0; cc < 2; ++cc) {
      const int n = lane + 32 * cc;
      if (n < p) {
        out[n] = acc_a[cc];
        out[p + n] = acc_g[cc];
      }
    }
  }
}

// ------------------------------------------------------------ M2M (a6)
// parent P at level lev (non-leaf): sum over children q of
//   alpha^P_m = sum_n MT_q[n][m] alpha^q_n,  gamma^P_m = sum_n MT_q[n][m] c^q_n,
//   c_n = gamma_n - (n-1) conj(e)/s_c alpha_{n-1},  e = z_P - z_q.
constexpr int kM2MWarps = 4;

__global__ void __launch_bounds__(kM2MWarps * 32)
m2m_kernel(int c0, int c1, const int* __restrict__ c_leaf, const int* __restrict__ c_ix,
           const int* __restrict__ c_iy, const int* __restrict__ first_child,
           const int* __restrict__ nchild, int p, const double2* __restrict__ opT,
           double2* __restrict__ mpole) {
  __shared__ double2 sh[kM2MWarps][2 * (kMaxP + 1)];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sa = sh[w];
  double2* scv = sh[w] + (kMaxP + 1);
  for (int c = c0 + blockIdx.x * kM2MWarps + w; c < c1; c += gridDim.x * kM2MWarps) {
    if (c_leaf[c]) continue;
    double2 acc_a[2], acc_g[2];
    acc_a[0] = acc_a[1] = acc_g[0] = acc_g[1] = make_double2(0.0, 0.0);
    const int f = first_child[c], nc = nchild[c];
    for (int q = f; q < f + nc; ++q) {
      const int quad = (c_ix[q] & 1) + 2 * (c_iy[q] & 1);
      // conj(e)/s_c with e = z_P - z_q = -((xb-1/2) + i (yb-1/2)) s_c
      const double2 eb = make_double2(-((c_ix[q] & 1) - 0.5), ((c_iy[q] & 1) - 0.5));
      const double2* mq = mpole + (size_t)q * 2 * p;
      for (int n = lane; n < p; n += 32) sa[n] = mq[n];
      __syncwarp();
      for (int n = lane; n < p; n += 32) {
        double2 cv = mq[p + n];
        if (n >= 1) cmac(cv, cscale(eb, -(double)n), sa[n - 1]);
        scv[n] = cv;
      }
      __syncwarp();
      const double2* M = opT + (size_t)quad * p * p;
      for (int cc = 0; cc < 2; ++cc) {
        const int m = lane + 32 * cc;
        if (m < p) {
          double2 a = acc_a[cc], g = acc_g[cc];
          for (int n = 0; n <= m; ++n) {
            const double2 t = M[(size_t)n * p + m];
            cmac(a, t, sa[n]);
            cmac(g, t, scv[n]);
          }
          acc_a[cc] = a;
          acc_g[cc] = g;
        }
      }
      __syncwarp();
    }
    double2* out = mpole + (size_t)c * 2 * p;
    for (int cc = 0; cc < 2; ++cc) {
      const int m = lane + 32 * cc;
      if (m < p) {
        out[m] = acc_a[cc];
        out[p + m] = acc_g[cc];
      }
    }
  }
}

// ------------------------------------------------------------ M2L (a7)
// target cell b, sources a in V(b):  with delta = (z_b - z_a)/s,
// h_k = (k-1)! delta^-k (table per offset class),
//   l_m = (-1)^m/m! sum_{n=1..p} [alpha_n/(n-1)!] h_{n+m}
//   g_m = (-1)^m/m! sum_{n=1..p+1} [c_n/(n-1)!] h_{n+m},  c_n = gamma_n - (n-1) conj(delta) alpha_{n-1}
constexpr int kM2LWarps = 8;

__global__ void __launch_bounds__(kM2LWarps * 32)
m2l_kernel(int c0, int c1, const int* __restrict__ v_off, const int* __restrict__ v_idx,
           const unsigned char* __restrict__ v_cls, int p, const double2* __restrict__ htab,
           const double* __restrict__ invfact, const double2* __restrict__ mpole,
           double2* __restrict__ local) {
  extern __shared__ double2 m2l_sh[];
  const int hs = 2 * p + 2;                          // entries per class
  double2* sh_h = m2l_sh;                            // [49][hs]
  double2* wbuf = m2l_sh + kNOffsets * hs;           // per warp [2][p+2]
  for (int f = threadIdx.x; f < kNOffsets * hs; f += blockDim.x) sh_h[f] = htab[f];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sa = wbuf + (size_t)w * 2 * (p + 2);
  double2* scv = sa + (p + 2);
  for (int c = c0 + blockIdx.x * kM2LWarps + w; c < c1; c += gridDim.x * kM2LWarps) {
    double2 al[2], ag[2];
    al[0] = al[1] = ag[0] = ag[1] = make_double2(0.0, 0.0);
    const int vb = v_off[c], ve = v_off[c + 1];
    for (int v = vb; v < ve; ++v) {
      const int a = v_idx[v];
      const int cls = v_cls[v];
      const int dxs = cls % 7 - 3, dys = cls / 7 - 3;   // source - target in cells
      const double2 dconj = make_double2(-(double)dxs, (double)dys);  // conj(delta), delta = -(dx + i dy)
      const double2* ma = mpole + (size_t)a * 2 * p;
      for (int n = lane; n < p; n += 32) sa[n] = ma[n];
      __syncwarp();
      for (int n = lane; n <= p; n += 32) {   // slot n <-> c_{n+1}
        double2 cv = (n < p) ? ma[p + n] : make_double2(0.0, 0.0);
        if (n >= 1) cmac(cv, cscale(dconj, -(double)n), sa[n - 1]);
        scv[n] = cscale(cv, invfact[n]);
      }
      __syncwarp();
      for (int n = lane; n < p; n += 32) sa[n] = cscale(sa[n], invfact[n]);
      __syncwarp();
      const double2* h = sh_h + cls * hs;
      for (int cc = 0; cc < 2; ++cc) {
        const int m = lane + 32 * cc;
        if (m < p) {
          double2 l = al[cc], g = ag[cc];
          // h index k = n + m with n = slot + 1
          for (int n = 0; n < p; ++n) {
            const double2 hk = h[n + 1 + m];
            cmac(l, sa[n], hk);
            cmac(g, scv[n], hk);
          }
          cmac(g, scv[p], h[p + 1 + m]);
          al[cc] = l;
          ag[cc] = g;
        }
      }
      __syncwarp();
    }
    double2* out = local + (size_t)c * 2 * p;
    for (int cc = 0; cc < 2; ++cc) {
      const int m = lane + 32 * cc;
      if (m < p) {
        const double sc = ((m & 1) ? -1.0 : 1.0) * invfact[m];
        out[m] = cscale(al[cc], sc);
        out[p + m] = cscale(ag[cc], sc);
      }
    }
  }
}

// ------------------------------------------------------------ L2L (a8)
// child c += shift of parent P:  g_k = gamma_k + (k+1) conj(eps) lambda_{k+1},
//   lambda^c_k += sum_m LT_q[m][k] lambda^P_m,  gamma^c_k += sum_m LT_q[m][k] g_m
constexpr int kL2LWarps = 4;

__global__ void __launch_bounds__(kL2LWarps * 32)
l2l_kernel(int c0, int c1, const int* __restrict__ c_parent, const int* __restrict__ c_ix,
           const int* __restrict__ c_iy, int p, const double2* __restrict__ opT,
           double2* __restrict__ local) {
  __shared__ double2 sh[kL2LWarps][2 * (kMaxP + 1)];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sl = sh[w];
  double2* sg = sh[w] + (kMaxP + 1);
  for (int c = c0 + blockIdx.x * kL2LWarps + w; c < c1; c += gridDim.x * kL2LWarps) {
    const int P = c_parent[c];
    const int xb = c_ix[c] & 1, yb = c_iy[c] & 1;
    const int quad = xb + 2 * yb;
    const double2 epsb = make_double2(0.5 * (xb - 0.5), -0.5 * (yb - 0.5));  // conj(eps)
    const double2* lp = local + (size_t)P * 2 * p;
    for (int m = lane; m < p; m += 32) sl[m] = lp[m];
    __syncwarp();
    for (int m = lane; m < p; m += 32) {
      double2 g = lp[p + m];
      if (m + 1 < p) cmac(g, cscale(epsb, (double)(m + 1)), sl[m + 1]);
      sg[m] = g;
    }
    __syncwarp();
    const double2* L = opT + (size_t)quad * p * p;
    double2* out = local + (size_t)c * 2 * p;
    for (int k = lane; k < p; k += 32) {
      double2 l = out[k], g = out[p + k];
      for (int m = k; m < p; ++m) {
        const double2 t = L[(size_t)m * p + k];
        cmac(l, t, sl[m]);
        cmac(g, t, sg[m]);
      }
      out[k] = l;
      out[p + k] = g;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ L2P + finalize (a9, a11)
// per owned sorted element: sum P2P partials in item order, add the far field
// from the leaf's local expansion, write (sigma_s, sigma_n).
__global__ void finalize_kernel(int64_t e_lo, int64_t e_hi, int ncomp,
                                const int* __restrict__ el_leaf, const int* __restrict__ leaves,
                                const int* __restrict__ c_level, const int* __restrict__ c_ix,
                                const int* __restrict__ c_iy, const int* __restrict__ c_start,
                                const int* __restrict__ c_count,
                                const int* __restrict__ item_off, const double2* __restrict__ part,
                                const double2* __restrict__ local, CellGeom cg, int p, double gc,
                                const double* __restrict__ ex, const double* __restrict__ ey,
                                const double* __restrict__ ec, const double* __restrict__ es,
                                const int* __restrict__ perm, double* __restrict__ y_user,
                                double* __restrict__ y_sorted) {
  const int64_t i = e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= e_hi) return;
  const int k = el_leaf[i];
  const int c = leaves[k];
  const int slot = (int)(i - c_start[c]);
  const int ngroups = (c_count[c] + kTgtGroup - 1) / kTgtGroup;
  const int i0 = item_off[k];
  const int nch = (item_off[k + 1] - i0) / ngroups;
  const int g = slot / kTgtGroup, ln = slot % kTgtGroup;
  double2 T = make_double2(0.0, 0.0);
  for (int h = 0; h < nch; ++h) T = cadd(T, part[(int64_t)(i0 + g * nch + h) * 32 + ln]);
  const int lev = c_level[c];
  if (lev >= 2) {
    const double s = cg.side(lev);
    const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
    const double2 u = make_double2((ex[i] - z0.x) / s, (ey[i] - z0.y) / s);
    const double2* L = local + (size_t)c * 2 * p;
    double2 phi = make_double2(0, 0), dphi = phi, psi = phi;
    for (int m = p - 1; m >= 0; --m) {
      if (m >= 1) dphi = cadd(cmul(dphi, u), cscale(L[m], (double)m));
      phi = cadd(cmul(phi, u), L[m]);
      psi = cadd(cmul(psi, u), L[p + m]);
    }
    // W = i G C (conj(u) dPhi + Psi~), T += 2 Re(i G C Phi) + e^{2 i b} W
    const double2 wv = cadd(cmul(cconj(u), dphi), psi);
    const double2 W = make_double2(-gc * wv.y, gc * wv.x);
    const double ct = ec[i], st = es[i];
    const double2 e2 = make_double2(ct * ct - st * st, 2.0 * ct * st);
    const double2 t = cmul(e2, W);
    T.x += t.y;
    T.y += t.x - 2.0 * gc * phi.y;
  }
  if (y_sorted) {
    y_sorted[i * ncomp + 0] = T.x;
    y_sorted[i * ncomp + 1] = T.y;
  }
  if (y_user) {
    const int j = perm[i];
    y_user[(int64_t)j * ncomp + 0] = T.x;
    y_user[(int64_t)j * ncomp + 1] = T.y;
  }
}

__global__ void scatter_direct(int64_t lo, int64_t hi, int ncomp, const double2* __restrict__ T,
                               const int* __restrict__ perm, double* __restrict__ y_user,
                               double* __restrict__ y_sorted) {
  const int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const double2 v = T[i];
  if (y_sorted) {
    y_sorted[i * ncomp] = v.x;
    y_sorted[i * ncomp + 1] = v.y;
  }
  if (y_user) {
    const int j = perm[i];
    y_user[(int64_t)j * ncomp] = v.x;
    y_user[(int64_t)j * ncomp + 1] = v.y;
  }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

double binom(int n, int k) {
  if (k < 0 || k > n) return 0.0;
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

int ensure_workspace(ddm_ctx_s* ctx, ddm_tree_s* t) {
  int rc;
  if (!t->mpole) {
    if ((rc = dalloc(ctx, &t->mpole, (size_t)t->ncells * 2 * t->p))) return rc;
    if ((rc = dalloc(ctx, &t->local, (size_t)t->ncells * 2 * t->p))) return rc;
    if ((rc = dalloc(ctx, &t->src, (size_t)t->n * 10))) return rc;
    if ((rc = dalloc(ctx, &t->part, (size_t)t->nitems * 32))) return rc;
    if ((rc = dalloc(ctx, &t->d_sorted, (size_t)t->n * 3))) return rc;
    if ((rc = dalloc(ctx, &t->y_sorted, (size_t)t->n * 3))) return rc;
    if ((rc = dalloc(ctx, &t->part_direct, (size_t)t->n * 2))) return rc;
  }
  return DDM_OK;
}

}  // namespace

// Translation operators (host, fp64), uploaded once per tree:
//   M2M_q[m][n] = rho^n C(m-1, n-1) eps^(m-n),     rho = 1/2, eps = (z_q - z_P)/s_P
//   L2L_q[k][m] = C(m, k) rho^k eps^(m-k)
//   h_o[k] = (k-1)! delta^-k, delta = -(dx + i dy)   (k = 1 .. 2p+1)
// stored transposed ([n][m] resp. [m][k]) for coalesced lane = output access.
int fmm_init_operators(ddm_tree_s* t, cudaStream_t s) {
  ddm_ctx_s* ctx = t->ctx;
  const int p = t->p;
  typedef std::vector<double2> V;
  V m2m((size_t)4 * p * p), l2l((size_t)4 * p * p), h((size_t)kNOffsets * (2 * p + 2));
  auto cpow = [](double re, double im, int k) {
    double a = 1.0, b = 0.0;
    for (int i = 0; i < k; ++i) {
      const double na = a * re - b * im, nb = a * im + b * re;
      a = na; b = nb;
    }
    return make_double2(a, b);
  };
  for (int q = 0; q < 4; ++q) {
    const double ex_ = 0.5 * ((q & 1) - 0.5), ey_ = 0.5 * ((q >> 1) - 0.5);
    for (int m = 1; m <= p; ++m)
      for (int n = 1; n <= p; ++n) {
        double2 v = make_double2(0.0, 0.0);
        if (n <= m) {
          const double2 e = cpow(ex_, ey_, m - n);
          const double f = std::ldexp(1.0, -n) * binom(m - 1, n - 1);
          v = make_double2(f * e.x, f * e.y);
        }
        m2m[(size_t)q * p * p + (size_t)(n - 1) * p + (m - 1)] = v;
      }
    for (int k = 0; k < p; ++k)
      for (int m = 0; m < p; ++m) {
        double2 v = make_double2(0.0, 0.0);
        if (m >= k) {
          const double2 e = cpow(ex_, ey_, m - k);
          const double f = std::ldexp(1.0, -k) * binom(m, k);
          v = make_double2(f * e.x, f * e.y);
        }
        l2l[(size_t)q * p * p + (size_t)m * p + k] = v;
      }
  }
  for (int o = 0; o < kNOffsets; ++o) {
    const int dx = o % 7 - 3, dy = o / 7 - 3;
    for (int k = 0; k < 2 * p + 2; ++k) h[(size_t)o * (2 * p + 2) + k] = make_double2(0.0, 0.0);
    if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
    // 1/delta = conj(delta)/|delta|^2, delta = -(dx + i dy)
    const double d2 = (double)dx * dx + (double)dy * dy;
    const double ir = -dx / d2, ii = dy / d2;
    double fact = 1.0;  // (k-1)!
    double pr = 1.0, pi = 0.0;
    for (int k = 1; k <= 2 * p + 1; ++k) {
      const double nr = pr * ir - pi * ii, ni = pr * ii + pi * ir;
      pr = nr; pi = ni;
      if (k >= 2) fact *= (k - 1);
      h[(size_t)o * (2 * p + 2) + k] = make_double2(fact * pr, fact * pi);
    }
  }
  std::vector<double> inv(2 * p + 2);
  double f = 1.0;
  for (int k = 0; k < 2 * p + 2; ++k) {
    if (k >= 1) f *= k;
    inv[k] = 1.0 / f;
  }
  int rc;
  if ((rc = dalloc(ctx, &t->op_m2m, m2m.size())) || (rc = dalloc(ctx, &t->op_l2l, l2l.size())) ||
      (rc = dalloc(ctx, &t->op_h, h.size())) || (rc = dalloc(ctx, &t->invfact, inv.size())))
    return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_m2m, m2m.data(), m2m.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_l2l, l2l.data(), l2l.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_h, h.data(), h.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->invfact, inv.data(), inv.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  return DDM_OK;
}

// Elastic matvec in sorted space.  D: user order [n][ncomp] (full on every
// rank).  Writes y_user (full user-order output, owned rows only) and/or
// y_sorted (owned rows).
int fmm_matvec_elastic(ddm_ctx_s* ctx, ddm_tree_s* t, double G, double nu, const double* D,
                       bool d_sorted, double* y_user, double* y_sorted, int mode,
                       cudaStream_t s) {
  int rc = ensure_workspace(ctx, t);
  if (rc) return rc;
  const int64_t n = t->n;
  const int ncomp = 2;
  const int p = t->p;
  const double gc = G / (4.0 * M_PI * (1.0 - nu));
  const CellGeom cg{t->x_min, t->y_min, t->W};
  const int64_t lo = t->own_el_lo, hi = t->own_el_hi;
  const int* perm_in = d_sorted ? nullptr : t->perm;

  stage_begin(ctx, DDM_ST_PREP, s);
  prep_sources<<<nblk(n, 256), 256, 0, s>>>(n, ncomp, perm_in, D, t->ex, t->ey, t->ea, t->ec,
                                            t->es, t->src, nullptr);
  DDM_CUDA(ctx, cudaGetLastError());
  stage_end(ctx, DDM_ST_PREP, s);

  if (mode == DDM_DIRECT) {
    double2* T = reinterpret_cast<double2*>(t->part_direct);
    stage_begin(ctx, DDM_ST_P2P, s);
    direct_kernel<<<nblk(hi - lo, kDirThreads), kDirThreads, 0, s>>>(
        n, lo, hi, t->src, t->ex, t->ey, t->ec, t->es, gc, T);
    DDM_CUDA(ctx, cudaGetLastError());
    stage_end(ctx, DDM_ST_P2P, s);
    scatter_direct<<<nblk(hi - lo, 256), 256, 0, s>>>(lo, hi, ncomp, T, t->perm, y_user, y_sorted);
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }

  // ---- upward pass: P2M on all leaves, M2M finest -> level 2
  stage_begin(ctx, DDM_ST_P2M, s);
  {
    const int stride = (p + 1) | 1;
    const size_t shm = (size_t)kP2MWarps * 32 * stride * 2 * sizeof(double2);
    if (shm > 48 * 1024)
      DDM_CUDA(ctx, cudaFuncSetAttribute(p2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)shm));
    const int nb = std::min(nblk(t->nleaves, kP2MWarps), 148u * 8);
    p2m_kernel<<<nb, kP2MWarps * 32, shm, s>>>(t->nleaves, t->leaves, t->c_level, t->c_ix,
                                               t->c_iy, t->c_start, t->c_count, cg, p, perm_in,
                                               D, ncomp, t->ex, t->ey, t->ea, t->ec, t->es,
                                               t->mpole);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  stage_end(ctx, DDM_ST_P2M, s);
  stage_begin(ctx, DDM_ST_M2M, s);
  for (int lev = t->nlevels - 2; lev >= 2; --lev) {
    const int c0 = t->level_off[lev], c1 = t->level_off[lev + 1];
    const int nb = std::min(nblk(c1 - c0, kM2MWarps), 148u * 8);
    m2m_kernel<<<nb, kM2MWarps * 32, 0, s>>>(c0, c1, t->c_leaf, t->c_ix, t->c_iy,
                                             t->c_first_child, t->c_nchild, p, t->op_m2m,
                                             t->mpole);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  stage_end(ctx, DDM_ST_M2M, s);

  // ---- downward pass: M2L at every level >= 2 (one launch), L2L top-down
  stage_begin(ctx, DDM_ST_M2L, s);
  if (t->nlevels > 2) {
    const int c0 = t->level_off[2], c1 = t->ncells;
    const size_t shm = ((size_t)kNOffsets * (2 * p + 2) + (size_t)kM2LWarps * 2 * (p + 2)) *
                       sizeof(double2);
    if (shm > 48 * 1024)
      DDM_CUDA(ctx, cudaFuncSetAttribute(m2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)shm));
    const int nb = std::min(nblk(c1 - c0, kM2LWarps), 148u * 2);
    m2l_kernel<<<nb, kM2LWarps * 32, shm, s>>>(c0, c1, t->v_off, t->v_idx, t->v_cls, p,
                                               t->op_h, t->invfact, t->mpole, t->local);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  stage_end(ctx, DDM_ST_M2L, s);
  stage_begin(ctx, DDM_ST_L2L, s);
  for (int lev = 3; lev < t->nlevels; ++lev) {
    const int c0 = t->level_off[lev], c1 = t->level_off[lev + 1];
    const int nb = std::min(nblk(c1 - c0, kL2LWarps), 148u * 8);
    l2l_kernel<<<nb, kL2LWarps * 32, 0, s>>>(c0, c1, t->c_parent, t->c_ix, t->c_iy, p,
                                             t->op_l2l, t->local);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  stage_end(ctx, DDM_ST_L2L, s);

  // ---- near field: P2P work items of owned leaves
  stage_begin(ctx, DDM_ST_P2P, s);
  {
    int ilo = 0, ihi = t->nitems;
    if (ctx->world > 1) {
      ilo = t->item_lo_owned;
      ihi = t->item_hi_owned;
    }
    if (ihi > ilo) {
      const int nb = std::min(nblk(ihi - ilo, kP2PWarps), 148u * 16);
      p2p_kernel<<<nb, kP2PWarps * 32, 0, s>>>(ilo, ihi, t->items, t->u_off, t->u_lo, t->u_hi,
                                               t->leaves, t->c_start, t->c_count, t->src, t->ex,
                                               t->ey, t->ec, t->es, gc, t->part);
      DDM_CUDA(ctx, cudaGetLastError());
    }
  }
  stage_end(ctx, DDM_ST_P2P, s);

  stage_begin(ctx, DDM_ST_FINAL, s);
  finalize_kernel<<<nblk(hi - lo, 128), 128, 0, s>>>(
      lo, hi, ncomp, t->el_leaf, t->leaves, t->c_level, t->c_ix, t->c_iy, t->c_start, t->c_count,
      t->item_off, t->part, t->local, cg, p, gc, t->ex, t->ey, t->ec, t->es, t->perm, y_user,
      y_sorted);
  DDM_CUDA(ctx, cudaGetLastError());
  stage_end(ctx, DDM_ST_FINAL, s);
  return DDM_OK;
}

}  // namespace ddm
