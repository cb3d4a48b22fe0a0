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

// Block-wide global -> shared copy with 8 loads in flight per thread (a plain
// strided loop waits one L2 round trip per element).
template <class T>
__device__ __forceinline__ void block_copy(T* __restrict__ dst, const T* __restrict__ src, int n) {
  const int step = blockDim.x;
  int f = threadIdx.x;
  for (; f + 7 * step < n; f += 8 * step) {
    T v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = src[f + k * step];
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[f + k * step] = v[k];
  }
  for (; f < n; f += step) dst[f] = src[f];
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
// One warp per work item (leaf k, group of nt <= kTgtGroup targets, interval
// of the leaf's concatenated source ranges).  The 32 lanes are split into
// S = 32 / nt source slices: lane l evaluates target l % nt against the
// sources j = l / nt (mod S) of each 32-source batch staged in shared memory;
// the S slice partials are then summed in a fixed order (deterministic).
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
  double2* buf = p2m_sh + (size_t)w * 32 * 17;     // [32 elements][16 (+1 pad)] per chunk
  const int nchunk = (p + 7) / 8;
  for (int k = blockIdx.x * kP2MWarps + w; k < nleaves; k += gridDim.x * kP2MWarps) {
    const int c = leaves[k];
    const int lev = c_level[c];
    const double s = cg.side(lev);
    const double is = 1.0 / s;
    const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
    const int e0 = c_start[c], ne = c_count[c];
    // lane < 16 owns column `lane` of every 8-coefficient chunk:
    // column j < 8 -> alpha slot 8 ch + j, column j >= 8 -> gamma slot 8 ch + j - 8
    double2 acc[kMaxP / 8];
#pragma unroll
    for (int q = 0; q < kMaxP / 8; ++q) acc[q] = make_double2(0.0, 0.0);
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
      const int rows = min(32, ne - r0);
#pragma unroll
      for (int ch = 0; ch < kMaxP / 8; ++ch) {
        if (ch < nchunk) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int n = 8 * ch + j + 1;        // coefficient index (slot n - 1)
            double2 alpha = make_double2(0.0, 0.0), gam = alpha;
            if (n <= p) {
              if (n >= 2) {
                pw1 = cmul(pw1, z1);
                pw2 = cmul(pw2, z2);
                Pm1 = Pm;
                Pm = csub(pw2, pw1);
              }
              alpha = cmul(B, Pm);
              gam = cmul(Q, Pm);
              double2 t = cscale(cmul(A, Pm1), (double)(n - 1));
              cmac(t, cscale(rr, (double)(n - 2)), Pm);
              cmac(gam, B, t);
            }
            buf[lane * 17 + j] = alpha;
            buf[lane * 17 + 8 + j] = gam;
          }
          __syncwarp();
          // column (lane & 15), rows of half (lane >> 4), fixed order
          const int col = lane & 15, h0 = (lane >> 4) * 16;
          double2 sum = make_double2(0.0, 0.0);
          for (int e = h0; e < min(rows, h0 + 16); ++e) sum = cadd(sum, buf[e * 17 + col]);
          sum.x += __shfl_down_sync(0xffffffffu, sum.x, 16);
          sum.y += __shfl_down_sync(0xffffffffu, sum.y, 16);
          acc[ch] = cadd(acc[ch], sum);
          __syncwarp();
        }
      }
    }
    double2* out = mpole + (size_t)c * 2 * p;
    if (lane < 16) {
#pragma unroll
      for (int ch = 0; ch < kMaxP / 8; ++ch) {
        const int slot = 8 * ch + (lane & 7);
        if (ch < nchunk && slot < p) out[(lane < 8 ? 0 : p) + slot] = acc[ch];
      }
    }
  }
}

// ------------------------------------------------------------ M2M (a6)
// parent P at level lev (non-leaf): sum over children q of
//   alpha^P_m = sum_n MT_q[n][m] alpha^q_n,  gamma^P_m = sum_n MT_q[n][m] c^q_n,
//   c_n = gamma_n - (n-1) conj(e)/s_c alpha_{n-1},  e = z_P - z_q.
// Warp per parent; the four quadrant operators live in shared memory and the
// children are accumulated in independent chains (ILP), summed in child order.
constexpr int kM2MWarps = 4;

__global__ void __launch_bounds__(kM2MWarps * 32)
m2m_kernel(int c0, int c1, const int* __restrict__ c_leaf, const int* __restrict__ c_ix,
           const int* __restrict__ c_iy, const int* __restrict__ first_child,
           const int* __restrict__ nchild, int p, const double2* __restrict__ opT,
           double2* __restrict__ mpole) {
  extern __shared__ double2 m2m_sh[];
  double2* ops = m2m_sh;                                   // [4][p][p]
  block_copy(ops, opT, 4 * p * p);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* xa = m2m_sh + 4 * p * p + (size_t)w * 8 * p;   // [4][p]
  double2* xc = xa + 4 * p;                                // [4][p]
  for (int c = c0 + blockIdx.x * kM2MWarps + w; c < c1; c += gridDim.x * kM2MWarps) {
    if (c_leaf[c]) continue;
    const int f = first_child[c], nc = nchild[c];
    int quad[4];
    for (int i = 0; i < 4; ++i) {
      quad[i] = 0;
      if (i < nc) {
        const int q = f + i;
        const int xb = c_ix[q] & 1, yb = c_iy[q] & 1;
        quad[i] = xb + 2 * yb;
        // conj(e)/s_c with e = z_P - z_q = -((xb-1/2) + i (yb-1/2)) s_c
        const double2 eb = make_double2(-(xb - 0.5), (yb - 0.5));
        const double2* mq = mpole + (size_t)q * 2 * p;
        for (int n = lane; n < p; n += 32) {
          xa[i * p + n] = mq[n];
          double2 cv = mq[p + n];
          if (n >= 1) cmac(cv, cscale(eb, -(double)n), mq[n - 1]);
          xc[i * p + n] = cv;
        }
      }
    }
    __syncwarp();
    double2* out = mpole + (size_t)c * 2 * p;
    for (int m = lane; m < p; m += 32) {
      double2 a[4], g[4];
      for (int i = 0; i < 4; ++i) a[i] = g[i] = make_double2(0.0, 0.0);
      for (int n = 0; n <= m; ++n) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < nc) {
            const double2 t = ops[(quad[i] * p + n) * p + m];
            cmac(a[i], t, xa[i * p + n]);
            cmac(g[i], t, xc[i * p + n]);
          }
        }
      }
      double2 sa = a[0], sg = g[0];
      for (int i = 1; i < 4; ++i) { sa = cadd(sa, a[i]); sg = cadd(sg, g[i]); }
      out[m] = sa;
      out[p + m] = sg;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ M2L (a7)
// target cell b, sources a in V(b):  with delta = (z_b - z_a)/s,
// h_k = (k-1)! delta^-k (table per offset class),
//   l_m = (-1)^m/m! sum_{n=1..p} [alpha_n/(n-1)!] h_{n+m}
//   g_m = (-1)^m/m! sum_{n=1..p+1} [c_n/(n-1)!] h_{n+m},  c_n = gamma_n - (n-1) conj(delta) alpha_{n-1}
// Rotated form: with delta = rho e^{i theta},
//   delta^-(n+m) = R_{n+m} e^{-i n theta} e^{-i m theta} / (n+m-1)!,
//   R_k = (k-1)! rho^-k (real), so each pair costs two real-Hankel sums over
//   rotated inputs plus one output rotation.  Tables per offset class:
//   rot[o][k] = e^{-i k theta}, R[o][k]; the next source's expansion is
//   prefetched into registers while the current one is applied.
constexpr int kM2LWarps = 8;

__global__ void __launch_bounds__(kM2LWarps * 32)
m2l_kernel(int c0, int c1, const int* __restrict__ v_off, const int* __restrict__ v_idx,
           const unsigned char* __restrict__ v_cls, int p, const double* __restrict__ rtab,
           const double2* __restrict__ rottab, const double* __restrict__ invfact,
           const double2* __restrict__ mpole, double2* __restrict__ local) {
  extern __shared__ double2 m2l_sh[];
  const int rs = 2 * p + 2;                          // R entries per class
  const int qs = p + 2;                              // rotation entries per class
  double2* sh_rot = m2l_sh;                          // [49][qs]
  double* sh_R = reinterpret_cast<double*>(m2l_sh + kNOffsets * qs);   // [49][rs]
  double2* wbuf = m2l_sh + kNOffsets * qs + (kNOffsets * rs + 1) / 2;
  block_copy(sh_rot, rottab, kNOffsets * qs);
  block_copy(sh_R, rtab, kNOffsets * rs);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sa = wbuf + (size_t)w * (3 * p + 2);      // raw alpha [p]
  double2* ap = sa + p;                               // rotated/scaled alpha [p]
  double2* cp = ap + p;                               // rotated/scaled c [p+1]
  for (int c = c0 + blockIdx.x * kM2LWarps + w; c < c1; c += gridDim.x * kM2LWarps) {
    double2 al[2], ag[2];
    al[0] = al[1] = ag[0] = ag[1] = make_double2(0.0, 0.0);
    const int vb = v_off[c], ve = v_off[c + 1];
    double2 na[2], ng[2];
    if (vb < ve) {
      const double2* ma = mpole + (size_t)v_idx[vb] * 2 * p;
      for (int cc = 0; cc < 2; ++cc) {
        const int n = lane + 32 * cc;
        na[cc] = n < p ? ma[n] : make_double2(0.0, 0.0);
        ng[cc] = n < p ? ma[p + n] : make_double2(0.0, 0.0);
      }
    }
    for (int v = vb; v < ve; ++v) {
      const int cls = v_cls[v];
      const double2 xa0 = na[0], xa1 = na[1], xg0 = ng[0], xg1 = ng[1];
      if (v + 1 < ve) {   // prefetch the next source
        const double2* ma = mpole + (size_t)v_idx[v + 1] * 2 * p;
        for (int cc = 0; cc < 2; ++cc) {
          const int n = lane + 32 * cc;
          if (n < p) {
            na[cc] = ma[n];
            ng[cc] = ma[p + n];
          }
        }
      }
      const int dxs = cls % 7 - 3, dys = cls / 7 - 3;   // source - target in cells
      const double2 dconj = make_double2(-(double)dxs, (double)dys);  // conj(delta)
      const double2* rot = sh_rot + cls * qs;
      const double* R = sh_R + cls * rs;
      if (lane < p) sa[lane] = xa0;
      if (lane + 32 < p) sa[lane + 32] = xa1;
      __syncwarp();
      for (int cc = 0; cc < 2; ++cc) {   // slot n <-> coefficient n + 1
        const int n = lane + 32 * cc;
        if (n <= p) {
          double2 cv = (n < p) ? (cc ? xg1 : xg0) : make_double2(0.0, 0.0);
          if (n >= 1) cmac(cv, cscale(dconj, -(double)n), sa[n - 1]);
          const double2 r = cscale(rot[n + 1], invfact[n]);
          cp[n] = cmul(cv, r);
          if (n < p) ap[n] = cmul(cc ? xa1 : xa0, r);
        }
      }
      __syncwarp();
      for (int cc = 0; cc < 2; ++cc) {
        const int m = lane + 32 * cc;
        if (m < p) {
          double2 sl = make_double2(0.0, 0.0), sg = sl;
          const double* Rm = R + 1 + m;
#pragma unroll 4
          for (int n = 0; n < p; ++n) {
            const double rk = Rm[n];
            const double2 a = ap[n], g = cp[n];
            sl.x = fma(a.x, rk, sl.x);
            sl.y = fma(a.y, rk, sl.y);
            sg.x = fma(g.x, rk, sg.x);
            sg.y = fma(g.y, rk, sg.y);
          }
          const double rk = Rm[p];
          sg.x = fma(cp[p].x, rk, sg.x);
          sg.y = fma(cp[p].y, rk, sg.y);
          const double2 ro = rot[m];
          cmac(al[cc], sl, ro);
          cmac(ag[cc], sg, ro);
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
// Warp per parent P (non-leaf, level lev-1): shifts P's local expansion to
// each of its children (independent chains), operators in shared memory.
constexpr int kL2LWarps = 4;

__global__ void __launch_bounds__(kL2LWarps * 32)
l2l_kernel(int c0, int c1, const int* __restrict__ c_leaf, const int* __restrict__ c_ix,
           const int* __restrict__ c_iy, const int* __restrict__ first_child,
           const int* __restrict__ nchild, int p, const double2* __restrict__ opT,
           double2* __restrict__ local) {
  extern __shared__ double2 l2l_sh[];
  double2* ops = l2l_sh;                                     // [4][p][p]
  block_copy(ops, opT, 4 * p * p);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sl = l2l_sh + 4 * p * p + (size_t)w * 2 * p;
  double2* sgv = sl + p;
  for (int P = c0 + blockIdx.x * kL2LWarps + w; P < c1; P += gridDim.x * kL2LWarps) {
    if (c_leaf[P]) continue;
    const double2* lp = local + (size_t)P * 2 * p;
    for (int m = lane; m < p; m += 32) {
      sl[m] = lp[m];
      sgv[m] = lp[p + m];
    }
    __syncwarp();
    const int f = first_child[P], nc = nchild[P];
    int quad[4];
    double2 epsb[4];
    for (int i = 0; i < 4; ++i) {
      const int q = f + min(i, nc - 1);
      const int xb = c_ix[q] & 1, yb = c_iy[q] & 1;
      quad[i] = xb + 2 * yb;
      epsb[i] = make_double2(0.5 * (xb - 0.5), -0.5 * (yb - 0.5));  // conj(eps)
    }
    for (int k = lane; k < p; k += 32) {
      double2 l[4], g[4];
      for (int i = 0; i < 4; ++i) l[i] = g[i] = make_double2(0.0, 0.0);
      for (int m = k; m < p; ++m) {
        const double2 lm = sl[m];
        const double2 gm = sgv[m];
        const double2 lm1 = (m + 1 < p) ? sl[m + 1] : make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < nc) {
            // g_m = gamma_m + (m+1) conj(eps) lambda_{m+1}
            double2 gv = gm;
            cmac(gv, cscale(epsb[i], (double)(m + 1)), lm1);
            const double2 t = ops[(quad[i] * p + m) * p + k];
            cmac(l[i], t, lm);
            cmac(g[i], t, gv);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nc) {
          double2* out = local + (size_t)(f + i) * 2 * p;
          out[k] = cadd(out[k], l[i]);
          out[p + k] = cadd(out[p + k], g[i]);
        }
      }
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
  for (int h = 0; h < nch; ++h) T = cadd(T, part[(int64_t)(i0 + g * nch + h) * kTgtGroup + ln]);
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
    if ((rc = dalloc(ctx, &t->part, (size_t)t->nitems * kTgtGroup))) return rc;
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
  // M2L tables per offset class: rot[o][k] = e^{-i k theta} (k = 0..p+1) and
  // R[o][k] = (k-1)! rho^-k (k = 1..2p+1), delta = -(dx + i dy) = rho e^{i theta}
  std::vector<double> R((size_t)kNOffsets * (2 * p + 2), 0.0);
  V rot((size_t)kNOffsets * (p + 2), make_double2(0.0, 0.0));
  for (int o = 0; o < kNOffsets; ++o) {
    const int dx = o % 7 - 3, dy = o / 7 - 3;
    if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
    const double rho = std::sqrt((double)dx * dx + (double)dy * dy);
    const double er = -dx / rho, ei = dy / rho;   // e^{-i theta} = conj(delta)/rho
    double pr = 1.0, pi = 0.0;
    for (int k = 0; k < p + 2; ++k) {
      rot[(size_t)o * (p + 2) + k] = make_double2(pr, pi);
      const double nr = pr * er - pi * ei, ni = pr * ei + pi * er;
      pr = nr; pi = ni;
    }
    double fact = 1.0, rp = 1.0;
    for (int k = 1; k <= 2 * p + 1; ++k) {
      if (k >= 2) fact *= (k - 1);
      rp /= rho;
      R[(size_t)o * (2 * p + 2) + k] = fact * rp;
    }
  }
  h = rot;
  std::vector<double> inv(2 * p + 2);
  double f = 1.0;
  for (int k = 0; k < 2 * p + 2; ++k) {
    if (k >= 1) f *= k;
    inv[k] = 1.0 / f;
  }
  int rc;
  if ((rc = dalloc(ctx, &t->op_m2m, m2m.size())) || (rc = dalloc(ctx, &t->op_l2l, l2l.size())) ||
      (rc = dalloc(ctx, &t->op_h, h.size())) || (rc = dalloc(ctx, &t->invfact, inv.size())) ||
      (rc = dalloc(ctx, &t->op_R, R.size())))
    return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_R, R.data(), R.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
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
    const size_t shm = (size_t)kP2MWarps * 32 * 17 * sizeof(double2);
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
  {
    const size_t shm = ((size_t)4 * p * p + (size_t)kM2MWarps * 8 * p) * sizeof(double2);
    if (shm > 48 * 1024)
      DDM_CUDA(ctx, cudaFuncSetAttribute(m2m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)shm));
    for (int lev = t->nlevels - 2; lev >= 2; --lev) {
      const int c0 = t->level_off[lev], c1 = t->level_off[lev + 1];
      const int nb = std::min(nblk(c1 - c0, kM2MWarps), 148u * 4);
      m2m_kernel<<<nb, kM2MWarps * 32, shm, s>>>(c0, c1, t->c_leaf, t->c_ix, t->c_iy,
                                                 t->c_first_child, t->c_nchild, p, t->op_m2m,
                                                 t->mpole);
      DDM_CUDA(ctx, cudaGetLastError());
    }
  }
  stage_end(ctx, DDM_ST_M2M, s);

  // ---- downward pass: M2L at every level >= 2 (one launch), L2L top-down
  stage_begin(ctx, DDM_ST_M2L, s);
  if (t->nlevels > 2) {
    const int c0 = t->level_off[2], c1 = t->ncells;
    const size_t shm = ((size_t)kNOffsets * (p + 2) + ((size_t)kNOffsets * (2 * p + 2) + 1) / 2 +
                        (size_t)kM2LWarps * (3 * p + 2)) * sizeof(double2);
    if (shm > 48 * 1024)
      DDM_CUDA(ctx, cudaFuncSetAttribute(m2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)shm));
    const int nb = std::min(nblk(c1 - c0, kM2LWarps), 148u * 4);
    m2l_kernel<<<nb, kM2LWarps * 32, shm, s>>>(c0, c1, t->v_off, t->v_idx, t->v_cls, p,
                                               t->op_R, t->op_h, t->invfact, t->mpole, t->local);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  stage_end(ctx, DDM_ST_M2L, s);
  stage_begin(ctx, DDM_ST_L2L, s);
  {
    const size_t shm = ((size_t)4 * p * p + (size_t)kL2LWarps * 2 * p) * sizeof(double2);
    if (shm > 48 * 1024)
      DDM_CUDA(ctx, cudaFuncSetAttribute(l2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)shm));
    // parents at level lev (>= 2) push to their children at lev + 1
    for (int lev = 2; lev + 1 < t->nlevels; ++lev) {
      const int c0 = t->level_off[lev], c1 = t->level_off[lev + 1];
      const int nb = std::min(nblk(c1 - c0, kL2LWarps), 148u * 4);
      l2l_kernel<<<nb, kL2LWarps * 32, shm, s>>>(c0, c1, t->c_leaf, t->c_ix, t->c_iy,
                                                 t->c_first_child, t->c_nchild, p, t->op_l2l,
                                                 t->local);
      DDM_CUDA(ctx, cudaGetLastError());
    }
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
