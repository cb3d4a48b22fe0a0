// Upward and downward passes of the FMM (DESIGN.md §4 rows a5-a9):
// P2M ("P2L", Eq.(p2l)), M2M (Eq.(m2m)), M2L (Eq.(m2l)
// P:841-851), L2L (Eq.(l2l)), L2P with the
// complex-variable expansions of DESIGN.md §5.
//
// Normalised storage (cell side s, centre z0):
//   multipole  Phi(z) = sum_{n=1..p} a_n ((z - z0)/s)^(-n)      (slot n-1)
//   local      Phi(z) = sum_{m=0..p-1} l_m ((z - z0)/s)^m       (slot m)
// and likewise for Psi~ = Psi + conj(z0) Phi'.  The factor i G C,
// C = 1/(4 pi (1 - nu)), is applied once, at evaluation.
//
// Scheduling: each pass is ONE persistent launch.  Warps take
// cells in topological order from an atomic ticket counter (upward: all leaves
// (P2M), then non-leaf cells deepest level first (M2M); downward: cells of
// level >= 2 top-down (M2L, then L2L from the parent)).  A cell waits for the
// cells it depends on through per-cell ready flags (release / acquire, tagged
// with a per-call epoch).  Everything a warp waits for holds a lower ticket,
// i.e. it was taken earlier by a running warp, so the wait cannot deadlock.
//
// Every kernel is a template on the expansion order PT (PT = 0: runtime p) so
// that, for the instantiated orders, inner loops unroll and loads pipeline.
#include <algorithm>
#include <cstdlib>

#include "kcommon.cuh"

namespace ddm {
namespace {

#define DDM_P_DISPATCH(p, F)              \
  switch (p) {                            \
    case 8: F(8); break;                  \
    case 12: F(12); break;                \
    case 16: F(16); break;                \
    case 20: F(20); break;                \
    case 24: F(24); break;                \
    case 28: F(28); break;                \
    case 32: F(32); break;                \
    case 40: F(40); break;                \
    default: F(0); break;                 \
  }

template <int PT>
__host__ __device__ constexpr int pmax() { return PT ? PT : kMaxP; }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// all lanes: spin until flag == epoch (acquire by every lane)
__device__ __forceinline__ void wait_ready(const int* flag, int epoch) {
  while (ld_acquire(flag) != epoch) __nanosleep(64);
}
// publish the warp's writes, then set the flag
__device__ __forceinline__ void publish(int* flag, int epoch, int lane) {
  __threadfence();
  __syncwarp();
  if (lane == 0) st_release(flag, epoch);
}

constexpr int kPassWarps = 8;

// ------------------------------------------------------------ P2M (a5)
// Warp per leaf; lane = element of a 32-element round.
//   alpha_n = (B/s) P_{n-1}
//   gamma_n = (1/s)[Q P_{n-1} + B((n-1) A P_{n-2} + (n-2) r P_{n-1})]
// zeta_{1,2} = (z_{1,2} - z0)/s, P_m = zeta2^m - zeta1^m, A = conj(zc - z0)/s - r (zc - z0)/s.
// Coefficients are produced in chunks of 8 and summed over the elements of
// the round through a padded [32][17] shared-memory transpose (fixed order).
template <int PT>
__device__ void p2m_cell(int c, int p, const int* __restrict__ c_level, const int* __restrict__ c_ix,
                         const int* __restrict__ c_iy, const int* __restrict__ c_start,
                         const int* __restrict__ c_count, const CellGeom& cg,
                         const int* __restrict__ perm, const double* __restrict__ D, int ncomp,
                         const double* __restrict__ ex, const double* __restrict__ ey,
                         const double* __restrict__ ea, const double* __restrict__ ec,
                         const double* __restrict__ es, double2* __restrict__ mpole, double2* buf,
                         int lane, const PoroFar& pf) {
  constexpr int NCH = (pmax<PT>() + 7) / 8;
  const int nchunk = (p + 7) / 8;
  const int lev = c_level[c];
  const double s = cg.side(lev);
  const double is = 1.0 / s;
  const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
  const int e0 = c_start[c], ne = c_count[c];
  // lane < 16 owns column `lane` of every chunk:
  // column j < 8 -> alpha slot 8 ch + j, column j >= 8 -> gamma slot 8 ch + j - 8
  double2 acc[NCH];
#pragma unroll
  for (int q = 0; q < NCH; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < ne; r0 += 32) {
    const int i = e0 + r0 + lane;
    const bool valid = r0 + lane < ne;
    double2 B = make_double2(0, 0), Q = B, rr = B, A = B, z1 = B, z2 = B;
    // poroelastic far field: B-part of Phi and Psi~ scaled by
    // fu, plus Wm conj(e) I2 and Wc B I4 in Psi~ (iGC factored out)
    double2 Wme = make_double2(0, 0), Bc = Wme;
    double fu = 1.0;
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
      if (pf.on) {
        const double qf = -D[(int64_t)j * ncomp + 2];          // J: q_formula = -q_ABI
        const double mu = -(pf.eta / pf.S) * dn;
        const double wm = (pf.eta * mu / M_PI + pf.eta * qf * pf.ct / (M_PI * pf.kappa)) / pf.gc;
        // (wm / i) conj(e) / s, and 48 eta k_p c tau B / s^3
        Wme = cscale(cmul(make_double2(0.0, -wm), make_double2(cb, -sb)), is);
        Bc = cscale(B, 48.0 * pf.eta * pf.kp * pf.ct * is * is * is);
        fu = pf.fu;
      }
      B = cscale(B, is);
      Q = cscale(Q, is);
    }
    double2 pw1 = make_double2(1.0, 0.0), pw2 = pw1;
    double2 Pm2 = make_double2(0.0, 0.0);   // P_{n-3}
    double2 Pm1 = make_double2(0.0, 0.0);   // P_{n-2}
    double2 Pm = make_double2(0.0, 0.0);    // P_{n-1}
    const int rows = min(32, ne - r0);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      if (ch < nchunk) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = 8 * ch + j + 1;        // coefficient index (slot n - 1)
          double2 alpha = make_double2(0.0, 0.0), gam = alpha;
          if (n <= p) {
            if (n >= 2) {
              pw1 = cmul(pw1, z1);
              pw2 = cmul(pw2, z2);
              Pm2 = Pm1;
              Pm1 = Pm;
              Pm = csub(pw2, pw1);
            }
            alpha = cscale(cmul(B, Pm), fu);
            gam = cmul(Q, Pm);
            double2 tt = cscale(cmul(A, Pm1), (double)(n - 1));
            cmac(tt, cscale(rr, (double)(n - 2)), Pm);
            cmac(gam, cscale(B, fu), tt);
            if (pf.on) {
              cmac(gam, Wme, Pm);
              if (n >= 4) cmac(gam, cscale(Bc, (n - 1) * (n - 2) / 6.0), Pm2);
            }
          }
          buf[lane * 17 + j] = alpha;
          buf[lane * 17 + 8 + j] = gam;
        }
        __syncwarp();
        const int col = lane & 15, h0 = (lane >> 4) * 16;
        double2 sum = make_double2(0.0, 0.0);
        const int hend = min(rows, h0 + 16);
        for (int e = h0; e < hend; ++e) sum = cadd(sum, buf[e * 17 + col]);
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
    for (int ch = 0; ch < NCH; ++ch) {
      const int slot = 8 * ch + (lane & 7);
      if (ch < nchunk && slot < p) out[(lane < 8 ? 0 : p) + slot] = acc[ch];
    }
  }
}

// ------------------------------------------------------------ M2M (a6)
// Parent c from its children q (all ready):
//   alpha^c_m = sum_q sum_n M_q[n][m] alpha^q_n,  gamma^c_m = sum_q sum_n M_q[n][m] c^q_n,
//   c_n = gamma_n - (n-1) conj(e)/s_q alpha_{n-1},  e = z_c - z_q,
// M_q[n][m] = 2^{-n} C(m-1, n-1) eps_q^{m-n} (zero for n > m), eps_q = (z_q - z_c)/s_c.
template <int PT>
__device__ void m2m_cell(int c, int p, const int* __restrict__ c_ix, const int* __restrict__ c_iy,
                         const int* __restrict__ first_child, const int* __restrict__ nchild,
                         const double2* ops, double2* __restrict__ mpole, double2* xa, double2* xc,
                         const int* ready, int epoch, int lane) {
  const int f = first_child[c], nc = nchild[c];
  int quad[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    quad[i] = 0;
    if (i < nc) {
      const int q = f + i;
      wait_ready(ready + q, epoch);
      const int xb = c_ix[q] & 1, yb = c_iy[q] & 1;
      quad[i] = xb + 2 * yb;
      const double2 eb = make_double2(-(xb - 0.5), (yb - 0.5));   // conj(e)/s_q
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
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = g[i] = make_double2(0.0, 0.0);
#pragma unroll
    for (int n = 0; n < pmax<PT>(); ++n) {
      if (!PT && n >= p) break;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nc) {
          const double2 tq = ops[(quad[i] * p + n) * p + m];
          cmac(a[i], tq, xa[i * p + n]);
          cmac(g[i], tq, xc[i * p + n]);
        }
      }
    }
    double2 sa = a[0], sg = g[0];
#pragma unroll
    for (int i = 1; i < 4; ++i) {
      sa = cadd(sa, a[i]);
      sg = cadd(sg, g[i]);
    }
    out[m] = sa;
    out[p + m] = sg;
  }
  __syncwarp();
}

// Upward pass: tickets [0, nleaves) = P2M of leaves[t]; then M2M of
// up_list[t - nleaves] (non-leaf cells of level >= 2, deepest level first).
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
upward_kernel(int nleaves, int nm2m, const int* __restrict__ leaves,
              const int* __restrict__ up_list, const int* __restrict__ c_level,
              const int* __restrict__ c_ix, const int* __restrict__ c_iy,
              const int* __restrict__ c_start, const int* __restrict__ c_count,
              const int* __restrict__ first_child, const int* __restrict__ nchild, CellGeom cg,
              int p_rt, const int* __restrict__ perm, const double* __restrict__ D, int ncomp,
              const double* __restrict__ ex, const double* __restrict__ ey,
              const double* __restrict__ ea, const double* __restrict__ ec,
              const double* __restrict__ es, const double2* __restrict__ opT,
              double2* __restrict__ mpole, int* __restrict__ ready, int epoch,
              int* __restrict__ ticket, PoroFar pf) {
  const int p = PT ? PT : p_rt;
  extern __shared__ double2 up_sh[];
  double2* ops = up_sh;                                      // [4][p][p] as [q][n][m]
  block_copy(ops, opT, 4 * p * p);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* wb = up_sh + 4 * p * p + (size_t)w * (32 * 17 > 8 * p ? 32 * 17 : 8 * p);
  const int total = nleaves + nm2m;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= total) break;
    int c;
    if (t < nleaves) {
      c = leaves[t];
      p2m_cell<PT>(c, p, c_level, c_ix, c_iy, c_start, c_count, cg, perm, D, ncomp, ex, ey, ea,
                   ec, es, mpole, wb, lane, pf);
    } else {
      c = up_list[t - nleaves];
      m2m_cell<PT>(c, p, c_ix, c_iy, first_child, nchild, ops, mpole, wb, wb + 4 * p, ready,
                   epoch, lane);
    }
    publish(ready + c, epoch, lane);
  }
}

// ------------------------------------------------------------ M2L (a7) + L2L (a8)
// Rotated M2L: with delta = (z_b - z_a)/s = rho e^{i theta},
//   l_m = (-1)^m/m! e^{-i m theta} sum_{n=1..p} [alpha_n e^{-i n theta}/(n-1)!] R_{n+m}
//   g_m = (-1)^m/m! e^{-i m theta} sum_{n=1..p+1} [c_n e^{-i n theta}/(n-1)!] R_{n+m}
//   c_n = gamma_n - (n-1) conj(delta) alpha_{n-1},  R_k = (k-1)! rho^-k (real)
// then L2L from the (final) parent P:
//   g'_m = gamma^P_m + (m+1) conj(eps) lambda^P_{m+1},  eps = (z_c - z_P)/s_P
//   lambda^c_k += sum_m L_q[m][k] lambda^P_m,  gamma^c_k += sum_m L_q[m][k] g'_m
// L_q[m][k] = C(m, k) 2^{-k} eps^{m-k} (zero for m < k).
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
downward_kernel(int c0, int c1, int64_t own_lo, int64_t own_hi, const int* __restrict__ v_off,
                const int* __restrict__ v_idx, const unsigned char* __restrict__ v_cls,
                const int* __restrict__ c_level, const int* __restrict__ c_ix,
                const int* __restrict__ c_iy, const int* __restrict__ c_start,
                const int* __restrict__ c_count, const int* __restrict__ c_parent, int p_rt,
                const double* __restrict__ rtab, const double2* __restrict__ rottab,
                const double* __restrict__ invfact, const double2* __restrict__ l2lT,
                const double2* __restrict__ mpole, double2* __restrict__ local,
                int* __restrict__ ready, int epoch, int* __restrict__ ticket) {
  const int p = PT ? PT : p_rt;
  extern __shared__ double2 dn_sh[];
  const int rs = 2 * p + 2;                          // R entries per class
  const int qs = p + 2;                              // rotation entries per class
  double2* sh_l2l = dn_sh;                           // [4][p][p] as [q][m][k]
  double2* sh_rot = sh_l2l + 4 * p * p;              // [49][qs]
  double* sh_R = reinterpret_cast<double*>(sh_rot + kNOffsets * qs);   // [49][rs]
  double2* wbuf = sh_rot + kNOffsets * qs + (kNOffsets * rs + 1) / 2;
  block_copy(sh_l2l, l2lT, 4 * p * p);
  block_copy(sh_rot, rottab, kNOffsets * qs);
  block_copy(sh_R, rtab, kNOffsets * rs);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sa = wbuf + (size_t)w * (3 * p + 2);      // raw alpha [p]      | parent lambda [p]
  double2* ap = sa + p;                               // rotated alpha [p]  | g' [p]
  double2* cp = ap + p;                               // rotated c [p+1]
  const int total = c1 - c0;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= total) break;
    const int c = c0 + t;
    const int cs = c_start[c], ce = cs + c_count[c];
    if (ce <= own_lo || cs >= own_hi) {   // subtree outside this rank's targets
      publish(ready + c, epoch, lane);
      continue;
    }
    double2 al[2], ag[2];
    al[0] = al[1] = ag[0] = ag[1] = make_double2(0.0, 0.0);
    const int vb = v_off[c], ve = v_off[c + 1];
    double2 na[2], ng[2];
    na[0] = na[1] = ng[0] = ng[1] = make_double2(0.0, 0.0);
    if (vb < ve) {
      const double2* ma = mpole + (size_t)v_idx[vb] * 2 * p;
      for (int cc = 0; cc < 2; ++cc) {
        const int n = lane + 32 * cc;
        if (n < p) {
          na[cc] = ma[n];
          ng[cc] = ma[p + n];
        }
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
          const double2 rr = cscale(rot[n + 1], invfact[n]);
          cp[n] = cmul(cv, rr);
          if (n < p) ap[n] = cmul(cc ? xa1 : xa0, rr);
        }
      }
      __syncwarp();
      for (int cc = 0; cc < 2; ++cc) {
        const int m = lane + 32 * cc;
        if (m < p) {
          double2 sl = make_double2(0.0, 0.0), sg = sl;
          const double* Rm = R + 1 + m;
#pragma unroll
          for (int n = 0; n < pmax<PT>(); ++n) {
            if (!PT && n >= p) break;
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
    for (int cc = 0; cc < 2; ++cc) {
      const int m = lane + 32 * cc;
      if (m < p) {
        const double sc = ((m & 1) ? -1.0 : 1.0) * invfact[m];
        al[cc] = cscale(al[cc], sc);
        ag[cc] = cscale(ag[cc], sc);
      }
    }
    // L2L from the parent (its local expansion is final once its flag is set)
    if (c_level[c] >= 3) {
      const int P = c_parent[c];
      wait_ready(ready + P, epoch);
      const double2* lp = local + (size_t)P * 2 * p;
      const int xb = c_ix[c] & 1, yb = c_iy[c] & 1;
      const int quad = xb + 2 * yb;
      const double2 epsb = make_double2(0.5 * (xb - 0.5), -0.5 * (yb - 0.5));   // conj(eps)
      double2* sl = sa;
      double2* sg = ap;
      for (int m = lane; m < p; m += 32) {
        sl[m] = lp[m];
        double2 gv = lp[p + m];
        if (m + 1 < p) cmac(gv, cscale(epsb, (double)(m + 1)), lp[m + 1]);
        sg[m] = gv;
      }
      __syncwarp();
      const double2* L = sh_l2l + (size_t)quad * p * p;
      for (int cc = 0; cc < 2; ++cc) {
        const int k = lane + 32 * cc;
        if (k < p) {
          double2 l = al[cc], g = ag[cc];
#pragma unroll
          for (int m = 0; m < pmax<PT>(); ++m) {
            if (!PT && m >= p) break;
            const double2 tq = L[m * p + k];
            cmac(l, tq, sl[m]);
            cmac(g, tq, sg[m]);
          }
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
        out[m] = al[cc];
        out[p + m] = ag[cc];
      }
    }
    publish(ready + c, epoch, lane);
  }
}

// ------------------------------------------------------------ L2P + finalize (a9, a11)
// per owned sorted element: sum P2P partials in item order, add the far field
// from the leaf's local expansion, write (sigma_s, sigma_n).
template <int PT>
__global__ void finalize_kernel(int64_t e_lo, int64_t e_hi, int ncomp,
                                const int* __restrict__ el_leaf, const int* __restrict__ leaves,
                                const int* __restrict__ c_level, const int* __restrict__ c_ix,
                                const int* __restrict__ c_iy, const int* __restrict__ c_start,
                                const int* __restrict__ c_count,
                                const int* __restrict__ item_off, const double* __restrict__ part,
                                const double2* __restrict__ local, CellGeom cg, int p_rt,
                                double gc, PoroFar pf, const double* __restrict__ ex,
                                const double* __restrict__ ey, const double* __restrict__ ec,
                                const double* __restrict__ es, const int* __restrict__ perm,
                                double* __restrict__ y_user, double* __restrict__ y_sorted) {
  const int p = PT ? PT : p_rt;
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
  double pr = 0.0;
  for (int h = 0; h < nch; ++h) {
    const double* pp = part + ((int64_t)(i0 + g * nch + h) * kTgtGroup + ln) * ncomp;
    T.x += pp[0];
    T.y += pp[1];
    if (ncomp == 3) pr += pp[2];
  }
  const int lev = c_level[c];
  if (lev >= 2) {
    const double s = cg.side(lev);
    const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
    const double2 u = make_double2((ex[i] - z0.x) / s, (ey[i] - z0.y) / s);
    const double2* L = local + (size_t)c * 2 * p;
    double2 phi = make_double2(0, 0), dphi = phi, psi = phi;
#pragma unroll
    for (int mm = pmax<PT>() - 1; mm >= 0; --mm) {
      if (!PT && mm >= p) continue;
      if (mm >= 1) dphi = cadd(cmul(dphi, u), cscale(L[mm], (double)mm));
      phi = cadd(cmul(phi, u), L[mm]);
      psi = cadd(cmul(psi, u), L[p + mm]);
    }
    // W = i G C (conj(u) dPhi + Psi~), T += 2 Re(i G C Phi) + e^{2 i b} W
    const double2 wv = cadd(cmul(cconj(u), dphi), psi);
    const double2 W = make_double2(-gc * wv.y, gc * wv.x);
    const double ct = ec[i], st = es[i];
    const double2 e2 = make_double2(ct * ct - st * st, 2.0 * ct * st);
    const double2 t2 = cmul(e2, W);
    T.x += t2.y;
    T.y += t2.x - 2.0 * gc * phi.y;
    // far pore pressure p = -4 k_p Re(i G C Phi)/fu (formula sign), ABI p = -that
    if (pf.on) pr -= 4.0 * pf.kp * gc * phi.y / pf.fu;
  }
  if (y_sorted) {
    y_sorted[i * ncomp + 0] = T.x;
    y_sorted[i * ncomp + 1] = T.y;
    if (ncomp == 3) y_sorted[i * ncomp + 2] = pr;
  }
  if (y_user) {
    const int j = perm[i];
    y_user[(int64_t)j * ncomp + 0] = T.x;
    y_user[(int64_t)j * ncomp + 1] = T.y;
    if (ncomp == 3) y_user[(int64_t)j * ncomp + 2] = pr;
  }
}

template <class K>
int set_smem(ddm_ctx_s* ctx, K kernel, size_t shm) {
  if (shm > 48 * 1024)
    DDM_CUDA(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  return DDM_OK;
}

int pass_grid(ddm_ctx_s* ctx, const void* kernel, size_t shm, int work) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kPassWarps * 32, shm);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
  const int by_work = (work + kPassWarps - 1) / kPassWarps;
  // DDM_PASS_BLOCKS_PER_SM caps the persistent grid so the concurrent near
  // field keeps SM slots (0 = occupancy limit)
  // default: 1 block per SM when the near field runs concurrently (measured
  // best), the occupancy limit when everything is serial
  static const int env_cap = [] {
    const char* e = getenv("DDM_PASS_BLOCKS_PER_SM");
    return e ? atoi(e) : -1;
  }();
  const int cap = env_cap >= 0 ? env_cap : (ctx->serial ? 0 : 1);
  if (cap > 0) per_sm = std::min(per_sm, cap);
  return std::max(1, std::min(std::max(per_sm, 1) * nsm, by_work));
}

}  // namespace

// upward pass: P2M on all leaves + M2M of every non-leaf cell of level >= 2
int launch_upward(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D, int ncomp,
                  const PoroFar& pf, cudaStream_t s) {
  const int p = t->p;
  const CellGeom cg{t->x_min, t->y_min, t->W};
  const size_t wsz = std::max(32 * 17, 8 * p);
  const size_t shm = ((size_t)4 * p * p + (size_t)kPassWarps * wsz) * sizeof(double2);
  ++t->epoch;
  DDM_CUDA(ctx, cudaMemsetAsync(t->tickets, 0, 2 * sizeof(int), s));
  int rc = DDM_OK;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if ((rc = set_smem(ctx, upward_kernel<PT>, shm))) return rc;                                \
    const int nb = pass_grid(ctx, (const void*)upward_kernel<PT>, shm, t->nleaves + t->n_up);   \
    upward_kernel<PT><<<nb, kPassWarps * 32, shm, s>>>(                                         \
        t->nleaves, t->n_up, t->leaves, t->up_list, t->c_level, t->c_ix, t->c_iy, t->c_start,   \
        t->c_count, t->c_first_child, t->c_nchild, cg, p, perm_in, D, ncomp, t->ex, t->ey,      \
        t->ea, t->ec, t->es, t->op_m2m, t->mpole, t->ready_up, t->epoch, t->tickets, pf);       \
  } while (0)
  DDM_P_DISPATCH(p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// downward pass: M2L + L2L of every cell of level >= 2, top-down
int launch_downward(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) {
  if (t->nlevels <= 2) return DDM_OK;
  const int p = t->p;
  const int c0 = t->level_off[2], c1 = t->ncells;
  const size_t shm = ((size_t)4 * p * p + (size_t)kNOffsets * (p + 2) +
                      ((size_t)kNOffsets * (2 * p + 2) + 1) / 2 +
                      (size_t)kPassWarps * (3 * p + 2)) * sizeof(double2);
  int rc = DDM_OK;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if ((rc = set_smem(ctx, downward_kernel<PT>, shm))) return rc;                              \
    const int nb = pass_grid(ctx, (const void*)downward_kernel<PT>, shm, c1 - c0);              \
    downward_kernel<PT><<<nb, kPassWarps * 32, shm, s>>>(                                       \
        c0, c1, t->own_el_lo, t->own_el_hi, t->v_off, t->v_idx, t->v_cls, t->c_level, t->c_ix,  \
        t->c_iy, t->c_start, t->c_count, t->c_parent, p, t->op_R, t->op_h, t->invfact,          \
        t->op_l2l, t->mpole, t->local, t->ready_down, t->epoch, t->tickets + 1);                \
  } while (0)
  DDM_P_DISPATCH(p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_finalize(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, int ncomp, double gc,
                    const PoroFar& pf, double* y_user, double* y_sorted, cudaStream_t s) {
  if (hi <= lo) return DDM_OK;
  const CellGeom cg{t->x_min, t->y_min, t->W};
  const unsigned nb = nblk(hi - lo, 128);
#define DDM_L(PT)                                                                               \
  finalize_kernel<PT><<<nb, 128, 0, s>>>(lo, hi, ncomp, t->el_leaf, t->leaves, t->c_level,      \
                                         t->c_ix, t->c_iy, t->c_start, t->c_count, t->item_off, \
                                         reinterpret_cast<const double*>(t->part), t->local, cg, \
                                         t->p, gc, pf, t->ex, t->ey, t->ec, t->es, t->perm,     \
                                         y_user, y_sorted)
  DDM_P_DISPATCH(t->p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

}  // namespace ddm
