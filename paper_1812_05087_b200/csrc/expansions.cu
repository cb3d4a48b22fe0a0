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
// Parent c from its children q (all ready), separable form (fmm.cu):
//   c^q_{n+1} = gamma^q_{n+1} - n conj(e)/s_q alpha^q_n,   e = z_c - z_q
//   xa^q_n = (2 eps_q)^{-(n+1)} alpha^q_{n+1},  xc^q_n = (2 eps_q)^{-(n+1)} c^q_{n+1}
//   alpha^c_{m+1} = sum_q eps_q^{m+1} sum_n C(m, n) xa^q_n     (gamma^c likewise from xc)
// Lane m reads the real Pascal entry C(m, n) (consecutive per lane) and the
// pre-scaled child coefficients (shared-memory broadcasts).
template <int PT>
__device__ void m2m_cell(int c, int p, const int* __restrict__ c_ix, const int* __restrict__ c_iy,
                         const int* __restrict__ first_child, const int* __restrict__ nchild,
                         const double* pasT, const double2* eps, const double2* e2i,
                         double2* __restrict__ mpole, double2* xa, double2* xc, const int* ready,
                         int epoch, int lane) {
  const int f = first_child[c], nc = nchild[c];
  const int pw = p + 2;
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
      const double2* Ei = e2i + quad[i] * pw;
      for (int n = lane; n < p; n += 32) {
        const double2 an = mq[n];
        double2 cv = mq[p + n];
        if (n >= 1) cmac(cv, cscale(eb, -(double)n), mq[n - 1]);
        const double2 sc = Ei[n + 1];
        xa[i * p + n] = cmul(an, sc);
        xc[i * p + n] = cmul(cv, sc);
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
      const double cm = pasT[n * p + m];   // C(m, n)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nc) {
          const double2 x = xa[i * p + n], y = xc[i * p + n];
          a[i].x = fma(x.x, cm, a[i].x);
          a[i].y = fma(x.y, cm, a[i].y);
          g[i].x = fma(y.x, cm, g[i].x);
          g[i].y = fma(y.y, cm, g[i].y);
        }
      }
    }
    double2 sa = make_double2(0.0, 0.0), sg = sa;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < nc) {
        const double2 em = eps[quad[i] * pw + m + 1];
        cmac(sa, a[i], em);
        cmac(sg, g[i], em);
      }
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
              const double* __restrict__ es, const double* __restrict__ pasT_g,
              const double2* __restrict__ eps_g, const double2* __restrict__ e2i_g,
              double2* __restrict__ mpole, int* __restrict__ ready, int epoch,
              int* __restrict__ ticket, PoroFar pf) {
  const int p = PT ? PT : p_rt;
  const int pw = p + 2;
  extern __shared__ double2 up_sh[];
  double2* eps = up_sh;                                       // [4][pw]
  double2* e2i = eps + 4 * pw;                                // [4][pw]
  double* pasT = reinterpret_cast<double*>(e2i + 4 * pw);     // [p][p] C(m,n) at n*p+m
  double2* wbase = e2i + 4 * pw + (p * p + 1) / 2;
  block_copy(eps, eps_g, 4 * pw);
  block_copy(e2i, e2i_g, 4 * pw);
  block_copy(pasT, pasT_g, p * p);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* wb = wbase + (size_t)w * (32 * 17 > 8 * p ? 32 * 17 : 8 * p);
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
      m2m_cell<PT>(c, p, c_ix, c_iy, first_child, nchild, pasT, eps, e2i, mpole, wb, wb + 4 * p,
                   ready, epoch, lane);
    }
    publish(ready + c, epoch, lane);
  }
}

// ------------------------------------------------------------ M2L (a7) + L2L (a8)
// M2L of V pair (target c, source b), delta = (z_c - z_b)/s, w = 1/delta:
//   c_{n+1} = gamma_{n+1} - n conj(delta) alpha_n                 (Psi~ coupling)
//   ap_n = w^{n+1} alpha_{n+1},  cp_n = w^{n+1} c_{n+1}           (pre-scale, lane n)
//   lambda_m += (-w)^m sum_n C(m+n, n) ap_n,  g_m += (-w)^m sum_n C(m+n, n) cp_n
// The real Pascal row C(m+n, n) of lane m is class independent: it lives in
// registers (PT <= 32), so the inner loop reads only the two broadcast
// coefficients per n from shared memory.  Then L2L from the (final) parent P:
//   g'_m = gamma^P_m + (m+1) conj(eps) lambda^P_{m+1},  eps = (z_c - z_P)/s_P
//   lambda^c_k += (2 eps)^{-k} sum_m C(m, k) eps^m lambda^P_m   (gamma^c likewise from g')
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
downward_kernel(int c0, int c1, int64_t own_lo, int64_t own_hi, const int* __restrict__ v_off,
                const int* __restrict__ v_idx, const unsigned char* __restrict__ v_cls,
                const int* __restrict__ c_level, const int* __restrict__ c_ix,
                const int* __restrict__ c_iy, const int* __restrict__ c_start,
                const int* __restrict__ c_count, const int* __restrict__ c_parent, int p_rt,
                const double2* __restrict__ w_g, const double2* __restrict__ eps_g,
                const double2* __restrict__ e2i_g, const double* __restrict__ pas_g,
                const double* __restrict__ pm2l_g, const double2* __restrict__ mpole,
                double2* __restrict__ local, int* __restrict__ ready, int epoch,
                int* __restrict__ ticket) {
  const int p = PT ? PT : p_rt;
  constexpr bool REG = PT > 0 && PT <= 32;   // Pascal row in registers, one output per lane
  constexpr int NCC = REG ? 1 : 2;           // outputs per lane: m = lane + 32 cc
  const int pw = p + 2;
  extern __shared__ double2 dn_sh[];
  double2* sh_w = dn_sh;                                        // [49][pw]
  double2* sh_eps = sh_w + kNOffsets * pw;                      // [4][pw]
  double2* sh_e2i = sh_eps + 4 * pw;                            // [4][pw]
  double* sh_pas = reinterpret_cast<double*>(sh_e2i + 4 * pw);  // [p][p] C(m,k) at m*p+k
  double* sh_pm2l = sh_pas + p * p;                             // [p+1][p] (runtime-p path)
  const int ndbl = p * p + (REG ? 0 : (p + 1) * p);
  double2* wbuf = sh_e2i + 4 * pw + (ndbl + 1) / 2;
  block_copy(sh_w, w_g, kNOffsets * pw);
  block_copy(sh_eps, eps_g, 4 * pw);
  block_copy(sh_e2i, e2i_g, 4 * pw);
  block_copy(sh_pas, pas_g, p * p);
  if (!REG) block_copy(sh_pm2l, pm2l_g, (p + 1) * p);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* sa = wbuf + (size_t)w * (3 * p + 1);      // raw alpha [p]      | eps^m lambda^P [p]
  double2* ap = sa + p;                               // pre-scaled alpha [p] | eps^m g' [p]
  double2* cp = ap + p;                               // pre-scaled c [p+1]
  // lane m's M2L Pascal row C(m+n, n), n = 0..PT (exact integers up to 2^53)
  double prow[REG ? PT + 1 : 1];
  if (REG) {
    double cb = 1.0;
    prow[0] = 1.0;
#pragma unroll
    for (int n = 1; n < (REG ? PT + 1 : 1); ++n) {
      cb = cb * (double)(lane + n) / (double)n;
      prow[n] = cb;
    }
  }
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
    double2 al[NCC], ag[NCC];
#pragma unroll
    for (int cc = 0; cc < NCC; ++cc) al[cc] = ag[cc] = make_double2(0.0, 0.0);
    const int vb = v_off[c], ve = v_off[c + 1];
    double2 na[NCC], ng[NCC];
#pragma unroll
    for (int cc = 0; cc < NCC; ++cc) na[cc] = ng[cc] = make_double2(0.0, 0.0);
    if (vb < ve) {
      const double2* ma = mpole + (size_t)v_idx[vb] * 2 * p;
#pragma unroll
      for (int cc = 0; cc < NCC; ++cc) {
        const int n = lane + 32 * cc;
        if (n < p) {
          na[cc] = ma[n];
          ng[cc] = ma[p + n];
        }
      }
    }
    for (int v = vb; v < ve; ++v) {
      const int cls = v_cls[v];
      double2 xa[NCC], xg[NCC];
#pragma unroll
      for (int cc = 0; cc < NCC; ++cc) {
        xa[cc] = na[cc];
        xg[cc] = ng[cc];
      }
      if (v + 1 < ve) {   // prefetch the next source
        const double2* ma = mpole + (size_t)v_idx[v + 1] * 2 * p;
#pragma unroll
        for (int cc = 0; cc < NCC; ++cc) {
          const int n = lane + 32 * cc;
          if (n < p) {
            na[cc] = ma[n];
            ng[cc] = ma[p + n];
          }
        }
      }
      const int dxs = cls % 7 - 3, dys = cls / 7 - 3;   // source - target in cells
      const double2 dconj = make_double2(-(double)dxs, (double)dys);  // conj(delta)
      const double2* W = sh_w + cls * pw;
#pragma unroll
      for (int cc = 0; cc < NCC; ++cc) {
        const int n = lane + 32 * cc;
        if (n < p) sa[n] = xa[cc];
      }
      __syncwarp();
      // pre-scale (slot n <-> coefficient n + 1); lane p also forms c_{p+1}
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int n = lane + 32 * cc;
        if (n <= p) {
          const bool in = n < p;
          double2 cv = make_double2(0.0, 0.0), av = cv;
          if (in) {
            cv = (cc == 0 || !REG) ? xg[cc < NCC ? cc : 0] : cv;
            av = (cc == 0 || !REG) ? xa[cc < NCC ? cc : 0] : av;
          }
          if (n >= 1) cmac(cv, cscale(dconj, -(double)n), sa[n - 1]);
          const double2 wn = W[n + 1];
          cp[n] = cmul(cv, wn);
          if (in) ap[n] = cmul(av, wn);
        }
      }
      __syncwarp();
#pragma unroll
      for (int cc = 0; cc < NCC; ++cc) {
        const int m = lane + 32 * cc;
        if (m < p) {
          double2 sl = make_double2(0.0, 0.0), sg = sl;
#pragma unroll
          for (int n = 0; n < pmax<PT>(); ++n) {
            if (!PT && n >= p) break;
            const double pc = REG ? prow[REG ? n : 0] : sh_pm2l[n * p + m];
            const double2 a = ap[n], g = cp[n];
            sl.x = fma(a.x, pc, sl.x);
            sl.y = fma(a.y, pc, sl.y);
            sg.x = fma(g.x, pc, sg.x);
            sg.y = fma(g.y, pc, sg.y);
          }
          const double pc = REG ? prow[REG ? PT : 0] : sh_pm2l[p * p + m];
          sg.x = fma(cp[p].x, pc, sg.x);
          sg.y = fma(cp[p].y, pc, sg.y);
          double2 wm = W[m];
          if (m & 1) wm = make_double2(-wm.x, -wm.y);
          cmac(al[cc], sl, wm);
          cmac(ag[cc], sg, wm);
        }
      }
      __syncwarp();
    }
    // L2L from the parent (its local expansion is final once its flag is set)
    if (c_level[c] >= 3) {
      const int P = c_parent[c];
      wait_ready(ready + P, epoch);
      const double2* lp = local + (size_t)P * 2 * p;
      const int xb = c_ix[c] & 1, yb = c_iy[c] & 1;
      const int quad = xb + 2 * yb;
      const double2 epsb = make_double2(0.5 * (xb - 0.5), -0.5 * (yb - 0.5));   // conj(eps)
      const double2* E = sh_eps + quad * pw;
      const double2* Ei = sh_e2i + quad * pw;
      double2* xl = sa;
      double2* xg = ap;
      for (int m = lane; m < p; m += 32) {
        double2 gv = lp[p + m];
        if (m + 1 < p) cmac(gv, cscale(epsb, (double)(m + 1)), lp[m + 1]);
        const double2 em = E[m];
        xl[m] = cmul(lp[m], em);
        xg[m] = cmul(gv, em);
      }
      __syncwarp();
#pragma unroll
      for (int cc = 0; cc < NCC; ++cc) {
        const int k = lane + 32 * cc;
        if (k < p) {
          double2 l = make_double2(0.0, 0.0), g = l;
#pragma unroll
          for (int m = 0; m < pmax<PT>(); ++m) {
            if (!PT && m >= p) break;
            const double pc = sh_pas[m * p + k];   // C(m, k)
            const double2 x = xl[m], y = xg[m];
            l.x = fma(x.x, pc, l.x);
            l.y = fma(x.y, pc, l.y);
            g.x = fma(y.x, pc, g.x);
            g.y = fma(y.y, pc, g.y);
          }
          const double2 ek = Ei[k];
          cmac(al[cc], l, ek);
          cmac(ag[cc], g, ek);
        }
      }
      __syncwarp();
    }
    double2* out = local + (size_t)c * 2 * p;
#pragma unroll
    for (int cc = 0; cc < NCC; ++cc) {
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
  const size_t shm = ((size_t)8 * (p + 2) + (size_t)(p * p + 1) / 2 + (size_t)kPassWarps * wsz) *
                     sizeof(double2);
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
        t->ea, t->ec, t->es, t->op_pasT, t->op_eps, t->op_e2i, t->mpole, t->ready_up, t->epoch, \
        t->tickets, pf);                                                                        \
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
  const bool reg = (p == 8 || p == 12 || p == 16 || p == 20 || p == 24 || p == 28 || p == 32);
  const size_t ndbl = (size_t)p * p + (reg ? 0 : (size_t)(p + 1) * p);
  const size_t shm = ((size_t)(kNOffsets + 8) * (p + 2) + (ndbl + 1) / 2 +
                      (size_t)kPassWarps * (3 * p + 1)) * sizeof(double2);
  int rc = DDM_OK;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if ((rc = set_smem(ctx, downward_kernel<PT>, shm))) return rc;                              \
    const int nb = pass_grid(ctx, (const void*)downward_kernel<PT>, shm, c1 - c0);              \
    downward_kernel<PT><<<nb, kPassWarps * 32, shm, s>>>(                                       \
        c0, c1, t->own_el_lo, t->own_el_hi, t->v_off, t->v_idx, t->v_cls, t->c_level, t->c_ix,  \
        t->c_iy, t->c_start, t->c_count, t->c_parent, p, t->op_w, t->op_eps, t->op_e2i,         \
        t->op_pas, t->op_pm2l, t->mpole, t->local, t->ready_down, t->epoch, t->tickets + 1);    \
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
