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
// Scheduling: P2M (warp per leaf) and M2L (warp per cell)
// have no dependencies and run as plain grids; M2M and L2L are launched one
// tree level at a time (M2M deepest level first, L2L top-down), so every
// dependency is a kernel boundary: no flags, no atomics, no spinning.  On the
// high-priority stream these short launches interleave with the concurrent
// near field (fmm.cu).
//
// Every kernel is a template on the expansion order PT (PT = 0: runtime p) so
// that, for the instantiated orders, inner loops unroll and loads pipeline.
#include <algorithm>
#include <functional>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

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
    case 30: F(30); break;                \
    case 32: F(32); break;                \
    default: F(0); break;                 \
  }

template <int PT>
__host__ __device__ constexpr int pmax() { return PT ? PT : kMaxP; }

constexpr int kPassWarps = 8;

// Programmatic dependent launch (sm_90+): a far-chain kernel is launched with
// programmatic stream serialisation, so its blocks are scheduled once every
// block of the previous kernel has started (that kernel triggers at entry);
// it waits for the previous kernel's results (griddepcontrol.wait) only where
// it first reads them, after any prologue that does not depend on them.
// Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }


// ------------------------------------------------------------ P2M (a5)
// Warp per RUN of consecutive whole leaves.  A leaf's
// elements are cut into half-blocks of 16 (rows [16h, 16h + 16) from the leaf
// start); the run's half-blocks are processed two per 32-lane round (lane
// slot = lane / 16), so a leaf of 40 elements takes 3 half-block slots
// instead of two full rounds.  Each lane uses its own leaf's centre and scale.
//   alpha_n = (B/s) P_{n-1}
//   gamma_n = (1/s)[Q P_{n-1} + B((n-1) A P_{n-2} + (n-2) r P_{n-1})]
// zeta_{1,2} = (z_{1,2} - z0)/s, P_m = zeta2^m - zeta1^m, A = conj(zc - z0)/s - r (zc - z0)/s.
// Coefficients are produced in chunks of 8 and summed over each half-block
// through a padded [32][17] shared-memory transpose; a leaf's moments are
// then (((h_0 + h_1) + h_2) + ...) in half-block order -- the same bits
// whatever run the leaf is in (replicated vs sharded upward pass).
#ifndef DDM_P2M_PREFETCH
#define DDM_P2M_PREFETCH 0
#endif
__device__ __forceinline__ void prefetch_l1(const void* a) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
}
template <int PT>
__device__ void p2m_run(int kk0, int nseg, int p, const int* __restrict__ leaves,
                        const int* __restrict__ c_level, const int* __restrict__ c_ix,
                        const int* __restrict__ c_iy, const int* __restrict__ c_start,
                        const int* __restrict__ c_count, const CellGeom& cg,
                        const int* __restrict__ perm, const double* __restrict__ D, int ncomp,
                        const double* __restrict__ ex, const double* __restrict__ ey,
                        const double* __restrict__ ea, const double* __restrict__ ec,
                        const double* __restrict__ es, double2* __restrict__ mpole, double2* buf,
                        int lane, const PoroFar& pf) {
  constexpr int NCH = (pmax<PT>() + 7) / 8;
  const int nchunk = (p + 7) / 8;
  const unsigned full = 0xffffffffu;
  // segment table, one leaf per lane (lanes < nseg); sg_h0 = the leaf's
  // first half-block in the run
  int sg_c = 0, sg_start = 0, sg_cnt = 0, sg_lev = 0, sg_ix = 0, sg_iy = 0, sg_nh = 0;
  if (lane < nseg) {
    sg_c = leaves[kk0 + lane];
    sg_start = c_start[sg_c];
    sg_cnt = c_count[sg_c];
    sg_lev = c_level[sg_c];
    sg_ix = c_ix[sg_c];
    sg_iy = c_iy[sg_c];
    sg_nh = (sg_cnt + 15) >> 4;
  }
  int sg_h0 = sg_nh;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(full, sg_h0, o);
    if (lane >= o) sg_h0 += v;
  }
  const int NH = __shfl_sync(full, sg_h0, 31);   // half-blocks of the run
  sg_h0 -= sg_nh;
  if (lane < nseg && sg_cnt == 0)   // an empty leaf (no half-block): zero moments
    for (int m = 0; m < 2 * p; ++m) mpole[(size_t)sg_c * 2 * p + m] = make_double2(0.0, 0.0);
  // lane < 16 owns column `lane` of every chunk (the running sum of the open
  // leaf): column j < 8 -> alpha slot 8 ch + j, column j >= 8 -> gamma slot 8 ch + j - 8
  double2 acc[NCH];
#pragma unroll
  for (int q = 0; q < NCH; ++q) acc[q] = make_double2(0.0, 0.0);
  const int slot2 = lane >> 4, row16 = lane & 15;
  for (int hb0 = 0; hb0 < NH; hb0 += 2) {
    const int hb = hb0 + slot2;
    // this lane's leaf: the last segment with sg_h0 <= hb
    int seg = 0;
    for (int q = 1; q < nseg; ++q)
      if (hb >= __shfl_sync(full, sg_h0, q)) seg = q;
    const int s_start = __shfl_sync(full, sg_start, seg);
    const int s_cnt = __shfl_sync(full, sg_cnt, seg);
    const int row = 16 * (hb - __shfl_sync(full, sg_h0, seg)) + row16;
    const bool valid = hb < NH && row < s_cnt;
    const int i = s_start + row;
    const int lev = __shfl_sync(full, sg_lev, seg);
    const double s = cg.side(lev);
    const double is = 1.0 / s;
    const double2 z0 = cg.centre(lev, __shfl_sync(full, sg_ix, seg), __shfl_sync(full, sg_iy, seg));
    // rows of each slot's half-block, and whether it ends its leaf
    const int nrow = hb < NH ? min(16, s_cnt - (row - row16)) : 0;
    const bool closes = hb < NH && (row - row16) + 16 >= s_cnt;
#if DDM_P2M_PREFETCH
    // next round's rows (half-blocks hb + 2): their geometry lines are asked
    // for now and the user index is held, so D can be asked for once it has
    // arrived (after this round's arithmetic).  Hints only: no result changes.
    int jn = -1;
    {
      const int hb2 = hb + 2;
      int seg2 = 0;
      for (int q = 1; q < nseg; ++q)
        if (hb2 >= __shfl_sync(full, sg_h0, q)) seg2 = q;
      const int row2 = 16 * (hb2 - __shfl_sync(full, sg_h0, seg2)) + row16;
      const int i2 = __shfl_sync(full, sg_start, seg2) + row2;
      const int cnt2 = __shfl_sync(full, sg_cnt, seg2);
      if (hb2 < NH && row2 < cnt2) {
        prefetch_l1(ex + i2);
        prefetch_l1(ey + i2);
        prefetch_l1(ea + i2);
        prefetch_l1(ec + i2);
        prefetch_l1(es + i2);
        jn = perm ? perm[i2] : i2;
      }
    }
#endif
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
        const double mu = pf.lin ? 0.0 : -(pf.eta / pf.S) * dn;
        const double wm = (pf.eta * mu / M_PI + pf.eta * qf * pf.ct / (M_PI * pf.kappa)) / pf.gc;
        // (wm / i) conj(e) / s, and 48 eta k_p c tau B / s^3
        Wme = cscale(cmul(make_double2(0.0, -wm), make_double2(cb, -sb)), is);
        Bc = cscale(B, 48.0 * pf.eta * pf.kp * pf.ct * is * is * is);
        fu = pf.fu;
        if (pf.lin) {   // tau-linear part only: no Phi series, no drained Psi terms
          fu = 0.0;
          Q = make_double2(0.0, 0.0);
        }
      }
      B = cscale(B, is);
      Q = cscale(Q, is);
    }
    // the two slots' leaves, row counts and closing flags, at lanes < 16
    const int cA = __shfl_sync(full, sg_c, __shfl_sync(full, seg, 0));
    const int cB = __shfl_sync(full, sg_c, __shfl_sync(full, seg, 16));
    const int nA = __shfl_sync(full, nrow, 0), nB = __shfl_sync(full, nrow, 16);
    const bool clA = __shfl_sync(full, closes, 0), clB = __shfl_sync(full, closes, 16);
    // per-element weights of the power sums (elastic: fu = 1, Wme = Bc = 0):
    //   alpha_n = ub P_{n-1},  gamma_n = y_n P_{n-1} + (n-1) x P_{n-2} [+ Bc (n-1)(n-2)/6 P_{n-3}]
    //   ub = fu B, wr = fu B r, x = fu B A, y_n = Q + (n-2) wr + Wme (y_1 = Q - wr + Wme)
    const double2 ub = cscale(B, fu);
    const double2 wr = cmul(ub, rr);
    const double2 xw = cmul(ub, A);
    double2 yn = cadd(csub(Q, wr), Wme);
    double2 xn = make_double2(0.0, 0.0);     // (n-1) x
    double2 pw1 = make_double2(1.0, 0.0), pw2 = pw1;
    double2 Pm2 = make_double2(0.0, 0.0);   // P_{n-3}
    double2 Pm1 = make_double2(0.0, 0.0);   // P_{n-2}
    double2 Pm = make_double2(0.0, 0.0);    // P_{n-1}
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
            alpha = cmul(ub, Pm);
            gam = cmul(yn, Pm);
            cmac(gam, xn, Pm1);
            if (pf.on && n >= 4) cmac(gam, cscale(Bc, (n - 1) * (n - 2) / 6.0), Pm2);
            yn = cadd(yn, wr);
            xn = cadd(xn, xw);
          }
          buf[lane * 17 + j] = alpha;
          buf[lane * 17 + 8 + j] = gam;
        }
        __syncwarp();
        // column row16 of half-block slot2: rows 16 slot2 + [0, nrow)
        double2 sum = make_double2(0.0, 0.0);
        for (int e = 0; e < nrow; ++e) sum = cadd(sum, buf[(16 * slot2 + e) * 17 + row16]);
        double2 sB;
        sB.x = __shfl_down_sync(full, sum.x, 16);
        sB.y = __shfl_down_sync(full, sum.y, 16);
        const int slot = 8 * ch + (lane & 7);
        if (lane < 16) {
          const int off = (lane < 8 ? 0 : p) + slot;
          if (nA > 0) {
            acc[ch] = cadd(acc[ch], sum);
            if (clA) {
              if (slot < p) mpole[(size_t)cA * 2 * p + off] = acc[ch];
              acc[ch] = make_double2(0.0, 0.0);
            }
          }
          if (nB > 0) {
            acc[ch] = cadd(acc[ch], sB);
            if (clB) {
              if (slot < p) mpole[(size_t)cB * 2 * p + off] = acc[ch];
              acc[ch] = make_double2(0.0, 0.0);
            }
          }
        }
        __syncwarp();
#if DDM_P2M_PREFETCH
        if (ch == 0 && jn >= 0) prefetch_l1(D + (int64_t)jn * ncomp);
#endif
      }
    }
  }
}

// Tree-static part of a parent's M2M (loaded before the PDL wait where the
// launch allows it): the cell, its children and their quadrants.
struct M2MStatic {
  int c, f, nc;
  int quad[4];
};
__device__ __forceinline__ M2MStatic m2m_static(int c, const int* __restrict__ c_ix,
                                                const int* __restrict__ c_iy,
                                                const int* __restrict__ first_child,
                                                const int* __restrict__ nchild) {
  M2MStatic st;
  st.c = c;
  st.f = first_child[c];
  st.nc = nchild[c];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = st.f + min(i, st.nc - 1);
    st.quad[i] = (c_ix[q] & 1) + 2 * (c_iy[q] & 1);
  }
  return st;
}

// The operator tables of the M2M / L2L passes staged in shared memory by the
// whole CTA (before the PDL wait): the real Pascal matrix [p][p] and the
// quadrant powers eps^k, (2 eps)^-k [4][p + 2]; tbl_doubles() = their size.
__host__ __device__ __forceinline__ int tbl_pas(int p) { return (p * p + 1) & ~1; }
__host__ __device__ __forceinline__ int tbl_doubles(int p) { return tbl_pas(p) + 16 * (p + 2); }
struct OpTables {
  const double* pas;    // pasT (M2M: C(m, n) at n p + m) or pas (L2L: C(m, k) at m p + k)
  const double2* eps;   // [4][p + 2]
  const double2* e2i;   // [4][p + 2]
};
__device__ __forceinline__ OpTables stage_tables(double* sh, int p, const double* __restrict__ pas_g,
                                                 const double2* __restrict__ eps_g,
                                                 const double2* __restrict__ e2i_g) {
  const int np = tbl_pas(p), pw4 = 4 * (p + 2);
  double2* e = reinterpret_cast<double2*>(sh + np);
  for (int i = threadIdx.x; i < p * p; i += blockDim.x) sh[i] = pas_g[i];
  for (int i = threadIdx.x; i < pw4; i += blockDim.x) {
    e[i] = eps_g[i];
    e[pw4 + i] = e2i_g[i];
  }
  return OpTables{sh, e, e + pw4};
}

// ------------------------------------------------------------ M2M (a6)
// Parent c from its children q (all ready), separable form (fmm.cu):
//   c^q_{n+1} = gamma^q_{n+1} - n conj(e)/s_q alpha^q_n,   e = z_c - z_q
//   xa^q_n = (2 eps_q)^{-(n+1)} alpha^q_{n+1},  xc^q_n = (2 eps_q)^{-(n+1)} c^q_{n+1}
//   alpha^c_{m+1} = sum_q eps_q^{m+1} sum_n C(m, n) xa^q_n     (gamma^c likewise from xc)
// Lane m reads the real Pascal entry C(m, n) (consecutive per lane) and the
// pre-scaled child coefficients (shared-memory broadcasts); the operator
// tables are in shared memory (stage_tables), so after the children's loads
// the cell's chain has no global round trip.
template <int PT>
__device__ void m2m_cell(const M2MStatic& st, int p, const OpTables& T,
                         double2* __restrict__ mpole, double2* xa, double2* xc, int lane) {
  const int f = st.f, nc = st.nc;
  const int pw = p + 2;
  constexpr int NC = PT ? (PT + 31) / 32 : 2;   // coefficients per lane
  // all children's coefficients in flight at once (lane n: slots n, n-1 of both series)
  double2 an[4][NC], gn[4][NC], ap[4][NC];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int q = f + min(i, nc - 1);
    const double2* mq = mpole + (size_t)q * 2 * p;
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
      const int n = lane + 32 * cc;
      const bool ok = i < nc && n < p;
      an[i][cc] = ok ? mq[n] : make_double2(0.0, 0.0);
      gn[i][cc] = ok ? mq[p + n] : make_double2(0.0, 0.0);
      ap[i][cc] = (ok && n >= 1) ? mq[n - 1] : make_double2(0.0, 0.0);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (i < nc) {
      const int xb = st.quad[i] & 1, yb = st.quad[i] >> 1;
      const double2 eb = make_double2(-(xb - 0.5), (yb - 0.5));   // conj(e)/s_q
      const double2* Ei = T.e2i + st.quad[i] * pw;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int n = lane + 32 * cc;
        if (n < p) {
          double2 cv = gn[i][cc];
          cmac(cv, cscale(eb, -(double)n), ap[i][cc]);
          const double2 sc = Ei[n + 1];
          xa[i * p + n] = cmul(an[i][cc], sc);
          xc[i * p + n] = cmul(cv, sc);
        }
      }
    }
  }
  __syncwarp();
  double2* out = mpole + (size_t)st.c * 2 * p;
  for (int m = lane; m < p; m += 32) {
    double2 a[4], g[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = g[i] = make_double2(0.0, 0.0);
#pragma unroll
    for (int n = 0; n < pmax<PT>(); ++n) {
      if (!PT && n >= p) break;
      const double cm = T.pas[n * p + m];   // C(m, n)
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
        const double2 em = T.eps[st.quad[i] * pw + m + 1];
        cmac(sa, a[i], em);
        cmac(sg, g[i], em);
      }
    }
    out[m] = sa;
    out[p + m] = sg;
  }
  __syncwarp();
}

// P2M of every leaf: no dependencies, warp per leaf (grid-stride).
#ifndef DDM_P2M_MINB
#define DDM_P2M_MINB 0
#endif
#if DDM_P2M_MINB > 0
#define DDM_P2M_BOUNDS __launch_bounds__(kPassWarps * 32, DDM_P2M_MINB)
#else
#define DDM_P2M_BOUNDS __launch_bounds__(kPassWarps * 32)
#endif
template <int PT>
__global__ void DDM_P2M_BOUNDS
p2m_kernel(int nruns, const int2* __restrict__ runs, const int* __restrict__ leaves,
           const int* __restrict__ c_level,
           const int* __restrict__ c_ix, const int* __restrict__ c_iy,
           const int* __restrict__ c_start, const int* __restrict__ c_count, CellGeom cg,
           int p_rt, const int* __restrict__ perm, const double* __restrict__ D, int ncomp,
           const double* __restrict__ ex,
           const double* __restrict__ ey, const double* __restrict__ ea,
           const double* __restrict__ ec, const double* __restrict__ es,
           double2* __restrict__ mpole, PoroFar pf) {
  const int p = PT ? PT : p_rt;
  pdl_trigger();
  extern __shared__ double2 p2m_sh[];   // [kPassWarps][32 * 17] transposition buffers
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = blockIdx.x * kPassWarps + w; k < nruns; k += gridDim.x * kPassWarps) {
    const int2 rn = runs[k];   // (first leaf, leaves)
    p2m_run<PT>(rn.x, rn.y, p, leaves, c_level, c_ix, c_iy, c_start, c_count, cg, perm, D, ncomp,
                ex, ey, ea, ec, es, mpole, p2m_sh + w * 32 * 17, lane, pf);
  }
}

// ------------------------------------------------------------ P2L (f3, X lists)
// Warp per owned target leaf B with a nonempty X list (tree.cu
// x_count): the elements of B's X leaves (coarser, not touching B) are
// expanded into B's local series about z0 = B's centre, written to
// local_x[k] and added to B's local by the L2P.  In P2M's notation (zeta_1,2
// the element's nodes, normalised by B's centre and side s; ub = B/s, wr = ub
// r, x = ub A, Q), the element's fields are the rational functions
//   Phi(t)  = ub sum_k sig_k / (t - zeta_k)
//   Psi~(t) = sum_k sig_k [(Q - wr)/(t - zeta_k) + (wr zeta_k + x)/(t - zeta_k)^2]
// (sig = +1 at zeta_2, -1 at zeta_1: their Laurent coefficients are exactly
// P2M's alpha_n and gamma_n), and with u_k = 1/zeta_k, R_j = u_2^j - u_1^j the
// Taylor coefficients about t = 0 (|t| < |zeta_k|: B's targets are closer to
// z0 than any node of a non-touching leaf) are
//   l^Phi_m  = -ub R_{m+1}
//   l^Psi~_m = (-Q + (m + 2) wr) R_{m+1} + (m + 1) x R_{m+2}.
// Lanes take the concatenated X elements 32 at a time; coefficient chunks of 8
// are summed over the 32 rows through the [32][17] transpose of P2M, rounds
// in order: deterministic.  Elastic only (the poroelastic paths keep U whole).
#ifndef DDM_P2L_MINB
#define DDM_P2L_MINB 1
#endif
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32, DDM_P2L_MINB)
p2l_kernel(int k_lo, int k_hi, const int* __restrict__ x_off, const int* __restrict__ x_idx,
           const int* __restrict__ leaves, const int* __restrict__ c_level,
           const int* __restrict__ c_ix, const int* __restrict__ c_iy,
           const int* __restrict__ c_start, const int* __restrict__ c_count, CellGeom cg, int p_rt,
           const int* __restrict__ perm, const double* __restrict__ D, int ncomp,
           const double* __restrict__ ex, const double* __restrict__ ey,
           const double* __restrict__ ea, const double* __restrict__ ec,
           const double* __restrict__ es, double2* __restrict__ local_x) {
  const int p = PT ? PT : p_rt;
  constexpr int NCH = (pmax<PT>() + 7) / 8;
  const int nchunk = (p + 7) / 8;
  const unsigned full = 0xffffffffu;
  extern __shared__ double2 p2m_sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* buf = p2m_sh + w * 32 * 17;
  for (int k = k_lo + blockIdx.x * kPassWarps + w; k < k_hi; k += gridDim.x * kPassWarps) {
    const int x0 = __ldg(x_off + k), x1 = __ldg(x_off + k + 1);
    if (x1 <= x0) continue;
    const int c = __ldg(leaves + k);
    const int lev = __ldg(c_level + c);
    const double s = cg.side(lev);
    const double is = 1.0 / s;
    const double2 z0 = cg.centre(lev, __ldg(c_ix + c), __ldg(c_iy + c));
    double2 acc[NCH];
#pragma unroll
    for (int q = 0; q < NCH; ++q) acc[q] = make_double2(0.0, 0.0);
    // X leaves in batches of 32: lane j holds leaf x0 + j's start and the
    // inclusive prefix of the element counts
    for (int xb = x0; xb < x1; xb += 32) {
      const int nb = min(32, x1 - xb);
      int ls = 0, lc = 0;
      if (lane < nb) {
        const int A = __ldg(x_idx + xb + lane);
        ls = __ldg(c_start + A);
        lc = __ldg(c_count + A);
      }
      int pre = lc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(full, pre, o);
        if (lane >= o) pre += v;
      }
      const int NE = __shfl_sync(full, pre, 31);
      for (int e0 = 0; e0 < NE; e0 += 32) {
        const int f = e0 + lane;
        // this lane's X leaf: the first with inclusive prefix > f
        int seg = 0;
        for (int q = 0; q < nb; ++q)
          if (__shfl_sync(full, pre, q) <= f) seg = q + 1;
        const bool valid = f < NE;
        seg = min(seg, nb - 1);
        const int sstart = __shfl_sync(full, ls, seg);
        const int sexcl = __shfl_sync(full, pre - lc, seg);
        double2 ub = make_double2(0, 0), Q = ub, wr = ub, xw = ub;
        double2 u1 = make_double2(1.0, 0.0), u2 = u1;
        if (valid) {
          const int i = sstart + (f - sexcl);
          const int j = perm ? perm[i] : i;
          const double ds = D[(int64_t)j * ncomp], dn = D[(int64_t)j * ncomp + 1];
          const double cb = ec[i], sb = es[i], a = ea[i];
          double2 B = make_double2(ds * cb - dn * sb, ds * sb + dn * cb);
          const double2 rr = make_double2(cb * cb - sb * sb, -2.0 * cb * sb);
          Q = cscale(csub(cmul(rr, B), cconj(B)), is);
          const double2 d = make_double2((ex[i] - z0.x) * is, (ey[i] - z0.y) * is);
          const double2 A = csub(cconj(d), cmul(rr, d));
          const double2 z1 = make_double2(d.x - a * cb * is, d.y - a * sb * is);
          const double2 z2 = make_double2(d.x + a * cb * is, d.y + a * sb * is);
          ub = cscale(B, is);
          wr = cmul(ub, rr);
          xw = cmul(ub, A);
          const double n1 = 1.0 / fma(z1.x, z1.x, z1.y * z1.y);
          const double n2 = 1.0 / fma(z2.x, z2.x, z2.y * z2.y);
          u1 = make_double2(z1.x * n1, -z1.y * n1);
          u2 = make_double2(z2.x * n2, -z2.y * n2);
        }
        const double2 nub = make_double2(-ub.x, -ub.y);
        double2 yv = csub(cscale(wr, 2.0), Q);   // -Q + (m + 2) wr at m = 0
        double2 xm = xw;                          // (m + 1) x at m = 0
        double2 pw1 = u1, pw2 = u2;
        double2 Ra = csub(u2, u1);                // R_{m+1}
        pw1 = cmul(pw1, u1);
        pw2 = cmul(pw2, u2);
        double2 Rb = csub(pw2, pw1);              // R_{m+2}
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          if (ch < nchunk) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int m = 8 * ch + jj;
              double2 lphi = make_double2(0.0, 0.0), lpsi = lphi;
              if (m < p) {
                lphi = cmul(nub, Ra);
                lpsi = cmul(yv, Ra);
                cmac(lpsi, xm, Rb);
                yv = cadd(yv, wr);
                xm = cadd(xm, xw);
                Ra = Rb;
                pw1 = cmul(pw1, u1);
                pw2 = cmul(pw2, u2);
                Rb = csub(pw2, pw1);
              }
              buf[lane * 17 + jj] = lphi;
              buf[lane * 17 + 8 + jj] = lpsi;
            }
            __syncwarp();
            if (lane < 16) {
              double2 sum = make_double2(0.0, 0.0);
#pragma unroll 8
              for (int r = 0; r < 32; ++r) sum = cadd(sum, buf[r * 17 + lane]);
              acc[ch] = cadd(acc[ch], sum);
            }
            __syncwarp();
          }
        }
      }
    }
    if (lane < 16) {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int slot = 8 * ch + (lane & 7);
        if (ch < nchunk && slot < p)
          local_x[(size_t)k * 2 * p + (lane < 8 ? 0 : p) + slot] = acc[ch];
      }
    }
  }
}

// M2M of the non-leaf cells up_list[u0, u1) of ONE level (launched deepest
// level first: every child is final when its parent's level runs).
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
m2m_level_kernel(int u0, int u1, const int* __restrict__ up_list, const int* __restrict__ c_ix,
                 const int* __restrict__ c_iy, const int* __restrict__ first_child,
                 const int* __restrict__ nchild, int p_rt, const double* __restrict__ pasT_g,
                 const double2* __restrict__ eps_g, const double2* __restrict__ e2i_g,
                 double2* __restrict__ mpole) {
  const int p = PT ? PT : p_rt;
  pdl_trigger();
  // tables | per warp: pre-scaled children [2][4][p]
  extern __shared__ double2 up_sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* wb = up_sh + tbl_doubles(p) / 2 + (size_t)w * 8 * p;
  // tree-static data first (operator tables, this warp's first parent and
  // its children), then wait for the children's multipoles (previous level
  // / P2M): with PDL only the coefficient loads follow the wait
  const OpTables T = stage_tables(reinterpret_cast<double*>(up_sh), p, pasT_g, eps_g, e2i_g);
  int k = u0 + blockIdx.x * kPassWarps + w;
  M2MStatic st{};
  if (k < u1) st = m2m_static(up_list[k], c_ix, c_iy, first_child, nchild);
  __syncthreads();
  pdl_wait();
  for (; k < u1; k += gridDim.x * kPassWarps) {
    if (k != u0 + blockIdx.x * kPassWarps + w) st = m2m_static(up_list[k], c_ix, c_iy, first_child, nchild);
    m2m_cell<PT>(st, p, T, mpole, wb, wb + 4 * p, lane);
  }
}

// ------------------------------------------------------------ M2L (a7) + L2L (a8)
// M2L of V pair (target c, source b), delta = (z_c - z_b)/s, w = 1/delta:
//   c_{n+1} = gamma_{n+1} - n conj(delta) alpha_n                 (Psi~ coupling)
//   ap_n = w^{n+1} alpha_{n+1},  cp_n = w^{n+1} c_{n+1}           (pre-scale)
//   lambda_m += (-w)^m sum_n C(m+n, n) ap_n,  g_m += (-w)^m sum_n C(m+n, n) cp_n
// The Pascal matrix C(m+n, n) is the same for every pair and offset class, so
// the middle step is one real GEMM per target cell:
//   Y[m][col] = sum_n P[m][n] X[n][col],  col = 4 v + (ap.re, ap.im, cp.re, cp.im)
// run on the fp64 tensor pipe (mma.sync m8n8k4 f64 = DMMA.8x8x4: same fp64 peak
// as DFMA on B200, scripts/micro/dmma.cu, at 1/8 of the issued instructions).
// Then L2L from the (final) parent P:
//   g'_m = gamma^P_m + (m+1) conj(eps) lambda^P_{m+1},  eps = (z_c - z_P)/s_P
//   lambda^c_k += (2 eps)^{-k} sum_m C(m, k) eps^m lambda^P_m   (gamma^c likewise from g')

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

#ifndef DDM_M2L_BATCH
#define DDM_M2L_BATCH 4
#endif
constexpr int kM2LBatch = DDM_M2L_BATCH;   // V pairs per pipelined batch (2 pairs per DMMA n-tile)

// Tensor-core M2L of cell c's V list [vb, ve) (PT <= 32).  Per batch of
// kM2LBatch pairs: (1) every lane loads the source coefficients of its
// ceil(batch x KB / 32) (pair, n) items at once (all loads in flight), then
// writes the pre-scaled X[col][n] (col = 4 pair + (ap.re, ap.im, cp.re,
// cp.im)); (2) the warp runs Y = P X on DMMA (two pairs = one 8-column
// n-tile) and post-scales.  Lane l owns output rows m = 8 i + l/4 of series
// (l%4)%2 for pair parity (l%4)/2; the parities are summed at the end.
// Results go to out_l[m], out_g[m] (m < p).
// conj(delta) of the 49 offset classes, delta = -(dx + i dy) (fmm.cu), i.e.
// conj(delta) = (-dx, dy) with dx = o % 7 - 3, dy = o / 7 - 3
__constant__ double2 c_dconj[kNOffsets] = {
#define DDM_DC(o) {-(double)((o) % 7 - 3), (double)((o) / 7 - 3)}
    DDM_DC(0), DDM_DC(1), DDM_DC(2), DDM_DC(3), DDM_DC(4), DDM_DC(5), DDM_DC(6),
    DDM_DC(7), DDM_DC(8), DDM_DC(9), DDM_DC(10), DDM_DC(11), DDM_DC(12), DDM_DC(13),
    DDM_DC(14), DDM_DC(15), DDM_DC(16), DDM_DC(17), DDM_DC(18), DDM_DC(19), DDM_DC(20),
    DDM_DC(21), DDM_DC(22), DDM_DC(23), DDM_DC(24), DDM_DC(25), DDM_DC(26), DDM_DC(27),
    DDM_DC(28), DDM_DC(29), DDM_DC(30), DDM_DC(31), DDM_DC(32), DDM_DC(33), DDM_DC(34),
    DDM_DC(35), DDM_DC(36), DDM_DC(37), DDM_DC(38), DDM_DC(39), DDM_DC(40), DDM_DC(41),
    DDM_DC(42), DDM_DC(43), DDM_DC(44), DDM_DC(45), DDM_DC(46), DDM_DC(47), DDM_DC(48)
#undef DDM_DC
};

constexpr int kXStride = 36;   // doubles per X column (>= p+1; = 4 mod 16: conflict-free fragments)

template <int PT>
__device__ void m2l_cell_tc(int vb, int ve, const int* __restrict__ v_idx,
                            const unsigned char* __restrict__ v_cls,
                            const double2* __restrict__ mpole, const double2* __restrict__ w_g,
                            const double* sh_afr, double* X, double2* out_l, double2* out_g,
                            int lane, int sub = 0, int S = 1) {
  constexpr int p = PT, pw = PT + 2, P2 = 2 * PT;
  constexpr int MT = (PT + 7) / 8, KS = (PT + 4) / 4, KB = 4 * KS;
  double2 acc[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) acc[i] = make_double2(0.0, 0.0);
  const int q = lane >> 2, j = lane & 3;
  for (int vc = vb; vc < ve; vc += 32) {   // V lists hold <= 27 entries
    const int K = min(32, ve - vc);
    int my_src = 0, my_cls = 0;
    if (lane < K) {
      my_src = v_idx[vc + lane];
      my_cls = v_cls[vc + lane];
    }
    // S warps share the cell: warp `sub` takes batches sub, sub + S, ...
    for (int b0 = sub * kM2LBatch; b0 < K; b0 += S * kM2LBatch) {
      const int nb = min(kM2LBatch, K - b0);
      // phase 1: lane n (rounds of 32 over n < KB) loads slots n, n-1 of every
      // pair of the batch at once (coalesced across lanes), then writes the
      // pre-scaled X[4 v + comp][n]
      constexpr int NR = (KB + 31) / 32;
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        const int n = lane + 32 * rr;
        // lane constants: which of slots n, n-1 exist; -n as a double
        const bool in_a = n < p, in_p = n >= 1 && n <= p, in_w = n <= p;
        const int na_ = in_a ? n : 0, np_ = in_p ? n - 1 : 0, nw_ = in_w ? n + 1 : 0;
        const double mn = -(double)n;
        double2 ra[kM2LBatch], rg[kM2LBatch], rp[kM2LBatch], rw[kM2LBatch], dc[kM2LBatch];
#pragma unroll
        for (int v = 0; v < kM2LBatch; ++v) {
          const int src = __shfl_sync(0xffffffffu, my_src, (b0 + v) & 31);
          const int cl = __shfl_sync(0xffffffffu, my_cls, (b0 + v) & 31);
          const double2* ma = mpole + (size_t)src * P2;   // src = 0 for v >= nb: valid memory
          ra[v] = __ldg(ma + na_);
          rg[v] = __ldg(ma + p + na_);
          rp[v] = __ldg(ma + np_);
          rw[v] = __ldg(w_g + cl * pw + nw_);
          dc[v] = c_dconj[cl];   // conj(delta) of the class (constant-cache broadcast)
        }
        if (n < KB) {
          const double2 z = make_double2(0.0, 0.0);
#pragma unroll
          for (int v = 0; v < kM2LBatch; ++v) {
            const bool ok = v < nb;
            const double2 wv = (ok && in_w) ? rw[v] : z;
            const double2 av = in_a ? cmul(ra[v], wv) : z;
            double2 cv = in_a ? rg[v] : z;
            if (in_p) cmac(cv, cscale(dc[v], mn), rp[v]);
            cv = cmul(cv, wv);
            double* xc = X + (size_t)(4 * v) * kXStride + n;
            xc[0] = av.x;
            xc[kXStride] = av.y;
            xc[2 * kXStride] = cv.x;
            xc[3 * kXStride] = cv.y;
          }
        }
      }
      __syncwarp();
      // phase 2: Y = P X on DMMA, two pairs (8 columns) per n-tile; post-scale
      for (int t = 0; t < (nb + 1) >> 1; ++t) {
        double d[MT][2];
#pragma unroll
        for (int i = 0; i < MT; ++i) d[i][0] = d[i][1] = 0.0;
        const double* xb = X + (size_t)(8 * t + q) * kXStride + j;
#pragma unroll
        for (int sk = 0; sk < KS; ++sk) {
          const double bv = xb[4 * sk];
#pragma unroll
          for (int i = 0; i < MT; ++i)
            dmma_884(d[i][0], d[i][1], sh_afr[(i * KS + sk) * 32 + lane], bv);
        }
        // lane holds rows m = 8 i + q, columns 8 t + 2 j + {0, 1}: pair 2 t + j/2,
        // series j % 2, (re, im)
        const int vloc = 2 * t + (j >> 1);
        const int cls = __shfl_sync(0xffffffffu, my_cls, (b0 + vloc) & 31);
        if (vloc < nb) {
#pragma unroll
          for (int i = 0; i < MT; ++i) {
            const int m = 8 * i + q;
            double2 wm = __ldg(w_g + cls * pw + min(m, p));
            if (m & 1) wm = make_double2(-wm.x, -wm.y);
            cmac(acc[i], make_double2(d[i][0], d[i][1]), wm);
          }
        }
      }
      __syncwarp();
    }
  }
  // sum the two pair parities (lanes l and l ^ 2), lanes with j < 2 write
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, 2);
    acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, 2);
    const int m = 8 * i + q;
    if (j < 2 && m < p) (j == 0 ? out_l : out_g)[m] = acc[i];
  }
}

// Runtime-p fallback M2L (DFMA, lane = m, Pascal entries from shared memory).
__device__ void m2l_cell_dfma(int p, int vb, int ve, const int* __restrict__ v_idx,
                              const unsigned char* __restrict__ v_cls,
                              const double2* __restrict__ mpole, const double2* sh_w,
                              const double* sh_pm2l, double2* sa, double2* ap, double2* cp,
                              double2* out_l, double2* out_g, int lane) {
  const int pw = p + 2;
  double2 al[2], ag[2];
  al[0] = al[1] = ag[0] = ag[1] = make_double2(0.0, 0.0);
  for (int v = vb; v < ve; ++v) {
    const int cls = v_cls[v];
    const double2* ma = mpole + (size_t)v_idx[v] * 2 * p;
    const int dxs = cls % 7 - 3, dys = cls / 7 - 3;
    const double2 dconj = make_double2(-(double)dxs, (double)dys);
    const double2* W = sh_w + cls * pw;
    for (int n = lane; n < p; n += 32) sa[n] = ma[n];
    __syncwarp();
    for (int n = lane; n <= p; n += 32) {
      double2 cv = n < p ? ma[p + n] : make_double2(0.0, 0.0);
      if (n >= 1) cmac(cv, cscale(dconj, -(double)n), sa[n - 1]);
      const double2 wn = W[n + 1];
      cp[n] = cmul(cv, wn);
      if (n < p) ap[n] = cmul(sa[n], wn);
    }
    __syncwarp();
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int m = lane + 32 * cc;
      if (m < p) {
        double2 sl = make_double2(0.0, 0.0), sg = sl;
        for (int n = 0; n < p; ++n) {
          const double pc = sh_pm2l[n * p + m];
          sl.x = fma(ap[n].x, pc, sl.x);
          sl.y = fma(ap[n].y, pc, sl.y);
          sg.x = fma(cp[n].x, pc, sg.x);
          sg.y = fma(cp[n].y, pc, sg.y);
        }
        const double pc = sh_pm2l[p * p + m];
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
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int m = lane + 32 * cc;
    if (m < p) {
      out_l[m] = al[cc];
      out_g[m] = ag[cc];
    }
  }
  __syncwarp();
}

// M2L of every cell of level >= 2 whose subtree holds owned targets: no
// dependencies (all multipoles are final), warp per cell (grid-stride).
#ifndef DDM_M2L_MINB
#define DDM_M2L_MINB 2
#endif
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32, DDM_M2L_MINB)
m2l_kernel(int c0, int c1, const int* __restrict__ clist, int64_t own_lo, int64_t own_hi,
           const int* __restrict__ v_off,
           const int* __restrict__ v_idx, const unsigned char* __restrict__ v_cls,
           const int* __restrict__ c_start, const int* __restrict__ c_count, int p_rt,
           const double2* __restrict__ w_g, const double* __restrict__ pm2l_g,
           const double2* __restrict__ mpole, double2* __restrict__ local,
           const int* __restrict__ x_slot, const double2* __restrict__ local_x, int S) {
  const int p = PT ? PT : p_rt;
  constexpr bool TC = PT > 0 && PT <= 32;   // tensor-core M2L
  if (!TC) S = 1;
  constexpr int MT = TC ? (PT + 7) / 8 : 1, KS = TC ? (PT + 4) / 4 : 1;
  const int pw = p + 2;
  extern __shared__ double2 dn_sh[];
  // dfma: W [49][pw] | C(m+n,n) [p+1][p] at n*p+m | per warp sa, ap, cp
  // tc:   A fragments [MT][KS][32] | per warp X [4 kM2LBatch][kXStride] doubles
  double2* sh_w = dn_sh;
  const int nw2 = TC ? 0 : kNOffsets * pw;
  double* sh_pm2l = reinterpret_cast<double*>(sh_w + nw2);
  const int ndbl = TC ? MT * KS * 32 : (p + 1) * p;
  double2* wbuf = sh_w + nw2 + (ndbl + 1) / 2;
  if (!TC) block_copy(sh_w, w_g, kNOffsets * pw);
  if (TC) {
    // A fragments of the Pascal matrix P[m][n] = C(m+n, n) (m < p, n <= p, else 0):
    // fragment (i, s), lane l holds P[8 i + l/4][4 s + l%4]
    for (int e = threadIdx.x; e < MT * KS * 32; e += blockDim.x) {
      const int l = e & 31, f = e >> 5, i = f / KS, sk = f - i * KS;
      const int m = 8 * i + (l >> 2), n = 4 * sk + (l & 3);
      sh_pm2l[e] = (m < p && n <= p) ? pm2l_g[n * p + m] : 0.0;
    }
  } else {
    block_copy(sh_pm2l, pm2l_g, (p + 1) * p);
  }
  __syncthreads();
  pdl_trigger();
  pdl_wait();   // all multipoles (the upward pass)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t wstride = TC ? (size_t)2 * kM2LBatch * kXStride : 3 * (size_t)p + 1;
  double2* ring = wbuf + (size_t)w * wstride;
  // S > 1 (small trees): S consecutive warps share a cell,
  // each takes every S-th batch of its V list; their partial series meet in
  // shared memory and the first warp sums them in warp order (named barrier
  // per cell slot).  S is fixed per tree: results do not depend on the rank.
  const int slot = w / S, sub = w - slot * S, per_cta = kPassWarps / S;
  double2* psum = wbuf + (size_t)kPassWarps * wstride + (size_t)w * 2 * p;
  for (int k = c0 + blockIdx.x * per_cta + slot; k < c1; k += gridDim.x * per_cta) {
    const int c = clist ? clist[k] : k;   // clist: this rank's cells (several ranks)
    const int cs = c_start[c], ce = cs + c_count[c];
    if (ce <= own_lo || cs >= own_hi) continue;   // subtree outside this rank's targets
    double2* out = local + (size_t)c * 2 * p;
    const int vb = v_off[c], ve = v_off[c + 1];
    if constexpr (TC) {
      if (S == 1) {
        m2l_cell_tc<PT>(vb, ve, v_idx, v_cls, mpole, w_g, sh_pm2l, reinterpret_cast<double*>(ring),
                        out, out + p, lane);
      } else {
        m2l_cell_tc<PT>(vb, ve, v_idx, v_cls, mpole, w_g, sh_pm2l, reinterpret_cast<double*>(ring),
                        psum, psum + p, lane, sub, S);
        asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * S) : "memory");
        if (sub == 0) {
          const double2* p0 = psum;
          for (int m = lane; m < 2 * p; m += 32) {
            double2 v = p0[m];
            for (int s2 = 1; s2 < S; ++s2) v = cadd(v, p0[(size_t)s2 * 2 * p + m]);
            out[m] = v;
          }
          __syncwarp();
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + slot), "r"(32 * S) : "memory");
        if (sub != 0) continue;
      }
    } else {
      m2l_cell_dfma(p, vb, ve, v_idx, v_cls, mpole, sh_w, sh_pm2l, ring, ring + p, ring + 2 * p,
                    out, out + p, lane);
    }
    // a leaf with an X list: + its P2L series (p2l_kernel, finished before this launch)
    const int xs = local_x ? __ldg(x_slot + c) : -1;
    if (xs >= 0) {
      const double2* lx = local_x + (size_t)xs * 2 * p;
      for (int m = lane; m < 2 * p; m += 32) out[m] = cadd(out[m], lx[m]);
      __syncwarp();
    }
  }
}

// L2L of the cells [c0, c1) of ONE level >= 3 whose subtree holds owned
// targets: local[c] (its M2L result) += L2L(parent's final local).  Launched
// top-down, one level at a time.
// L2L of one cell c (its M2L result in local[c]) from its parent's final local
// (separable form); one warp.
// Tree-static part of a cell's L2L: the cell, its parent and its quadrant
// (skip: no owned target below the cell).
struct L2LStatic {
  int c, P, quad;
  bool skip;
};
__device__ __forceinline__ L2LStatic l2l_static(int c, int64_t own_lo, int64_t own_hi,
                                                const int* __restrict__ c_start,
                                                const int* __restrict__ c_count,
                                                const int* __restrict__ c_ix,
                                                const int* __restrict__ c_iy,
                                                const int* __restrict__ c_parent) {
  L2LStatic st;
  st.c = c;
  const int cs = c_start[c], ce = cs + c_count[c];
  st.skip = ce <= own_lo || cs >= own_hi;
  st.P = c_parent[c];
  st.quad = (c_ix[c] & 1) + 2 * (c_iy[c] & 1);
  return st;
}

template <int PT>
__device__ __forceinline__ void l2l_cell(const L2LStatic& st, int p, const OpTables& T,
                                         double2* __restrict__ local, double2* xl, double2* xg,
                                         int lane) {
  const int pw = p + 2;
  constexpr int NC = PT ? (PT + 31) / 32 : 2;   // coefficients per lane
  const double2* lp = local + (size_t)st.P * 2 * p;
  double2* out = local + (size_t)st.c * 2 * p;
  const int quad = st.quad;
  // loads first: parent coefficients (slots m, m+1 of lambda, m of gamma) and
  // this cell's own M2L result
  double2 pl[NC], pl1[NC], pg[NC], ol[NC], og[NC];
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    const int m = lane + 32 * cc;
    const bool ok = m < p;
    const double2 z = make_double2(0.0, 0.0);
    pl[cc] = ok ? lp[m] : z;
    pl1[cc] = (ok && m + 1 < p) ? lp[m + 1] : z;
    pg[cc] = ok ? lp[p + m] : z;
    ol[cc] = ok ? out[m] : z;
    og[cc] = ok ? out[p + m] : z;
  }
  const double2 epsb = make_double2(0.5 * ((quad & 1) - 0.5), -0.5 * ((quad >> 1) - 0.5));
  const double2* E = T.eps + quad * pw;
  const double2* Ei = T.e2i + quad * pw;
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    const int m = lane + 32 * cc;
    if (m < p) {
      double2 gv = pg[cc];
      cmac(gv, cscale(epsb, (double)(m + 1)), pl1[cc]);
      const double2 em = E[m];
      xl[m] = cmul(pl[cc], em);
      xg[m] = cmul(gv, em);
    }
  }
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < NC; ++cc) {
    const int k = lane + 32 * cc;
    if (k < p) {
      double2 l = make_double2(0.0, 0.0), g = l;
#pragma unroll
      for (int m = 0; m < pmax<PT>(); ++m) {
        if (!PT && m >= p) break;
        const double pc = T.pas[m * p + k];   // C(m, k)
        const double2 x = xl[m], y = xg[m];
        l.x = fma(x.x, pc, l.x);
        l.y = fma(x.y, pc, l.y);
        g.x = fma(y.x, pc, g.x);
        g.y = fma(y.y, pc, g.y);
      }
      const double2 ek = Ei[k];
      double2 al = ol[cc], ag = og[cc];
      cmac(al, l, ek);
      cmac(ag, g, ek);
      out[k] = al;
      out[p + k] = ag;
    }
  }
  __syncwarp();
}

template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
l2l_level_kernel(int c0, int c1, const int* __restrict__ clist, int64_t own_lo, int64_t own_hi,
                 const int* __restrict__ c_ix,
                 const int* __restrict__ c_iy, const int* __restrict__ c_start,
                 const int* __restrict__ c_count, const int* __restrict__ c_parent, int p_rt,
                 const double2* __restrict__ eps_g, const double2* __restrict__ e2i_g,
                 const double* __restrict__ pas_g, double2* __restrict__ local) {
  const int p = PT ? PT : p_rt;
  extern __shared__ double2 l2_sh[];   // tables | per warp: xl [p] | xg [p]
  pdl_trigger();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* xl = l2_sh + tbl_doubles(p) / 2 + (size_t)w * 2 * p;
  double2* xg = xl + p;
  // tree-static data before the wait for the parents' final locals
  const OpTables T = stage_tables(reinterpret_cast<double*>(l2_sh), p, pas_g, eps_g, e2i_g);
  const int k0 = c0 + blockIdx.x * kPassWarps + w;
  L2LStatic st{};
  if (k0 < c1)
    st = l2l_static(clist ? clist[k0] : k0, own_lo, own_hi, c_start, c_count, c_ix, c_iy, c_parent);
  __syncthreads();
  pdl_wait();   // the parents' final locals (previous level / M2L)
  for (int k = k0; k < c1; k += gridDim.x * kPassWarps) {
    if (k != k0)
      st = l2l_static(clist ? clist[k] : k, own_lo, own_hi, c_start, c_count, c_ix, c_iy, c_parent);
    if (st.skip) continue;   // no owned target below c
    l2l_cell<PT>(st, p, T, local, xl, xg, lane);
  }
}

// Subtree passes for small trees: CTA per cell R of the split
// level Ls.  Upward: M2M of R's non-leaf descendants, deepest level first, and
// of R itself (levels nlevels-1 .. Ls); downward: L2L of R's descendants,
// levels Ls+1 .. nlevels-1 (R's local is final from the per-level kernels).
// Levels are separated by __syncthreads (every cell of a level inside one
// CTA): one launch per pass instead of one per level.  rng[R * nsl + (l - Ls)]
// = the range of level l's entries below R: into up_list (upward) or into the
// level's cells (downward).
template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
m2m_subtree_kernel(int Ls, int nlev, int nsl, const int2* __restrict__ rng,
                   const int* __restrict__ up_list, const int* __restrict__ c_ix,
                   const int* __restrict__ c_iy, const int* __restrict__ first_child,
                   const int* __restrict__ nchild, int p_rt, const double* __restrict__ pasT_g,
                   const double2* __restrict__ eps_g, const double2* __restrict__ e2i_g,
                   double2* __restrict__ mpole) {
  const int p = PT ? PT : p_rt;
  pdl_trigger();
  extern __shared__ double2 up_sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* wb = up_sh + tbl_doubles(p) / 2 + (size_t)w * 8 * p;
  const OpTables T = stage_tables(reinterpret_cast<double*>(up_sh), p, pasT_g, eps_g, e2i_g);
  __syncthreads();
  pdl_wait();   // leaf multipoles (P2M)
  for (int l = nlev - 1; l >= Ls; --l) {
    const int2 r = rng[(size_t)blockIdx.x * nsl + (l - Ls)];
    for (int k = r.x + w; k < r.y; k += kPassWarps)
      m2m_cell<PT>(m2m_static(up_list[k], c_ix, c_iy, first_child, nchild), p, T, mpole, wb,
                   wb + 4 * p, lane);
    __syncthreads();
  }
}

template <int PT>
__global__ void __launch_bounds__(kPassWarps * 32)
l2l_subtree_kernel(int Ls, int nlev, int nsl, const int2* __restrict__ rng, int64_t own_lo,
                   int64_t own_hi, const int* __restrict__ c_ix, const int* __restrict__ c_iy,
                   const int* __restrict__ c_start, const int* __restrict__ c_count,
                   const int* __restrict__ c_parent, int p_rt, const double2* __restrict__ eps_g,
                   const double2* __restrict__ e2i_g, const double* __restrict__ pas_g,
                   double2* __restrict__ local) {
  const int p = PT ? PT : p_rt;
  extern __shared__ double2 l2_sh[];
  pdl_trigger();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* xl = l2_sh + tbl_doubles(p) / 2 + (size_t)w * 2 * p;
  double2* xg = xl + p;
  const OpTables T = stage_tables(reinterpret_cast<double*>(l2_sh), p, pas_g, eps_g, e2i_g);
  __syncthreads();
  pdl_wait();   // the roots' final locals
  for (int l = Ls + 1; l < nlev; ++l) {
    const int2 r = rng[(size_t)blockIdx.x * nsl + (l - Ls)];
    for (int c = r.x + w; c < r.y; c += kPassWarps) {
      const L2LStatic st = l2l_static(c, own_lo, own_hi, c_start, c_count, c_ix, c_iy, c_parent);
      if (st.skip) continue;
      l2l_cell<PT>(st, p, T, local, xl, xg, lane);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ L2P (a9)
// Thread per owned element (on the far-field stream, overlapping the near
// field): Phi, Phi', Psi~ of the leaf's local series by Horner (the series are
// read through L1: the threads of a leaf share them), projected onto the
// element's frame: y_far[i] = (sigma_s, sigma_n[, p]) in sorted order.
//   W = i G C (conj(u) Phi' + Psi~),  T = sigma_n + i sigma_s = 2 Re(i G C Phi) + e^{2 i b} W
#ifndef DDM_L2P_MINB
#define DDM_L2P_MINB 4   // 64 registers, 32 warps per SM (measured: 161 -> 150 us on config 5)
#endif
#if DDM_L2P_MINB > 0
#define DDM_L2P_BOUNDS __launch_bounds__(256, DDM_L2P_MINB)
#else
#define DDM_L2P_BOUNDS __launch_bounds__(256)
#endif
template <int PT>
__global__ void DDM_L2P_BOUNDS
l2p_kernel(int64_t e_lo, int64_t e_hi, int ncomp, const int* __restrict__ el_leaf,
           const int* __restrict__ leaves, const int* __restrict__ c_level,
           const int* __restrict__ c_ix, const int* __restrict__ c_iy,
           const double2* __restrict__ local, const int* __restrict__ w_off,
           const int* __restrict__ w_idx, const double2* __restrict__ mpole, CellGeom cg,
           int p_rt, double gc, PoroFar pf, const double* __restrict__ ex,
           const double* __restrict__ ey, const double* __restrict__ ec,
           const double* __restrict__ es, double* __restrict__ y_far) {
  const int p = PT ? PT : p_rt;
  pdl_wait();   // the leaves' final locals (L2L)
  const int64_t i = e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= e_hi) return;
  const int k = __ldg(el_leaf + i);
  const int c = __ldg(leaves + k);
  const int lev = __ldg(c_level + c);
  const double x = ex[i], y = ey[i];
  // Phi and X = conj(u) dPhi/du + Psi~ summed over the local series and the
  // multipoles of the leaf's W cells (each in its own normalised coordinate)
  double2 phi_t = make_double2(0.0, 0.0), X_t = phi_t;
  if (lev >= 2) {   // no local expansion above level 2
    const double s = cg.side(lev), is = 1.0 / s;
    const double2 z0 = cg.centre(lev, __ldg(c_ix + c), __ldg(c_iy + c));
    const double2 u = make_double2((x - z0.x) * is, (y - z0.y) * is);
    const double2* L = local + (size_t)c * 2 * p;
    double2 phi = make_double2(0, 0), dphi = phi, psi = phi;
#pragma unroll
    for (int mm = pmax<PT>() - 1; mm >= 0; --mm) {
      if (!PT && mm >= p) continue;
      const double2 lm = __ldg(L + mm), gm = __ldg(L + p + mm);
      if (mm >= 1) {   // dphi = dphi u + mm L[mm]
        const double fm = (double)mm;
        dphi = make_double2(fma(dphi.x, u.x, fma(-dphi.y, u.y, fm * lm.x)),
                            fma(dphi.x, u.y, fma(dphi.y, u.x, fm * lm.y)));
      }
      phi = make_double2(fma(phi.x, u.x, fma(-phi.y, u.y, lm.x)),
                         fma(phi.x, u.y, fma(phi.y, u.x, lm.y)));
      psi = make_double2(fma(psi.x, u.x, fma(-psi.y, u.y, gm.x)),
                         fma(psi.x, u.y, fma(psi.y, u.x, gm.y)));
    }
    phi_t = phi;
    X_t = cadd(cmul(cconj(u), dphi), psi);
  }
  // M2P (W list): the multipole of each W cell D at this target,
  // in D's normalised coordinate u = (z - z_D)/s_D, v = 1/u:
  //   Phi = v f(v), f = sum_{n>=1} a_n v^(n-1);  dPhi/du = -v^2 (f + v f');
  //   Psi~ = v g(v), g = sum c_n v^(n-1)   (f, f', g by Horner)
  for (int wi = __ldg(w_off + k), we = __ldg(w_off + k + 1); wi < we; ++wi) {
    const int D = __ldg(w_idx + wi);
    const int ld = __ldg(c_level + D);
    const double isd = ldexp(1.0 / cg.W, ld);   // 1/s_D (exact power-of-two scaling)
    const double2 zd = cg.centre(ld, __ldg(c_ix + D), __ldg(c_iy + D));
    const double2 u = make_double2((x - zd.x) * isd, (y - zd.y) * isd);
    const double inn = 1.0 / fma(u.x, u.x, u.y * u.y);
    const double2 v = make_double2(u.x * inn, -u.y * inn);
    const double2* M = mpole + (size_t)D * 2 * p;
    double2 f = make_double2(0, 0), fd = f, g = f;
#pragma unroll
    for (int n = pmax<PT>(); n >= 1; --n) {
      if (!PT && n > p) continue;
      const double2 an = __ldg(M + n - 1), cn = __ldg(M + p + n - 1);
      fd = make_double2(fma(fd.x, v.x, fma(-fd.y, v.y, f.x)), fma(fd.x, v.y, fma(fd.y, v.x, f.y)));
      f = make_double2(fma(f.x, v.x, fma(-f.y, v.y, an.x)), fma(f.x, v.y, fma(f.y, v.x, an.y)));
      g = make_double2(fma(g.x, v.x, fma(-g.y, v.y, cn.x)), fma(g.x, v.y, fma(g.y, v.x, cn.y)));
    }
    const double2 dPdv = cadd(f, cmul(v, fd));
    const double2 v2 = cmul(v, v);
    const double2 dPdu = make_double2(-(v2.x * dPdv.x - v2.y * dPdv.y),
                                      -(v2.x * dPdv.y + v2.y * dPdv.x));
    phi_t = cadd(phi_t, cmul(f, v));
    X_t = cadd(X_t, cadd(cmul(cconj(u), dPdu), cmul(g, v)));
  }
  // W = i G C X, T = sigma_n + i sigma_s = 2 Re(i G C Phi) + e^{2 i b} W
  const double2 W = make_double2(-gc * X_t.y, gc * X_t.x);
  const double ct = ec[i], st = es[i];
  const double2 e2 = make_double2(ct * ct - st * st, 2.0 * ct * st);
  const double2 t2 = cmul(e2, W);
  y_far[i * ncomp + 0] = t2.y;
  y_far[i * ncomp + 1] = t2.x - 2.0 * gc * phi_t.y;
  // far pore pressure p = -4 k_p Re(i G C Phi)/fu (formula sign), ABI p = -that
  if (ncomp == 3) y_far[i * ncomp + 2] = pf.on ? -4.0 * pf.kp * gc * phi_t.y / pf.fu : 0.0;
}

// Block-staged L2P: a CTA of 128 threads takes 128
// consecutive owned elements (a few leaves).  The leaves' geometry and local
// series and the multipoles of their W cells (contiguous in the W CSR) are
// first copied into shared memory by all threads at once -- the per-element
// chain el_leaf -> leaves -> cell geometry -> coefficients becomes a few
// block-wide load stages -- then every thread evaluates its element exactly
// as l2p_kernel does (same Horner order: bitwise identical results) from
// shared memory.  Runs of elements with more than kL2PLeaves leaves or
// kL2PW W cells take the global-memory path of l2p_kernel.
constexpr int kL2PThreads = 128;
constexpr int kL2PLeaves = 16;
constexpr int kL2PW = 32;

template <int PT>
__device__ __forceinline__ void l2p_eval(int p, double x, double y, bool has_local, double2 z0,
                                         double is, const double2* L, int nwc,
                                         const double4* wg, const double2* WM, int wstride,
                                         double2& phi_t, double2& X_t) {
  phi_t = make_double2(0.0, 0.0);
  X_t = phi_t;
  if (has_local) {
    const double2 u = make_double2((x - z0.x) * is, (y - z0.y) * is);
    double2 phi = make_double2(0, 0), dphi = phi, psi = phi;
    // Horner for Phi and, by synthetic division, Phi' (dphi = dphi u + phi
    // before phi takes its next coefficient)
#pragma unroll
    for (int mm = pmax<PT>() - 1; mm >= 0; --mm) {
      if (!PT && mm >= p) continue;
      const double2 lm = L[mm], gm = L[p + mm];
      if (mm <= p - 2)
        dphi = make_double2(fma(dphi.x, u.x, fma(-dphi.y, u.y, phi.x)),
                            fma(dphi.x, u.y, fma(dphi.y, u.x, phi.y)));
      phi = make_double2(fma(phi.x, u.x, fma(-phi.y, u.y, lm.x)),
                         fma(phi.x, u.y, fma(phi.y, u.x, lm.y)));
      psi = make_double2(fma(psi.x, u.x, fma(-psi.y, u.y, gm.x)),
                         fma(psi.x, u.y, fma(psi.y, u.x, gm.y)));
    }
    phi_t = phi;
    X_t = cadd(cmul(cconj(u), dphi), psi);
  }
  for (int wi = 0; wi < nwc; ++wi) {
    const double4 g = wg[wi];
    const double2 u = make_double2((x - g.x) * g.z, (y - g.y) * g.z);
    const double inn = 1.0 / fma(u.x, u.x, u.y * u.y);
    const double2 v = make_double2(u.x * inn, -u.y * inn);
    const double2* M = WM + (size_t)wi * wstride;
    double2 f = make_double2(0, 0), fd = f, g2 = f;
#pragma unroll
    for (int n = pmax<PT>(); n >= 1; --n) {
      if (!PT && n > p) continue;
      const double2 an = M[n - 1], cn = M[p + n - 1];
      fd = make_double2(fma(fd.x, v.x, fma(-fd.y, v.y, f.x)), fma(fd.x, v.y, fma(fd.y, v.x, f.y)));
      f = make_double2(fma(f.x, v.x, fma(-f.y, v.y, an.x)), fma(f.x, v.y, fma(f.y, v.x, an.y)));
      g2 = make_double2(fma(g2.x, v.x, fma(-g2.y, v.y, cn.x)), fma(g2.x, v.y, fma(g2.y, v.x, cn.y)));
    }
    const double2 dPdv = cadd(f, cmul(v, fd));
    const double2 v2 = cmul(v, v);
    const double2 dPdu = make_double2(-(v2.x * dPdv.x - v2.y * dPdv.y),
                                      -(v2.x * dPdv.y + v2.y * dPdv.x));
    phi_t = cadd(phi_t, cmul(f, v));
    X_t = cadd(X_t, cadd(cmul(cconj(u), dPdu), cmul(g2, v)));
  }
}

#ifndef DDM_L2P_TMA
#define DDM_L2P_TMA 1
#endif
#ifndef DDM_L2PB_MINB
#define DDM_L2PB_MINB 8
#endif
template <int PT>
__global__ void __launch_bounds__(kL2PThreads, DDM_L2PB_MINB)
l2p_block_kernel(int64_t e_lo, int64_t e_hi, int ncomp, const int4* __restrict__ runs,
                 const int* __restrict__ order,
                 const double4* __restrict__ leaf_geo, const double4* __restrict__ w_geo,
                 const int* __restrict__ el_leaf,
                 const int* __restrict__ leaves, const int* __restrict__ c_level,
                 const int* __restrict__ c_ix, const int* __restrict__ c_iy,
                 const double2* __restrict__ local, const int* __restrict__ w_off,
                 const int* __restrict__ w_idx, const double2* __restrict__ mpole, CellGeom cg,
                 int p_rt, double gc, PoroFar pf, const double* __restrict__ ex,
                 const double* __restrict__ ey, const double* __restrict__ ec,
                 const double* __restrict__ es, double* __restrict__ y_far) {
  const int p = PT ? PT : p_rt;
  const int P2 = 2 * p;
  extern __shared__ double2 l2p_sh[];   // [kL2PLeaves][2p] locals | [kL2PW][2p] W multipoles
  double2* shL = l2p_sh;
  double2* shW = l2p_sh + (size_t)kL2PLeaves * P2;
  __shared__ double4 kgeo[kL2PLeaves];   // (z0.x, z0.y, 1/s, has local)
  __shared__ double4 wgeo[kL2PW];        // (z_D.x, z_D.y, 1/s_D, -)
  __shared__ int kcell[kL2PLeaves], kw[kL2PLeaves + 1], wcell[kL2PW];
  __shared__ __align__(8) unsigned long long l2p_bar;
  const int tid = threadIdx.x;
#if DDM_L2P_TMA
  if (tid == 0) mbar_init(smem_u32(&l2p_bar), 1);
#endif
  const int rb = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x;
  const int64_t i0 = e_lo + (int64_t)rb * kL2PThreads;
  const int64_t i = i0 + tid;
  const bool valid = i < e_hi;
  // the run's descriptor (precomputed per owned range): the staging is two
  // block-wide load rounds -- the leaves' / W cells' ids and geometry, then
  // their coefficients -- independent of the element loads
  const int4 rd = __ldg(runs + rb);
  const int k0 = rd.x, nk = rd.y, w0 = rd.z, nw = rd.w;
  const int k = valid ? __ldg(el_leaf + i) : -1;
  // the element's own data, loaded before the staging (their latency would
  // otherwise be exposed after the evaluation)
  const double x = valid ? __ldg(ex + i) : 0.0, y = valid ? __ldg(ey + i) : 0.0;
  const double ct = valid ? __ldg(ec + i) : 1.0, st = valid ? __ldg(es + i) : 0.0;
  const bool staged = nk <= kL2PLeaves && nw <= kL2PW;
  if (staged) {
    if (tid < nk) {
      kcell[tid] = __ldg(leaves + k0 + tid);
      kgeo[tid] = leaf_geo[k0 + tid];
      kw[tid] = __ldg(w_off + k0 + tid) - w0;
      if (tid == nk - 1) kw[nk] = nw;
    } else if (tid >= 64 && tid - 64 < nw) {
      wcell[tid - 64] = __ldg(w_idx + w0 + tid - 64);
      wgeo[tid - 64] = w_geo[w0 + tid - 64];
    }
    __syncthreads();
    pdl_wait();   // the leaves' final locals (L2L)
#if DDM_L2P_TMA
    // coefficient rows by 1-D bulk copies (one per leaf / W cell, 2p double2
    // each) issued by warp 0, completion counted on one mbarrier
    if (tid < 32) {
      const unsigned rowb = (unsigned)P2 * sizeof(double2);
      if (tid == 0) mbar_expect_tx(smem_u32(&l2p_bar), (unsigned)(nk + nw) * rowb);
      __syncwarp();
      for (int r = tid; r < nk + nw; r += 32) {
        if (r < nk)
          bulk_g2s(smem_u32(shL + (size_t)r * P2), local + (size_t)kcell[r] * P2, rowb,
                   smem_u32(&l2p_bar));
        else
          bulk_g2s(smem_u32(shW + (size_t)(r - nk) * P2), mpole + (size_t)wcell[r - nk] * P2,
                   rowb, smem_u32(&l2p_bar));
      }
    }
    mbar_wait(smem_u32(&l2p_bar), 0);
#else
    for (int e = tid; e < nk * P2; e += kL2PThreads) {
      const int kl = e / P2, m = e - kl * P2;
      shL[e] = local[(size_t)kcell[kl] * P2 + m];
    }
    for (int e = tid; e < nw * P2; e += kL2PThreads) {
      const int wl = e / P2, m = e - wl * P2;
      shW[e] = __ldg(mpole + (size_t)wcell[wl] * P2 + m);
    }
    __syncthreads();
#endif
  } else {
    pdl_wait();
  }
  if (!valid) return;
  double2 phi_t, X_t;
  if (staged) {
    const int kl = k - k0;
    const double4 g = kgeo[kl];
    const int wa = kw[kl], wb = kw[kl + 1];
    l2p_eval<PT>(p, x, y, g.w != 0.0, make_double2(g.x, g.y), g.z, shL + (size_t)kl * P2, wb - wa,
                 wgeo + wa, shW + (size_t)wa * P2, P2, phi_t, X_t);
  } else {
    // global-memory path (rare: many tiny leaves or W cells in one run)
    const int c = __ldg(leaves + k);
    const int lev = __ldg(c_level + c);
    const double2 z0 = cg.centre(lev, __ldg(c_ix + c), __ldg(c_iy + c));
    phi_t = make_double2(0.0, 0.0);
    X_t = phi_t;
    double2 ph, Xl;
    l2p_eval<PT>(p, x, y, lev >= 2, z0, 1.0 / cg.side(lev), local + (size_t)c * P2, 0, nullptr,
                 nullptr, P2, ph, Xl);
    phi_t = ph;
    X_t = Xl;
    for (int wi = __ldg(w_off + k), we = __ldg(w_off + k + 1); wi < we; ++wi) {
      const int D = __ldg(w_idx + wi);
      const int ld = __ldg(c_level + D);
      const double2 zd = cg.centre(ld, __ldg(c_ix + D), __ldg(c_iy + D));
      const double4 wg1 = make_double4(zd.x, zd.y, ldexp(1.0 / cg.W, ld), 0.0);
      double2 pw, Xw;
      l2p_eval<PT>(p, x, y, false, z0, 0.0, nullptr, 1, &wg1, mpole + (size_t)D * P2, P2, pw, Xw);
      phi_t = cadd(phi_t, pw);
      X_t = cadd(X_t, Xw);
    }
  }
  const double2 W = make_double2(-gc * X_t.y, gc * X_t.x);
  const double2 e2 = make_double2(ct * ct - st * st, 2.0 * ct * st);
  const double2 t2 = cmul(e2, W);
  y_far[i * ncomp + 0] = t2.y;
  y_far[i * ncomp + 1] = t2.x - 2.0 * gc * phi_t.y;
  if (ncomp == 3) y_far[i * ncomp + 2] = pf.on ? -4.0 * pf.kp * gc * phi_t.y / pf.fu : 0.0;
}

// ------------------------------------------------------------ finalize (a11)
// per owned sorted element: near field (sum of the P2P partials of its target
// group, in item order) + far field (y_far), written in user and/or sorted order
__global__ void finalize_kernel(int64_t e_lo, int64_t e_hi, int ncomp,
                                const int* __restrict__ el_leaf, const int* __restrict__ leaves,
                                const int* __restrict__ c_start, const int* __restrict__ c_count,
                                const int* __restrict__ item_off, const double* __restrict__ part,
                                const double* __restrict__ y_far, const int* __restrict__ perm,
                                double* __restrict__ y_user, double* __restrict__ y_sorted) {
  // a PDL-launched successor (the GMRES step's first CGS kernel) may start early;
  // it waits for this grid before reading anything
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t i = e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= e_hi) return;
  const int k = el_leaf[i];
  const int c = leaves[k];
  const int slot = (int)(i - c_start[c]);
  const int ngroups = (c_count[c] + kTgtGroup - 1) / kTgtGroup;
  const int i0 = item_off[k];
  const int nch = (item_off[k + 1] - i0) / ngroups;
  const int g = slot / kTgtGroup, ln = slot % kTgtGroup;
  double t0 = y_far[i * ncomp], t1 = y_far[i * ncomp + 1];
  double pr = ncomp == 3 ? y_far[i * ncomp + 2] : 0.0;
  for (int h = 0; h < nch; ++h) {
    const double* pp = part + ((int64_t)(i0 + g * nch + h) * kTgtGroup + ln) * ncomp;
    t0 += pp[0];
    t1 += pp[1];
    if (ncomp == 3) pr += pp[2];
  }
  if (y_sorted) {
    y_sorted[i * ncomp + 0] = t0;
    y_sorted[i * ncomp + 1] = t1;
    if (ncomp == 3) y_sorted[i * ncomp + 2] = pr;
  }
  if (y_user) {
    const int j = perm[i];
    y_user[(int64_t)j * ncomp + 0] = t0;
    y_user[(int64_t)j * ncomp + 1] = t1;
    if (ncomp == 3) y_user[(int64_t)j * ncomp + 2] = pr;
  }
}

// Host-side launch configuration is cached per (kernel, shared-memory size,
// device): the attribute and occupancy queries cost microseconds of host time
// per call, which would otherwise sit between the kernels of every matvec.
struct LaunchCfg {
  const void* kernel;
  size_t shm;
  int device;
  int per_sm, nsm;
};
std::mutex g_cfg_mu;
std::vector<LaunchCfg> g_cfg;

template <class K>
int set_smem(ddm_ctx_s* ctx, K kernel, size_t shm) {
  // dynamic + static shared memory above 48 KB needs the opt-in attribute
  // (static use of these kernels stays below 17 KB)
  if (shm <= 30 * 1024) return DDM_OK;
  std::lock_guard<std::mutex> lk(g_cfg_mu);
  for (const auto& c : g_cfg)
    if (c.kernel == (const void*)kernel && c.shm >= shm && c.device == ctx->device && c.per_sm < 0)
      return DDM_OK;
  DDM_CUDA(ctx, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  g_cfg.push_back({(const void*)kernel, shm, ctx->device, -1, 0});
  return DDM_OK;
}

// integer environment knob, read once per name
static int env_int(const char* name, int dflt) {
  static std::mutex mu;
  static std::vector<std::pair<std::string, int>> seen;
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& kv : seen)
    if (kv.first == name) return kv.second;
  const char* e = getenv(name);
  const int v = e ? atoi(e) : dflt;
  seen.emplace_back(name, v);
  return v;
}

int pass_grid(ddm_ctx_s* ctx, const void* kernel, size_t shm, int work, int kcap = -1) {
  int per_sm = -1, nsm = 148;
  {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    for (const auto& c : g_cfg)
      if (c.kernel == kernel && c.shm == shm && c.device == ctx->device && c.per_sm >= 0) {
        per_sm = c.per_sm;
        nsm = c.nsm;
        break;
      }
  }
  if (per_sm < 0) {
    per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kPassWarps * 32, shm);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    g_cfg.push_back({kernel, shm, ctx->device, per_sm, nsm});
  }
  const int by_work = (work + kPassWarps - 1) / kPassWarps;
  // DDM_PASS_BLOCKS_PER_SM caps the grids of the pass kernels so the
  // concurrent near field keeps SM slots (0 = occupancy limit); default: 2
  // block per SM when the near field runs concurrently, the occupancy limit
  // when everything is serial
  static const int env_cap = [] {
    const char* e = getenv("DDM_PASS_BLOCKS_PER_SM");
    return e ? atoi(e) : -1;
  }();
  const int cap = (kcap >= 0 && !ctx->serial) ? kcap : env_cap >= 0 ? env_cap : (ctx->serial ? 0 : 2);
  if (cap > 0) per_sm = std::min(per_sm, cap);
  return std::max(1, std::min(std::max(per_sm, 1) * nsm, by_work));
}

}  // namespace

// Launch with programmatic stream serialisation (PDL, see pdl_wait) when the
// far chain is latency bound: small trees, where the chain is the matvec's
// critical path (config 3: 114 -> 110 us, config 4: 64 -> 60 us).  On large
// trees the early-resident dependent blocks take SM slots from the concurrent
// near field (config 5: 1.16 -> 1.28 ms), so there it is off -- except on
// several ranks, where each rank's near field shrinks by the rank count and the
// replicated far chain becomes the critical path.  DDM_PDL=0/1 overrides.
static bool use_pdl(const ddm_tree_s* t) {
  static const int env = [] {
    const char* e = getenv("DDM_PDL");
    return e ? atoi(e) : -1;
  }();
  return env >= 0 ? env != 0 : (t->n <= 200000 || t->ctx->world > 1);
}

// Subtree passes (one launch per pass below the split level) on small trees,
// where the per-level launches are the chain's latency; DDM_SUBTREE=0/1
// overrides.
static bool use_subtrees(const ddm_tree_s* t) {
  static const int env = [] {
    const char* e = getenv("DDM_SUBTREE");
    return e ? atoi(e) : -1;
  }();
  if (t->sub_n <= 0) return false;
  return env >= 0 ? env != 0 : (t->n <= 200000 || t->ctx->world > 1);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool on, void (*kernel)(KArgs...), unsigned grid, unsigned block,
                       size_t shm, cudaStream_t s, Args... args) {
  const bool off = !on;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = shm;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// upward pass: P2M on all leaves, then M2M one level at a time (deepest
// first), replicated on every rank
int launch_upward(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D, int ncomp,
                  const PoroFar& pf, cudaStream_t s, int scope) {
  // D in user order (perm_in = sorted -> user, read through it) or sorted (nullptr)
  const int p = t->p;
  const bool do_p2m = scope != kUpStrad;
  if (do_p2m && (!t->p2m_runs || t->p2m_own_lo != t->own_leaf_lo || t->p2m_own_hi != t->own_leaf_hi))
    return set_error(ctx, DDM_ERR_ARG, "internal: P2M runs not prepared (fmm_workspace)");
  const int nlv = scope == kUpOwn ? t->own_leaf_hi - t->own_leaf_lo : t->nleaves;
  const int* ulist = scope == kUpFull ? t->up_list : scope == kUpOwn ? t->up_own : t->up_strad;
  const std::vector<int>& uoff =
      scope == kUpFull ? t->up_level_off : scope == kUpOwn ? t->up_own_off : t->up_strad_off;
  const CellGeom cg{t->x_min, t->y_min, t->W};
  const size_t shm = (size_t)tbl_doubles(p) * sizeof(double) + (size_t)kPassWarps * 8 * p * sizeof(double2);
  const size_t shp = (size_t)kPassWarps * 32 * 17 * sizeof(double2);
  int rc = DDM_OK;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if (do_p2m && nlv > 0) {                                                                    \
      if ((rc = set_smem(ctx, p2m_kernel<PT>, shp))) return rc;                                 \
      const int nrun = scope == kUpOwn ? t->p2m_nruns_own : t->p2m_nruns;                       \
      const int2* rtab = scope == kUpOwn ? t->p2m_runs_own : t->p2m_runs;                       \
      const int nb = pass_grid(ctx, (const void*)p2m_kernel<PT>, shp, nrun, env_int("DDM_P2M_CAP", -1)); \
      stage_begin(ctx, DDM_ST_P2M, s);                                                          \
      p2m_kernel<PT><<<nb, kPassWarps * 32, shp, s>>>(nrun, rtab, t->leaves, t->c_level,        \
                                                      t->c_ix, t->c_iy, t->c_start, t->c_count, \
                                                      cg, p, perm_in, D,                        \
                                                      ncomp, t->ex, t->ey, t->ea, t->ec, t->es, \
                                                      t->mpole, pf);                            \
      stage_end(ctx, DDM_ST_P2M, s);                                                            \
    }                                                                                           \
    if ((rc = set_smem(ctx, m2m_level_kernel<PT>, shm))) return rc;                             \
    stage_begin(ctx, DDM_ST_M2M, s);                                                            \
    int top = t->nlevels - 1;                                                                   \
    if (scope == kUpFull && use_subtrees(t)) {                                                  \
      if ((rc = set_smem(ctx, m2m_subtree_kernel<PT>, shm))) return rc;                         \
      DDM_CUDA(ctx, launch_pdl(use_pdl(t), m2m_subtree_kernel<PT>, t->sub_n, kPassWarps * 32,   \
                               shm, s, t->sub_Ls, t->nlevels, t->sub_nsl,                       \
                               (const int2*)t->sub_up, (const int*)t->up_list,                  \
                               (const int*)t->c_ix, (const int*)t->c_iy,                        \
                               (const int*)t->c_first_child, (const int*)t->c_nchild, p,        \
                               (const double*)t->op_pasT, (const double2*)t->op_eps,            \
                               (const double2*)t->op_e2i, t->mpole));                           \
      top = t->sub_Ls - 1;                                                                      \
    }                                                                                           \
    for (int lev = top; lev >= 2; --lev) {                                                      \
      const int u0 = uoff[2 * lev], u1 = uoff[2 * lev + 1];                                     \
      if (u1 <= u0) continue;                                                                   \
      const int nb2 = pass_grid(ctx, (const void*)m2m_level_kernel<PT>, shm, u1 - u0);          \
      DDM_CUDA(ctx, launch_pdl(use_pdl(t), m2m_level_kernel<PT>, nb2, kPassWarps * 32, shm, s, u0, u1,     \
                               (const int*)ulist, (const int*)t->c_ix,                         \
                               (const int*)t->c_iy, (const int*)t->c_first_child,              \
                               (const int*)t->c_nchild, p, (const double*)t->op_pasT,          \
                               (const double2*)t->op_eps, (const double2*)t->op_e2i,           \
                               t->mpole));                                                     \
    }                                                                                           \
    stage_end(ctx, DDM_ST_M2M, s);                                                              \
  } while (0)
  DDM_P_DISPATCH(p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// Multipole exchange of the sharded upward pass: pack this
// rank's complete cells (xr_cells[xr_off[rank] ..]) into xsend; after the
// all-gather (xrecv = every rank's pack, padded to xr_max cells), scatter the
// other ranks' cells into mpole.
__global__ void mpole_pack_kernel(int ncell, const int* __restrict__ cells, int P2,
                                  const double2* __restrict__ mpole, double2* __restrict__ out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)ncell * P2) return;
  const int k = (int)(e / P2), m = (int)(e - (int64_t)k * P2);
  out[e] = mpole[(size_t)cells[k] * P2 + m];
}

__global__ void mpole_unpack_kernel(const int* __restrict__ cells, const int* __restrict__ xr_off,
                                    int world, int rank, int xr_max, int P2,
                                    const double2* __restrict__ in, double2* __restrict__ mpole) {
  const int r = blockIdx.y;
  if (r == rank) return;   // own cells are already in place
  const int c0 = xr_off[r], nc = xr_off[r + 1] - c0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nc * P2;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / P2), m = (int)(e - (int64_t)k * P2);
    mpole[(size_t)cells[c0 + k] * P2 + m] = in[((size_t)r * xr_max + k) * P2 + m];
  }
}

int launch_mpole_pack(ddm_ctx_s* ctx, ddm_tree_s* t, int rank, cudaStream_t s) {
  const int P2 = 2 * t->p;
  const int c0 = t->xr_off[rank], nc = t->xr_off[rank + 1] - c0;
  if (nc <= 0) return DDM_OK;
  if (!t->xsend) return set_error(ctx, DDM_ERR_ARG, "no multipole exchange buffers (one rank)");
  mpole_pack_kernel<<<nblk((int64_t)nc * P2, 256), 256, 0, s>>>(nc, t->xr_cells + c0, P2, t->mpole,
                                                                t->xsend);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_mpole_unpack(ddm_ctx_s* ctx, ddm_tree_s* t, int rank, int world, cudaStream_t s) {
  const int P2 = 2 * t->p;
  if (t->xr_max <= 0) return DDM_OK;
  if (!t->xrecv) return set_error(ctx, DDM_ERR_ARG, "no multipole exchange buffers (one rank)");
  dim3 grid(std::max(1u, std::min(nblk((int64_t)t->xr_max * P2, 256), 1184u)), world);
  mpole_unpack_kernel<<<grid, 256, 0, s>>>(t->xr_cells, t->xr_off_dev, world, rank, t->xr_max, P2,
                                           t->xrecv, t->mpole);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// downward pass: M2L of every cell of level >= 2, then L2L one level at a
// time (top-down), both restricted to subtrees holding owned targets
int launch_downward(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s, bool use_x) {
  if (t->nlevels <= 2) return DDM_OK;
  // use_x: the M2L adds the P2L series of the leaves with X lists (the caller
  // made s wait for the P2L; the M2L is then launched without PDL)
  const int* xsl = use_x ? t->x_slot : nullptr;
  const double2* lxp = use_x ? t->local_x : nullptr;
  const int p = t->p;
  // several ranks: iterate this rank's cell list instead of every cell
  const int* cl = t->dn_own;
  const int c0 = cl ? t->dn_own_off[2] : t->level_off[2];
  const int c1 = cl ? t->dn_own_off[t->nlevels] : t->ncells;
  const bool tc = (p == 8 || p == 12 || p == 16 || p == 20 || p == 24 || p == 28 || p == 30 || p == 32);
  const size_t ndbl = tc ? (size_t)((p + 7) / 8) * ((p + 4) / 4) * 32 : (size_t)(p + 1) * p;
  const size_t wstride = tc ? (size_t)2 * kM2LBatch * kXStride : 3 * (size_t)p + 1;
  const size_t shm = ((tc ? 0 : (size_t)kNOffsets * (p + 2)) + (ndbl + 1) / 2 +
                      (size_t)kPassWarps * wstride + (tc ? (size_t)kPassWarps * 2 * p : 0)) *
                     sizeof(double2);
  // warps per cell (small trees: a cell's V list over S warps, §4.4d); a
  // property of the whole tree, so every rank sums the same way
  static const int m2l_s_env = env_int("DDM_M2L_SPLIT", -1);
  // M2L blocks per SM: on large trees (no PDL: the M2L overlaps the near
  // field) one block per SM leaves the near field its slots (config 5 step
  // 0.951 -> 0.941 ms); DDM_M2L_CAP overrides
  static const int m2l_cap_env = env_int("DDM_M2L_CAP", -1);
  const int m2l_cap = m2l_cap_env >= 0 ? m2l_cap_env : (use_pdl(t) ? -1 : 1);
  const int64_t ncell2 = (int64_t)t->ncells - t->level_off[2];
  const int S = !tc ? 1 : m2l_s_env >= 0 ? std::max(1, std::min(4, m2l_s_env))
                        : ncell2 <= 768 ? 4 : 1;
  const size_t shm2 = (size_t)tbl_doubles(p) * sizeof(double) + (size_t)kPassWarps * 2 * p * sizeof(double2);
  int rc = DDM_OK;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if ((rc = set_smem(ctx, m2l_kernel<PT>, shm))) return rc;                                   \
    const int nb = pass_grid(ctx, (const void*)m2l_kernel<PT>, shm, (c1 - c0) * S, m2l_cap);  \
    stage_begin(ctx, DDM_ST_M2L, s);                                                            \
    DDM_CUDA(ctx, launch_pdl(use_pdl(t) && !use_x, m2l_kernel<PT>, nb, kPassWarps * 32, shm, s, \
                             c0, c1,                                                           \
                             (const int*)cl, (int64_t)t->own_el_lo, (int64_t)t->own_el_hi,     \
                             (const int*)t->v_off, (const int*)t->v_idx,                       \
                             (const unsigned char*)t->v_cls, (const int*)t->c_start,           \
                             (const int*)t->c_count, p, (const double2*)t->op_w,               \
                             (const double*)t->op_pm2l, (const double2*)t->mpole, t->local,    \
                             xsl, lxp, S));                                                    \
    stage_end(ctx, DDM_ST_M2L, s);                                                              \
    if ((rc = set_smem(ctx, l2l_level_kernel<PT>, shm2))) return rc;                            \
    stage_begin(ctx, DDM_ST_L2L, s);                                                            \
    const bool sub = use_subtrees(t);                                                           \
    for (int lev = 3; lev < (sub ? t->sub_Ls + 1 : t->nlevels); ++lev) {                        \
      const int a = cl ? t->dn_own_off[lev] : t->level_off[lev];                                \
      const int b = cl ? t->dn_own_off[lev + 1] : t->level_off[lev + 1];                        \
      if (b <= a) continue;                                                                     \
      const int nb2 = pass_grid(ctx, (const void*)l2l_level_kernel<PT>, shm2, b - a);           \
      DDM_CUDA(ctx, launch_pdl(use_pdl(t), l2l_level_kernel<PT>, nb2, kPassWarps * 32, shm2, s, a, b,      \
                               (const int*)cl, (int64_t)t->own_el_lo, (int64_t)t->own_el_hi,   \
                               (const int*)t->c_ix, (const int*)t->c_iy,                       \
                               (const int*)t->c_start, (const int*)t->c_count,                 \
                               (const int*)t->c_parent, p, (const double2*)t->op_eps,          \
                               (const double2*)t->op_e2i, (const double*)t->op_pas,            \
                               t->local));                                                     \
    }                                                                                           \
    if (sub) {                                                                                  \
      if ((rc = set_smem(ctx, l2l_subtree_kernel<PT>, shm2))) return rc;                        \
      DDM_CUDA(ctx, launch_pdl(use_pdl(t), l2l_subtree_kernel<PT>, t->sub_n, kPassWarps * 32,   \
                               shm2, s, t->sub_Ls, t->nlevels, t->sub_nsl,                      \
                               (const int2*)t->sub_cells, (int64_t)t->own_el_lo,                \
                               (int64_t)t->own_el_hi, (const int*)t->c_ix,                      \
                               (const int*)t->c_iy, (const int*)t->c_start,                     \
                               (const int*)t->c_count, (const int*)t->c_parent, p,              \
                               (const double2*)t->op_eps, (const double2*)t->op_e2i,            \
                               (const double*)t->op_pas, t->local));                            \
    }                                                                                           \
    stage_end(ctx, DDM_ST_L2L, s);                                                              \
  } while (0)
  DDM_P_DISPATCH(p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// static geometry of every leaf and every W entry (block-staged L2P)
__global__ void l2p_geo_kernel(int nleaves, int64_t nw, const int* __restrict__ leaves,
                               const int* __restrict__ w_idx, const int* __restrict__ c_level,
                               const int* __restrict__ c_ix, const int* __restrict__ c_iy,
                               CellGeom cg, double4* __restrict__ leaf_geo,
                               double4* __restrict__ w_geo) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < nleaves) {
    const int c = leaves[j];
    const int lev = c_level[c];
    const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
    leaf_geo[j] = make_double4(z0.x, z0.y, 1.0 / cg.side(lev), lev >= 2 ? 1.0 : 0.0);
  } else if (j - nleaves < nw) {
    const int D = w_idx[j - nleaves];
    const int ld = c_level[D];
    const double2 zd = cg.centre(ld, c_ix[D], c_iy[D]);
    w_geo[j - nleaves] = make_double4(zd.x, zd.y, ldexp(1.0 / cg.W, ld), 0.0);
  }
}

// run r = elements [e_lo + 128 r, ...) of the owned range: (first leaf,
// leaves, first W entry, W entries)
__global__ void l2p_runs_kernel(int nruns, int64_t e_lo, int64_t e_hi, const int* __restrict__ el_leaf,
                                const int* __restrict__ w_off, int4* __restrict__ runs,
                                int* __restrict__ work) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  const int64_t a = e_lo + (int64_t)r * kL2PThreads;
  const int64_t b = min(e_hi, a + kL2PThreads) - 1;
  const int k0 = el_leaf[a], k1 = el_leaf[b];
  runs[r] = make_int4(k0, k1 - k0 + 1, w_off[k0], w_off[k1 + 1] - w_off[k0]);
  // work estimate (series evaluations) of the run, for the launch order
  int wk = 0;
  for (int64_t i = a; i <= b; ++i) {
    const int k = el_leaf[i];
    wk += 1 + w_off[k + 1] - w_off[k];
  }
  work[r] = wk;
}

static int l2p_tables(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) {
  int rc;
  const CellGeom cg{t->x_min, t->y_min, t->W};
  if (!t->leaf_geo) {
    if ((rc = talloc(ctx, &t->leaf_geo, (size_t)t->nleaves, s)) ||
        (rc = talloc(ctx, &t->w_geo, (size_t)std::max<int64_t>(t->nw, 1), s)))
      return rc;
    const int64_t tot = t->nleaves + t->nw;
    l2p_geo_kernel<<<nblk(tot, 256), 256, 0, s>>>(t->nleaves, t->nw, t->leaves, t->w_idx,
                                                   t->c_level, t->c_ix, t->c_iy, cg, t->leaf_geo,
                                                   t->w_geo);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  // P2M runs: consecutive whole leaves of at most DDM_P2M_RUN_HB half-blocks
  // of 16 elements in all (a larger leaf is a run of its own; DESIGN.md
  // §4.12).  For all leaves (replicated upward pass) and for the owned leaves
  // (sharded pass)
  if (!t->p2m_runs || t->p2m_own_lo != t->own_leaf_lo || t->p2m_own_hi != t->own_leaf_hi) {
    std::vector<int> hl(t->nleaves), hc(t->ncells);
    DDM_CUDA(ctx, cudaMemcpyAsync(hl.data(), t->leaves, t->nleaves * sizeof(int),
                                  cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaMemcpyAsync(hc.data(), t->c_count, t->ncells * sizeof(int),
                                  cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    auto build = [&](int l0, int l1, std::vector<int2>& out) {
      out.clear();
      int k = l0;
      auto nh = [&](int kk) { return (hc[hl[kk]] + 15) / 16; };
      // half-blocks per run (at most): up to 8 while that leaves >= 4 runs per
      // resident warp of the GPU (config 5), 2 = one round on small trees
      // (latency bound: one run per warp)
      int64_t tot_hb = 0;
      for (int kk = l0; kk < l1; ++kk) tot_hb += nh(kk);
      const int hb_env = env_int("DDM_P2M_RUN_HB", 0);
      const int hbmax = hb_env > 0 ? hb_env
                                   : (int)std::min<int64_t>(8, std::max<int64_t>(2, tot_hb / (4 * 148 * 16)));
      while (k < l1) {
        int tot = nh(k), m = 1;
        while (k + m < l1 && m < 32 && tot + nh(k + m) <= hbmax) tot += nh(k + m++);
        out.push_back(make_int2(k, m));
        k += m;
      }
    };
    std::vector<int2> rf, ro;
    build(0, t->nleaves, rf);
    build(t->own_leaf_lo, t->own_leaf_hi, ro);
    if (t->p2m_runs) cudaFree(t->p2m_runs);
    if (t->p2m_runs_own) cudaFree(t->p2m_runs_own);
    t->p2m_runs = t->p2m_runs_own = nullptr;
    if ((rc = talloc(ctx, &t->p2m_runs, std::max<size_t>(rf.size(), 1), s)) ||
        (rc = talloc(ctx, &t->p2m_runs_own, std::max<size_t>(ro.size(), 1), s)))
      return rc;
    if (!rf.empty())
      DDM_CUDA(ctx, cudaMemcpyAsync(t->p2m_runs, rf.data(), rf.size() * sizeof(int2),
                                    cudaMemcpyHostToDevice, s));
    if (!ro.empty())
      DDM_CUDA(ctx, cudaMemcpyAsync(t->p2m_runs_own, ro.data(), ro.size() * sizeof(int2),
                                    cudaMemcpyHostToDevice, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    t->p2m_nruns = (int)rf.size();
    t->p2m_nruns_own = (int)ro.size();
    t->p2m_own_lo = t->own_leaf_lo;
    t->p2m_own_hi = t->own_leaf_hi;
    // near-field leaf blocks longest-first (targets x staged records), so the
    // launch does not end on a heavy leaf; DDM_P2P_ORDER=0 keeps Morton order
    if (t->p2p_leaf_order) cudaFree(t->p2p_leaf_order);
    t->p2p_leaf_order = nullptr;
    // 1: by work; 2: by work in power-of-two classes, Morton order within a
    // class (keeps neighbouring leaves, which share source records in L2,
    // close in launch order); 3: the heaviest tenth first, then Morton order
    const int p2p_ord = env_int("DDM_P2P_ORDER", 1);
    const int nlo = t->own_leaf_hi - t->own_leaf_lo;
    if (p2p_ord > 0 && nlo > 0 && t->leaf_info && t->lr_rng) {
      // the work of the elastic series path: U minus X when there are X lists
      const bool ux = t->nx > 0 && t->leaf_info_x && t->lr_rng_x;
      const int64_t nur = ux ? t->nux : t->nu;
      std::vector<int4> li(t->nleaves);
      std::vector<int2> lr(std::max<int64_t>(nur, 1));
      DDM_CUDA(ctx, cudaMemcpyAsync(li.data(), ux ? t->leaf_info_x : t->leaf_info,
                                    li.size() * sizeof(int4), cudaMemcpyDeviceToHost, s));
      if (nur > 0)
        DDM_CUDA(ctx, cudaMemcpyAsync(lr.data(), ux ? t->lr_rng_x : t->lr_rng, nur * sizeof(int2),
                                      cudaMemcpyDeviceToHost, s));
      DDM_CUDA(ctx, cudaStreamSynchronize(s));
      std::vector<int64_t> wk(nlo);
      std::vector<int> ord(nlo);
      for (int k = 0; k < nlo; ++k) {
        const int4 v = li[t->own_leaf_lo + k];
        int64_t rec = 0;
        for (int r = v.z; r < v.w; ++r) rec += lr[r].y - lr[r].x + 1;
        wk[k] = (int64_t)v.y * rec;
        ord[k] = k;
      }
      if (p2p_ord == 2) {
        for (auto& v : wk) v = v > 0 ? 63 - __builtin_clzll((unsigned long long)v) : 0;
      } else if (p2p_ord == 3) {
        std::vector<int64_t> srt(wk);
        std::nth_element(srt.begin(), srt.begin() + nlo / 10, srt.end(), std::greater<int64_t>());
        const int64_t thr = srt[nlo / 10];
        for (auto& v : wk) v = v >= thr ? 1 : 0;
      }
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return wk[a] > wk[b]; });
      if ((rc = talloc(ctx, &t->p2p_leaf_order, (size_t)nlo, s))) return rc;
      DDM_CUDA(ctx, cudaMemcpyAsync(t->p2p_leaf_order, ord.data(), nlo * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
      DDM_CUDA(ctx, cudaStreamSynchronize(s));
    }
  }
  if (t->l2p_lo != t->own_el_lo || t->l2p_hi != t->own_el_hi) {
    if (t->l2p_runs) cudaFree(t->l2p_runs);
    t->l2p_runs = nullptr;
    const int64_t ne = t->own_el_hi - t->own_el_lo;
    t->l2p_nruns = (int)((ne + kL2PThreads - 1) / kL2PThreads);
    if ((rc = talloc(ctx, &t->l2p_runs, (size_t)std::max(t->l2p_nruns, 1), s))) return rc;
    if (t->l2p_order) cudaFree(t->l2p_order);
    t->l2p_order = nullptr;
    if (t->l2p_nruns > 0) {
      int* work = nullptr;
      if ((rc = talloc(ctx, &work, (size_t)t->l2p_nruns, s))) return rc;
      l2p_runs_kernel<<<nblk(t->l2p_nruns, 256), 256, 0, s>>>(t->l2p_nruns, t->own_el_lo,
                                                               t->own_el_hi, t->el_leaf, t->w_off,
                                                               t->l2p_runs, work);
      DDM_CUDA(ctx, cudaGetLastError());
      // longest runs first: the launch's tail is short runs
      static const bool ord_env = [] {
        const char* e = getenv("DDM_L2P_ORDER");
        return !(e && e[0] == '0');
      }();
      if (ord_env) {
        std::vector<int> hw(t->l2p_nruns), ord(t->l2p_nruns);
        DDM_CUDA(ctx, cudaMemcpyAsync(hw.data(), work, hw.size() * sizeof(int),
                                      cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaStreamSynchronize(s));
        for (int r = 0; r < t->l2p_nruns; ++r) ord[r] = r;
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hw[a] > hw[b]; });
        if ((rc = talloc(ctx, &t->l2p_order, ord.size(), s))) return rc;
        DDM_CUDA(ctx, cudaMemcpyAsync(t->l2p_order, ord.data(), ord.size() * sizeof(int),
                                      cudaMemcpyHostToDevice, s));
        DDM_CUDA(ctx, cudaStreamSynchronize(s));
      }
      DDM_CUDA(ctx, cudaFreeAsync(work, s));
    }
    t->l2p_lo = t->own_el_lo;
    t->l2p_hi = t->own_el_hi;
  }
  return DDM_OK;
}

// prepare the static L2P tables (called from fmm_workspace, outside captures)
int l2p_prepare(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) { return l2p_tables(ctx, t, s); }

// L2P of the owned elements into t->y_far (far-field stream): block-staged
// kernel by default, DDM_L2P_BLOCK=0 the thread-per-element kernel
int launch_l2p(ddm_ctx_s* ctx, ddm_tree_s* t, int ncomp, double gc, const PoroFar& pf,
               cudaStream_t s) {
  const int64_t lo = t->own_el_lo, hi = t->own_el_hi;
  if (hi <= lo) return DDM_OK;
  const CellGeom cg{t->x_min, t->y_min, t->W};
  static const bool blk_env = [] {
    const char* e = getenv("DDM_L2P_BLOCK");
    return !(e && e[0] == '0');
  }();
  // the runs must match the owned range (built by l2p_prepare, outside captures)
  const bool blk = blk_env && t->l2p_runs && t->l2p_lo == lo && t->l2p_hi == hi;
  const unsigned nb = nblk(hi - lo, 256);
  const unsigned nbb = nblk(hi - lo, kL2PThreads);
  const size_t shb = (size_t)(kL2PLeaves + kL2PW) * 2 * t->p * sizeof(double2);
  int rc = DDM_OK;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if (blk) {                                                                                  \
      if ((rc = set_smem(ctx, l2p_block_kernel<PT>, shb))) return rc;                           \
      DDM_CUDA(ctx, launch_pdl(use_pdl(t), l2p_block_kernel<PT>, nbb, kL2PThreads, shb, s,      \
                               (int64_t)lo, (int64_t)hi, ncomp, (const int4*)t->l2p_runs,       \
                               (const int*)t->l2p_order,                                        \
                               (const double4*)t->leaf_geo, (const double4*)t->w_geo,           \
                               (const int*)t->el_leaf,                                          \
                               (const int*)t->leaves, (const int*)t->c_level,                  \
                               (const int*)t->c_ix, (const int*)t->c_iy,                       \
                               (const double2*)t->local, (const int*)t->w_off,                 \
                               (const int*)t->w_idx, (const double2*)t->mpole, cg, t->p, gc,   \
                               pf, (const double*)t->ex, (const double*)t->ey,                 \
                               (const double*)t->ec, (const double*)t->es, t->y_far));         \
    } else {                                                                                    \
      DDM_CUDA(ctx, launch_pdl(use_pdl(t), l2p_kernel<PT>, nb, 256, 0, s, (int64_t)lo,          \
                               (int64_t)hi, ncomp, (const int*)t->el_leaf,                     \
                               (const int*)t->leaves, (const int*)t->c_level,                  \
                               (const int*)t->c_ix, (const int*)t->c_iy,                       \
                               (const double2*)t->local, (const int*)t->w_off,                 \
                               (const int*)t->w_idx, (const double2*)t->mpole, cg, t->p, gc,   \
                               pf, (const double*)t->ex, (const double*)t->ey,                 \
                               (const double*)t->ec, (const double*)t->es, t->y_far));         \
    }                                                                                           \
  } while (0)
  DDM_P_DISPATCH(t->p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// P2L of the owned leaves' X lists into t->local_x (elastic; D read through
// perm_in when given, as the early P2M)
int launch_p2l(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D, int ncomp,
               cudaStream_t s) {
  if (t->nx <= 0 || t->own_leaf_hi <= t->own_leaf_lo) return DDM_OK;
  int rc = DDM_OK;
  if (!t->local_x && (rc = talloc(ctx, &t->local_x, (size_t)t->nleaves * 2 * t->p, s))) return rc;
  const CellGeom cg{t->x_min, t->y_min, t->W};
  const size_t shp = (size_t)kPassWarps * 32 * 17 * sizeof(double2);
  const int nl = t->own_leaf_hi - t->own_leaf_lo;
#define DDM_L(PT)                                                                               \
  do {                                                                                          \
    if ((rc = set_smem(ctx, p2l_kernel<PT>, shp))) return rc;                                   \
    const int nb = pass_grid(ctx, (const void*)p2l_kernel<PT>, shp, nl);                         \
    p2l_kernel<PT><<<nb, kPassWarps * 32, shp, s>>>(t->own_leaf_lo, t->own_leaf_hi, t->x_off,   \
                                                    t->x_idx, t->leaves, t->c_level, t->c_ix,   \
                                                    t->c_iy, t->c_start, t->c_count, cg, t->p,  \
                                                    perm_in, D, ncomp, t->ex, t->ey, t->ea,     \
                                                    t->ec, t->es, t->local_x);                  \
  } while (0)
  DDM_P_DISPATCH(t->p, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_finalize(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, int ncomp, double gc,
                    const PoroFar& pf, double* y_user, double* y_sorted, cudaStream_t s) {
  (void)gc;
  (void)pf;
  if (hi <= lo) return DDM_OK;
  finalize_kernel<<<nblk(hi - lo, 256), 256, 0, s>>>(
      lo, hi, ncomp, t->el_leaf, t->leaves, t->c_start, t->c_count, t->item_off,
      reinterpret_cast<const double*>(t->part), t->y_far, t->perm, y_user, y_sorted);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

}  // namespace ddm
