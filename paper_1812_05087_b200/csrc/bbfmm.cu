// Chebyshev black-box FMM far field: the
// paper's own far-field engine, a second far field of ddm_matvec
// (mode DDM_BBFMM | n << 8, elastic).  PAPER.md §3.2:
//   S_n(xbar, x) = 1/n + (2/n) sum_{k=1}^{n-1} T_k(xbar) T_k(x)
//   P2M  W_m^I = sum_j b(y_j) S_n(ybar_m^I, y_j)                    (Eq.(p2l))
//   M2M  W_m^I = sum_J sum_m' W_m'^J S_n(ybar_m^I, ybar_m'^J)       (Eq.(m2m))
//   M2L  g_l^I = sum_{J in V(I)} sum_m K(xbar_l^I, ybar_m^J) W_m^J  (Eq.(m2l))
//   L2L  f_l^I = g_l^I + sum_l' f_l'^P S_n(xbar_l'^P, xbar_l^I)     (Eq.(l2l))
//   L2P  f(x)  = sum_l f_l^I S_n(xbar_l^I, x)
// with 2D cardinal functions as products of the 1D ones.  Kernel (reading
// R21): the constant-DD element as line integrals of the analytic point
// kernels k2 = (z - zeta)^-2 and k3 = (z - zeta)^-3 (three densities per
// element: rho1 = i G C B e, rho2 = i G C Q e, rho3 = 2 i G C B e conj(zeta - c)),
// giving Phi, Phi' and Psi~ = Psi + conj(c) Phi' (about each cell's centre c)
// at the Chebyshev nodes.  The segment integral of S_n times a density is
// n-point Gauss-Legendre along the element (exact for this polynomial degree).
//
// Every stage maps one thread to one (cell, Chebyshev node) pair: n^2 <= 64
// threads per cell, the cell's data read through L1 as warp broadcasts.  The
// M2L evaluates k2 and k3 at the node pairs on the fly (fp64 ALU: ~34
// instructions per node pair, no tables to stream).
#include <cmath>
#include <mutex>
#include <vector>

#include "kcommon.cuh"

namespace ddm {
namespace {

constexpr int kBBMaxN = 8;
__constant__ double c_bbT[kBBMaxN + 1][kBBMaxN][kBBMaxN];      // [n][i][k] T_k(xbar_i)
__constant__ double c_bbS[kBBMaxN + 1][2][kBBMaxN][kBBMaxN];   // [n][h][i][k] S_n(xbar_i, h-1/2 + xbar_k/2)
__constant__ double c_bbX[kBBMaxN + 1][kBBMaxN];               // [n][i] xbar_i
__constant__ double c_bbGx[kBBMaxN + 1][kBBMaxN];              // [n][g] Gauss-Legendre nodes
__constant__ double c_bbGw[kBBMaxN + 1][kBBMaxN];              // [n][g] Gauss-Legendre weights

// S_n(xbar_i, x) for i < N: T_0..T_{N-1}(x) by the recurrence, then the
// sums against T_k(xbar_i)
template <int N>
__device__ __forceinline__ void card_all(double x, double (&S)[N]) {
  double T[N];
  T[0] = 1.0;
  if (N > 1) T[1] = x;
#pragma unroll
  for (int k = 2; k < N; ++k) T[k] = fma(2.0 * x, T[k - 1], -T[k - 2]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 1; k < N; ++k) s = fma(c_bbT[N][i][k], T[k], s);
    S[i] = (1.0 + 2.0 * s) * (1.0 / N);
  }
}

__device__ __forceinline__ bool owns(int cs, int cn, int64_t lo, int64_t hi) {
  return cs + cn > lo && cs < hi;
}

// ---------------------------------------------------------------- P2M
// warp per leaf (Eq.(p2l)).  The leaf's (element, Gauss-Legendre point)
// pairs are taken 32 at a time: phase 1, lane = pair: the 1D cardinal values
// S_n(xbar_i, xi), S_n(xbar_k, eta) of its point and its three densities
// (times the quadrature weight) into shared memory; phase 2, lane = node
// m = i N + k (two rounds when N^2 > 32): W_m += sum_pairs Sx_i Sy_k c_pair.
template <int N>
struct BBP2MSmem {
  double sx[32][N], sy[32][N];
  double2 c1[32], c2[32], c3[32];
};

template <int N>
__global__ void __launch_bounds__(128)
bb_p2m_kernel(int nleaves, const int* __restrict__ leaves, const int* __restrict__ c_level,
              const int* __restrict__ c_ix, const int* __restrict__ c_iy,
              const int* __restrict__ c_start, const int* __restrict__ c_count, CellGeom cg,
              const double* __restrict__ D, int ncomp, const double* __restrict__ ex,
              const double* __restrict__ ey, const double* __restrict__ ea,
              const double* __restrict__ ec, const double* __restrict__ es, double gc,
              double2* __restrict__ bbw) {
  constexpr int NN = N * N;
  constexpr int NR = (NN + 31) / 32;
  __shared__ BBP2MSmem<N> sm_all[4];
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (k >= nleaves) return;
  BBP2MSmem<N>& sm = sm_all[threadIdx.x >> 5];
  const int c = leaves[k];
  const int lev = c_level[c];
  const double hs = 0.5 * cg.side(lev), ihs = 1.0 / hs;
  const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
  const int e0 = c_start[c], npair = c_count[c] * N;
  double2 w1[NR], w2[NR], w3[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) w1[r] = w2[r] = w3[r] = make_double2(0, 0);
  for (int p0 = 0; p0 < npair; p0 += 32) {
    const int pr = p0 + lane;
    if (pr < npair) {
      const int e = e0 + pr / N, g = pr % N;
      const double ds = D[(int64_t)e * ncomp], dn = D[(int64_t)e * ncomp + 1];
      const double cb = ec[e], sb = es[e], a = ea[e];
      const double2 eb = make_double2(cb, sb);
      const double2 B = make_double2(ds * cb - dn * sb, ds * sb + dn * cb);
      const double2 r = make_double2(cb * cb - sb * sb, -2.0 * cb * sb);
      const double2 Q = csub(cmul(r, B), cconj(B));
      const double tg = c_bbGx[N][g], wa = c_bbGw[N][g] * a;
      const double xi = fma(tg, a * cb * ihs, (ex[e] - z0.x) * ihs);
      const double eta = fma(tg, a * sb * ihs, (ey[e] - z0.y) * ihs);
      double Sx[N], Sy[N];
      card_all<N>(xi, Sx);
      card_all<N>(eta, Sy);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        sm.sx[lane][i] = Sx[i];
        sm.sy[lane][i] = Sy[i];
      }
      // densities / (i gc) times wg a:  Be, Qe, 2 Be conj(zeta - c) = 2 hs Be (xi - i eta)
      const double2 Be = cmul(B, eb);
      sm.c1[lane] = cscale(Be, wa);
      sm.c2[lane] = cscale(cmul(Q, eb), wa);
      sm.c3[lane] = cscale(cmul(Be, make_double2(xi, -eta)), 2.0 * hs * wa);
    }
    __syncwarp();
    const int np = min(32, npair - p0);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m < NN) {
        const int mi = m / N, mk = m % N;
        for (int q = 0; q < np; ++q) {
          const double S = sm.sx[q][mi] * sm.sy[q][mk];
          const double2 v1 = sm.c1[q], v2 = sm.c2[q], v3 = sm.c3[q];
          w1[r].x = fma(S, v1.x, w1[r].x); w1[r].y = fma(S, v1.y, w1[r].y);
          w2[r].x = fma(S, v2.x, w2[r].x); w2[r].y = fma(S, v2.y, w2[r].y);
          w3[r].x = fma(S, v3.x, w3[r].x); w3[r].y = fma(S, v3.y, w3[r].y);
        }
      }
    }
    __syncwarp();
  }
  // times i gc
  double2* W = bbw + (size_t)c * 3 * NN;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int m = lane + 32 * r;
    if (m < NN) {
      W[m] = make_double2(-gc * w1[r].y, gc * w1[r].x);
      W[NN + m] = make_double2(-gc * w2[r].y, gc * w2[r].x);
      W[2 * NN + m] = make_double2(-gc * w3[r].y, gc * w3[r].x);
    }
  }
}

// ---------------------------------------------------------------- M2M / L2L
// Both are the 2D interpolation between a parent's nodes and a child's nodes,
// a product of two 1D N x N matrices (c_bbS), applied separably (2 N^3 per
// density instead of N^4) by one warp per cell through shared memory.
template <int N>
struct BBTransSmem {
  double2 a[3][N * N], b[3][N * N];
};

// dst[d][i*N + l] = sum_k M[i][k] src[d][k*N + l]   (first index)   when FIRST,
// dst[d][i*N + l] = sum_k M[l][k] src[d][i*N + k]   (second index)  otherwise;
// M(i, k) = S[h][i][k] (M2M, parent node i <- child node k) or S[h][k][i] (L2L)
template <int N, bool FIRST, bool TRANS>
__device__ __forceinline__ void bb_pass(const double (*S)[N][N], int h, const double2 (*src)[N * N],
                                        double2 (*dst)[N * N], int lane) {
  constexpr int NN = N * N;
  for (int m = lane; m < NN; m += 32) {
    const int i = m / N, l = m % N;
    const int row = FIRST ? i : l;
    double2 t[3] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const double M = TRANS ? S[h][k][row] : S[h][row][k];
      const int q = FIRST ? k * N + l : i * N + k;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        t[d].x = fma(M, src[d][q].x, t[d].x);
        t[d].y = fma(M, src[d][q].y, t[d].y);
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) dst[d][m] = t[d];
  }
}

template <int N>
__device__ __forceinline__ void bb_stage_S(double (*sS)[N][N]) {
  for (int f = threadIdx.x; f < 2 * N * N; f += blockDim.x)
    sS[f / (N * N)][(f / N) % N][f % N] = c_bbS[N][f / (N * N)][(f / N) % N][f % N];
  __syncthreads();
}

// warp per parent of one level (Eq.(m2m)); the third weight re-centred on
// the parent: w3 += 2 conj(c_child - c_parent) w1
template <int N>
__global__ void __launch_bounds__(128)
bb_m2m_level_kernel(int u0, int u1, const int* __restrict__ up_list,
                    const int* __restrict__ c_level, const int* __restrict__ c_ix,
                    const int* __restrict__ c_iy, const int* __restrict__ c_first_child,
                    const int* __restrict__ c_nchild, CellGeom cg, double2* __restrict__ bbw) {
  constexpr int NN = N * N;
  __shared__ double sS[2][N][N];
  __shared__ BBTransSmem<N> sm_all[4];
  bb_stage_S<N>(sS);
  const int lane = threadIdx.x & 31;
  const int idx = u0 + blockIdx.x * 4 + (threadIdx.x >> 5);
  if (idx >= u1) return;
  BBTransSmem<N>& sm = sm_all[threadIdx.x >> 5];
  const int P = up_list[idx];
  const double q4 = 0.25 * cg.side(c_level[P]);
  constexpr int NR = (NN + 31) / 32;
  double2 acc[3][NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) acc[0][r] = acc[1][r] = acc[2][r] = make_double2(0, 0);
  for (int q = c_first_child[P], q1 = q + c_nchild[P]; q < q1; ++q) {
    const int hx = c_ix[q] & 1, hy = c_iy[q] & 1;
    // 2 conj(c_q - c_P) = 2 q4 ((2hx - 1) - i (2hy - 1))
    const double2 sh = make_double2(2.0 * q4 * (2 * hx - 1), -2.0 * q4 * (2 * hy - 1));
    const double2* Wq = bbw + (size_t)q * 3 * NN;
    for (int m = lane; m < NN; m += 32) {
      const double2 v1 = Wq[m];
      sm.a[0][m] = v1;
      sm.a[1][m] = Wq[NN + m];
      sm.a[2][m] = cadd(Wq[2 * NN + m], cmul(sh, v1));
    }
    __syncwarp();
    bb_pass<N, true, false>(sS, hx, sm.a, sm.b, lane);    // parent x-node <- child x-node
    __syncwarp();
    bb_pass<N, false, false>(sS, hy, sm.b, sm.a, lane);   // parent y-node <- child y-node
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m < NN)
        for (int d = 0; d < 3; ++d) acc[d][r] = cadd(acc[d][r], sm.a[d][m]);
    }
    __syncwarp();
  }
  double2* W = bbw + (size_t)P * 3 * NN;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int m = lane + 32 * r;
    if (m < NN)
      for (int d = 0; d < 3; ++d) W[d * NN + m] = acc[d][r];
  }
}

// node-pair kernel sums of one source cell's weights at the point u (units of
// the source half-side hs, relative to the source centre):
//   t1 = sum k2 w1, t3 = sum k3 w1, t2a = sum k2 w2, t2b = sum k3 w3
// with k2 = delta^-2, k3 = delta^-3, delta = u - ubar_m
template <int N>
__device__ __forceinline__ void node_sums(double2 u, const double2* __restrict__ Wb, double2& t1,
                                          double2& t3, double2& t2a, double2& t2b) {
  constexpr int NN = N * N;
  double dyk[N];
#pragma unroll
  for (int k = 0; k < N; ++k) dyk[k] = u.y - c_bbX[N][k];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double dx = u.x - c_bbX[N][i], dx2 = dx * dx;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int mm = i * N + k;
      const double dy = dyk[k];
      const double r = fast_rcp(fma(dy, dy, dx2));
      const double2 inv = make_double2(dx * r, -dy * r);
      const double2 inv2 = make_double2(fma(inv.x, inv.x, -inv.y * inv.y), 2.0 * inv.x * inv.y);
      const double2 inv3 = cmul(inv2, inv);
      const double2 v1 = Wb[mm], v2 = Wb[NN + mm], v3 = Wb[2 * NN + mm];
      cmac(t1, inv2, v1);
      cmac(t3, inv3, v1);
      cmac(t2a, inv2, v2);
      cmac(t2b, inv3, v3);
    }
  }
}

// ---------------------------------------------------------------- M2L
// thread = (cell of level >= 2 holding owned targets, node l): Eq.(m2l) at
// the node, over the cell's V list (same level, so one half-side h):
//   Phi = h^-2 sum t1,  Phi' = -2 h^-3 sum t3,
//   Psi~ = sum [h^-2 t2a + h^-3 t2b + 2 conj(c_b - c_c) h^-3 t3]
template <int N>
__global__ void __launch_bounds__(128)
bb_m2l_kernel(int c0, int c1, int64_t own_lo, int64_t own_hi, const int* __restrict__ v_off,
              const int* __restrict__ v_idx, const int* __restrict__ c_level,
              const int* __restrict__ c_ix, const int* __restrict__ c_iy,
              const int* __restrict__ c_start, const int* __restrict__ c_count, CellGeom cg,
              const double2* __restrict__ bbw, double2* __restrict__ bbf) {
  constexpr int NN = N * N;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int c = c0 + (int)(gid / NN);
  if (c >= c1) return;
  if (!owns(c_start[c], c_count[c], own_lo, own_hi)) return;
  const int m = (int)(gid % NN);
  const double h = 0.5 * cg.side(c_level[c]), ih = 1.0 / h;
  const double ul_x = c_bbX[N][m / N], ul_y = c_bbX[N][m % N];
  const int ixc = c_ix[c], iyc = c_iy[c];
  double2 phi = make_double2(0, 0), dphi = phi, psa = phi, psb = phi;
  for (int vi = v_off[c], ve = v_off[c + 1]; vi < ve; ++vi) {
    const int b = v_idx[vi];
    const int dx = c_ix[b] - ixc, dy = c_iy[b] - iyc;
    // target node relative to the source centre, in units of h: -2 (dx, dy) + ul
    const double2 u = make_double2(ul_x - 2.0 * dx, ul_y - 2.0 * dy);
    double2 t1 = make_double2(0, 0), t3 = t1, t2a = t1, t2b = t1;
    node_sums<N>(u, bbw + (size_t)b * 3 * NN, t1, t3, t2a, t2b);
    phi = cadd(phi, t1);
    dphi = cadd(dphi, t3);
    // 2 conj(c_b - c_c) h^-3 = 4 (dx - i dy) h^-2
    psa = cadd(psa, cadd(t2a, cmul(make_double2(4.0 * dx, -4.0 * dy), t3)));
    psb = cadd(psb, t2b);
  }
  const double ih2 = ih * ih, ih3 = ih2 * ih;
  double2* F = bbf + (size_t)c * 3 * NN;
  F[m] = cscale(phi, ih2);
  F[NN + m] = cscale(dphi, -2.0 * ih3);
  F[2 * NN + m] = cadd(cscale(psa, ih2), cscale(psb, ih3));
}

// ---------------------------------------------------------------- L2L
// warp per cell of one level >= 3 holding owned targets (Eq.(l2l)): the
// parent's node values, Psi~ re-centred on the child (Psi~ + conj(c_c - c_P)
// Phi'), interpolated at the child's nodes and added to its M2L result
template <int N>
__global__ void __launch_bounds__(128)
bb_l2l_level_kernel(int a, int b, int64_t own_lo, int64_t own_hi, const int* __restrict__ c_level,
                    const int* __restrict__ c_ix, const int* __restrict__ c_iy,
                    const int* __restrict__ c_start, const int* __restrict__ c_count,
                    const int* __restrict__ c_parent, CellGeom cg, double2* __restrict__ bbf) {
  constexpr int NN = N * N;
  __shared__ double sS[2][N][N];
  __shared__ BBTransSmem<N> sm_all[4];
  bb_stage_S<N>(sS);
  const int lane = threadIdx.x & 31;
  const int c = a + blockIdx.x * 4 + (threadIdx.x >> 5);
  if (c >= b) return;
  if (!owns(c_start[c], c_count[c], own_lo, own_hi)) return;
  BBTransSmem<N>& sm = sm_all[threadIdx.x >> 5];
  const int P = c_parent[c];
  const int hx = c_ix[c] & 1, hy = c_iy[c] & 1;
  // conj(c_c - c_P) = s_c/2 ((2hx - 1) - i (2hy - 1))
  const double hc = 0.5 * cg.side(c_level[c]);
  const double2 sh = make_double2(hc * (2 * hx - 1), -hc * (2 * hy - 1));
  const double2* FP = bbf + (size_t)P * 3 * NN;
  for (int m = lane; m < NN; m += 32) {
    const double2 v2 = FP[NN + m];
    sm.a[0][m] = FP[m];
    sm.a[1][m] = v2;
    sm.a[2][m] = cadd(FP[2 * NN + m], cmul(sh, v2));
  }
  __syncwarp();
  bb_pass<N, true, true>(sS, hx, sm.a, sm.b, lane);    // child x-node <- parent x-node
  __syncwarp();
  bb_pass<N, false, true>(sS, hy, sm.b, sm.a, lane);   // child y-node <- parent y-node
  __syncwarp();
  double2* F = bbf + (size_t)c * 3 * NN;
  for (int m = lane; m < NN; m += 32)
    for (int d = 0; d < 3; ++d) F[d * NN + m] = cadd(F[d * NN + m], sm.a[d][m]);
}

// ---------------------------------------------------------------- L2P + W
// thread per owned element: interpolation of the leaf's node values at the
// element centre, plus the W cells' weights evaluated at it (node-to-point
// Eq.(m2l)); T = 2 Re Phi + e^{2 i b} (conj(z - c) Phi' + Psi~),
// y_far = (Im T, Re T) = (sigma_s, sigma_n), sorted order
template <int N>
__global__ void __launch_bounds__(128)
bb_l2p_kernel(int64_t e_lo, int64_t e_hi, int ncomp, const int* __restrict__ el_leaf,
              const int* __restrict__ leaves, const int* __restrict__ c_level,
              const int* __restrict__ c_ix, const int* __restrict__ c_iy,
              const double2* __restrict__ bbf, const int* __restrict__ w_off,
              const int* __restrict__ w_idx, const double2* __restrict__ bbw, CellGeom cg,
              const double* __restrict__ ex, const double* __restrict__ ey,
              const double* __restrict__ ec, const double* __restrict__ es,
              double* __restrict__ y_far) {
  constexpr int NN = N * N;
  const int64_t i = e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= e_hi) return;
  const int k = el_leaf[i];
  const int c = leaves[k];
  const int lev = c_level[c];
  const double x = ex[i], y = ey[i];
  const double h = 0.5 * cg.side(lev);
  const double2 z0 = cg.centre(lev, c_ix[c], c_iy[c]);
  double2 phi = make_double2(0, 0), dphi = phi, psi = phi;
  if (lev >= 2) {
    double Sx[N], Sy[N];
    card_all<N>((x - z0.x) / h, Sx);
    card_all<N>((y - z0.y) / h, Sy);
    const double2* F = bbf + (size_t)c * 3 * NN;
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double2 t1 = make_double2(0, 0), t2 = t1, t3 = t1;
#pragma unroll
      for (int bq = 0; bq < N; ++bq) {
        const int mm = a * N + bq;
        const double S = Sy[bq];
        const double2 v1 = F[mm], v2 = F[NN + mm], v3 = F[2 * NN + mm];
        t1.x = fma(S, v1.x, t1.x); t1.y = fma(S, v1.y, t1.y);
        t2.x = fma(S, v2.x, t2.x); t2.y = fma(S, v2.y, t2.y);
        t3.x = fma(S, v3.x, t3.x); t3.y = fma(S, v3.y, t3.y);
      }
      phi.x = fma(Sx[a], t1.x, phi.x); phi.y = fma(Sx[a], t1.y, phi.y);
      dphi.x = fma(Sx[a], t2.x, dphi.x); dphi.y = fma(Sx[a], t2.y, dphi.y);
      psi.x = fma(Sx[a], t3.x, psi.x); psi.y = fma(Sx[a], t3.y, psi.y);
    }
  }
  for (int wi = w_off[k], we = w_off[k + 1]; wi < we; ++wi) {
    const int Dc = w_idx[wi];
    const int ld = c_level[Dc];
    const double hd = 0.5 * cg.side(ld), ihd = 1.0 / hd;
    const double2 zd = cg.centre(ld, c_ix[Dc], c_iy[Dc]);
    const double2 u = make_double2((x - zd.x) * ihd, (y - zd.y) * ihd);
    double2 t1 = make_double2(0, 0), t3 = t1, t2a = t1, t2b = t1;
    node_sums<N>(u, bbw + (size_t)Dc * 3 * NN, t1, t3, t2a, t2b);
    const double i2 = ihd * ihd, i3 = i2 * ihd;
    phi = cadd(phi, cscale(t1, i2));
    dphi = cadd(dphi, cscale(t3, -2.0 * i3));
    // Psi~ about z0: + 2 conj(zd - z0) k3 w1
    const double2 sh = make_double2(2.0 * (zd.x - z0.x), -2.0 * (zd.y - z0.y));
    psi = cadd(psi, cadd(cscale(t2a, i2), cscale(cadd(t2b, cmul(sh, t3)), i3)));
  }
  const double2 T = cadd(make_double2(2.0 * phi.x, 0.0),
                         cmul(make_double2(ec[i] * ec[i] - es[i] * es[i], 2.0 * ec[i] * es[i]),
                              cadd(cmul(make_double2(x - z0.x, z0.y - y), dphi), psi)));
  y_far[i * ncomp + 0] = T.y;
  y_far[i * ncomp + 1] = T.x;
  if (ncomp == 3) y_far[i * ncomp + 2] = 0.0;
}

// ---------------------------------------------------------------- tables
// host, long double: Chebyshev nodes, T_k at the nodes, the child-node
// cardinal matrices of M2M / L2L, Gauss-Legendre rules (Newton on P_n)
std::mutex g_bb_mu;
std::vector<int> g_bb_dev;

int bb_init_tables(ddm_ctx_s* ctx) {
  std::lock_guard<std::mutex> lk(g_bb_mu);
  for (int d : g_bb_dev)
    if (d == ctx->device) return DDM_OK;
  static double T[kBBMaxN + 1][kBBMaxN][kBBMaxN], S[kBBMaxN + 1][2][kBBMaxN][kBBMaxN],
      X[kBBMaxN + 1][kBBMaxN], Gx[kBBMaxN + 1][kBBMaxN], Gw[kBBMaxN + 1][kBBMaxN];
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int n = 1; n <= kBBMaxN; ++n) {
    long double xb[kBBMaxN];
    for (int i = 0; i < n; ++i) {
      xb[i] = cosl((2.0L * (i + 1) - 1.0L) * pi / (2.0L * n));
      X[n][i] = (double)xb[i];
      for (int k = 0; k < n; ++k) T[n][i][k] = (double)cosl(k * acosl(xb[i]));
    }
    auto card = [&](int i, long double x) {
      long double s = 1.0L / n, tkm = 1.0L, tk = x;
      for (int k = 1; k < n; ++k) {
        s += 2.0L / n * cosl(k * acosl(xb[i])) * tk;
        const long double tn = 2.0L * x * tk - tkm;
        tkm = tk;
        tk = tn;
      }
      return s;
    };
    for (int hh = 0; hh < 2; ++hh)
      for (int i = 0; i < n; ++i)
        for (int k = 0; k < n; ++k)
          S[n][hh][i][k] = (double)card(i, (hh - 0.5L) + 0.5L * xb[k]);
    for (int g = 0; g < n; ++g) {
      long double x = cosl(pi * (g + 0.75L) / (n + 0.5L)), dp = 1.0L;
      for (int it = 0; it < 100; ++it) {
        long double p0 = 1.0L, p1 = x;
        for (int j = 2; j <= n; ++j) {
          const long double p2 = ((2.0L * j - 1.0L) * x * p1 - (j - 1.0L) * p0) / j;
          p0 = p1;
          p1 = p2;
        }
        if (n == 1) { p1 = x; p0 = 1.0L; }
        dp = n * (x * p1 - p0) / (x * x - 1.0L);
        const long double dx = p1 / dp;
        x -= dx;
        if (fabsl(dx) < 1e-30L) break;
      }
      Gx[n][g] = (double)x;
      Gw[n][g] = (double)(2.0L / ((1.0L - x * x) * dp * dp));
    }
  }
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_bbT, T, sizeof(T)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_bbS, S, sizeof(S)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_bbX, X, sizeof(X)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_bbGx, Gx, sizeof(Gx)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_bbGw, Gw, sizeof(Gw)));
  g_bb_dev.push_back(ctx->device);
  return DDM_OK;
}

#define DDM_BB_DISPATCH(n, F) \
  switch (n) {                \
    case 2: F(2); break;      \
    case 3: F(3); break;      \
    case 4: F(4); break;      \
    case 5: F(5); break;      \
    case 6: F(6); break;      \
    case 7: F(7); break;      \
    case 8: F(8); break;      \
    default: break;           \
  }

}  // namespace

int bb_prepare(ddm_ctx_s* ctx, ddm_tree_s* t, int n) {
  if (n < 2 || n > kBBMaxN) return set_error(ctx, DDM_ERR_ARG, "bbFMM needs 2 <= n <= 8 nodes");
  int rc = bb_init_tables(ctx);
  if (rc) return rc;
  if (t->bb_n != n) {
    drop_graphs(t);   // captured bbFMM graphs hold the old node arrays
    if (t->bb_w) cudaFree(t->bb_w);
    if (t->bb_f) cudaFree(t->bb_f);
    t->bb_w = t->bb_f = nullptr;
    t->bb_n = 0;
    if ((rc = dalloc(ctx, &t->bb_w, (size_t)t->ncells * 3 * n * n))) return rc;
    if ((rc = dalloc(ctx, &t->bb_f, (size_t)t->ncells * 3 * n * n))) return rc;
    t->bb_n = n;
  }
  return DDM_OK;
}

// far chain of the bbFMM (P2M, M2M per level, M2L, L2L per level, L2P + W)
// into t->y_far; D in sorted order [n][ncomp]
int launch_bb_far(ddm_ctx_s* ctx, ddm_tree_s* t, int n, const double* D, int ncomp, double gc,
                  cudaStream_t s) {
  const CellGeom cg{t->x_min, t->y_min, t->W};
  const int64_t lo = t->own_el_lo, hi = t->own_el_hi;
  const int NN = n * n;
#define DDM_L(NT)                                                                               \
  do {                                                                                          \
    stage_begin(ctx, DDM_ST_P2M, s);                                                            \
    bb_p2m_kernel<NT><<<nblk(t->nleaves, 4), 128, 0, s>>>(                      \
        t->nleaves, t->leaves, t->c_level, t->c_ix, t->c_iy, t->c_start, t->c_count, cg, D,     \
        ncomp, t->ex, t->ey, t->ea, t->ec, t->es, gc, t->bb_w);                                 \
    stage_end(ctx, DDM_ST_P2M, s);                                                              \
    stage_begin(ctx, DDM_ST_M2M, s);                                                            \
    for (int lev = t->nlevels - 1; lev >= 2; --lev) {                                           \
      const int u0 = t->up_level_off[2 * lev], u1 = t->up_level_off[2 * lev + 1];               \
      if (u1 <= u0) continue;                                                                   \
      bb_m2m_level_kernel<NT><<<nblk(u1 - u0, 4), 128, 0, s>>>(               \
          u0, u1, t->up_list, t->c_level, t->c_ix, t->c_iy, t->c_first_child, t->c_nchild, cg,  \
          t->bb_w);                                                                             \
    }                                                                                           \
    stage_end(ctx, DDM_ST_M2M, s);                                                              \
    if (t->nlevels > 2) {                                                                       \
      const int c0 = t->level_off[2], c1 = t->ncells;                                           \
      stage_begin(ctx, DDM_ST_M2L, s);                                                          \
      bb_m2l_kernel<NT><<<nblk((int64_t)(c1 - c0) * NN, 128), 128, 0, s>>>(                     \
          c0, c1, lo, hi, t->v_off, t->v_idx, t->c_level, t->c_ix, t->c_iy, t->c_start,         \
          t->c_count, cg, t->bb_w, t->bb_f);                                                    \
      stage_end(ctx, DDM_ST_M2L, s);                                                            \
      stage_begin(ctx, DDM_ST_L2L, s);                                                          \
      for (int lev = 3; lev < t->nlevels; ++lev) {                                              \
        const int a = t->level_off[lev], b = t->level_off[lev + 1];                             \
        if (b <= a) continue;                                                                   \
        bb_l2l_level_kernel<NT><<<nblk(b - a, 4), 128, 0, s>>>(               \
            a, b, lo, hi, t->c_level, t->c_ix, t->c_iy, t->c_start, t->c_count, t->c_parent,    \
            cg, t->bb_f);                                                                       \
      }                                                                                         \
      stage_end(ctx, DDM_ST_L2L, s);                                                            \
    }                                                                                           \
    if (hi > lo) {                                                                              \
      stage_begin(ctx, DDM_ST_L2P, s);                                                          \
      bb_l2p_kernel<NT><<<nblk(hi - lo, 128), 128, 0, s>>>(                                     \
          lo, hi, ncomp, t->el_leaf, t->leaves, t->c_level, t->c_ix, t->c_iy, t->bb_f,          \
          t->w_off, t->w_idx, t->bb_w, cg, t->ex, t->ey, t->ec, t->es, t->y_far);               \
      stage_end(ctx, DDM_ST_L2P, s);                                                            \
    }                                                                                           \
  } while (0)
  DDM_BB_DISPATCH(n, DDM_L);
#undef DDM_L
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

}  // namespace ddm
