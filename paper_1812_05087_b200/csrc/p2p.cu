// Near field (a10) and direct evaluation of the elastic constant-DD kernel
// (rows a5-prep and a10).  The exact element influence is
// evaluated in Kolosov–Muskhelishvili form: "the direct
// multiplication ... is used for points that are not well-separated"
// (P:536-538), "P2P term, to account for the self and neighbor interactions"
// (P:868-877).
#include <algorithm>

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

// ---------------------------------------------------------------- stream
// Near-field source stream.  Constant DD elements of one
// fracture share their end nodes, and I2 = r2 - r1 only needs the reciprocal
// r = 1/(z - node) of each NODE: an element whose first node is the previous
// element's second node reuses that reciprocal.  The elements of each leaf are
// therefore reordered along chains of node-sharing elements (a permutation
// within the leaf, so every U-list range [lo, hi) of sorted elements is the
// same range of stream slots); a chain start is preceded by a break record
// (its first node, zero coefficients).  Record of slot q:
//   {second node, P1, P2, Bh, Q'} (x sign: a flipped element, first node =
//   z2, has I2 negated, so its coefficients are negated), 10 doubles.
// Node sharing is decided by coordinates equal up to 8 ulp of the coordinate
// magnitude; the shared node is then the previous element's computed node,
// an O(ulp) change of the element's own endpoint (reading R22).

__device__ __forceinline__ double2 end_node(const double* ex, const double* ey,
                                            const double* ea, const double* ec,
                                            const double* es, int i, int ep) {
  const double a = ep ? ea[i] : -ea[i];
  return make_double2(ex[i] + a * ec[i], ey[i] + a * es[i]);
}

// Thread per leaf: node-sharing neighbours (O(count^2) endpoint matching),
// then chains walked from their free ends in sorted-index order (closed loops
// last).  st_code bit 0: flipped, bit 1: linked to the previous slot.
__global__ void chain_order_kernel(int nleaves, const int* __restrict__ leaves,
                                   const int* __restrict__ c_start,
                                   const int* __restrict__ c_count, const double* __restrict__ ex,
                                   const double* __restrict__ ey, const double* __restrict__ ea,
                                   const double* __restrict__ ec, const double* __restrict__ es,
                                   int* __restrict__ st_elem, unsigned char* __restrict__ st_code) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int c = leaves[k];
  const int cs = c_start[c], cnt = c_count[c];
  if (cnt > kChainMax) {   // Morton order, every element a chain of its own
    for (int i = 0; i < cnt; ++i) {
      st_elem[cs + i] = cs + i;
      st_code[cs + i] = 0;
    }
    return;
  }
  // nb[i][ep] = 2 j + ep_j of the element endpoint coinciding with (i, ep), or -1
  short nb[kChainMax][2];
  unsigned char vis[kChainMax];
  for (int i = 0; i < cnt; ++i) {
    nb[i][0] = nb[i][1] = -1;
    vis[i] = 0;
  }
  const double eps8 = 8.0 * 2.220446049250313e-16;
  for (int i = 0; i < cnt; ++i)
    for (int ei = 0; ei < 2; ++ei) {
      if (nb[i][ei] >= 0) continue;
      const double2 p = end_node(ex, ey, ea, ec, es, cs + i, ei);
      const double tol = eps8 * (fabs(p.x) + fabs(p.y));
      for (int j = i + 1; j < cnt && nb[i][ei] < 0; ++j)
        for (int ej = 0; ej < 2; ++ej) {
          if (nb[j][ej] >= 0) continue;
          const double2 q = end_node(ex, ey, ea, ec, es, cs + j, ej);
          if (fabs(p.x - q.x) <= tol && fabs(p.y - q.y) <= tol) {
            nb[i][ei] = (short)(2 * j + ej);
            nb[j][ej] = (short)(2 * i + ei);
            break;
          }
        }
    }
  int out = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int s0 = 0; s0 < cnt; ++s0) {
      if (vis[s0]) continue;
      if (pass == 0 && nb[s0][0] >= 0 && nb[s0][1] >= 0) continue;   // interior of a chain
      int cur = s0, first = (pass == 0 && nb[s0][0] >= 0) ? 1 : 0;
      bool link = false;
      while (true) {
        vis[cur] = 1;
        st_elem[cs + out] = cs + cur;
        st_code[cs + out] = (unsigned char)((first ? 1 : 0) | (link ? 2 : 0));
        ++out;
        const int n = nb[cur][1 - first];
        if (n < 0 || vis[n >> 1]) break;
        cur = n >> 1;
        first = n & 1;
        link = true;
      }
    }
}

__global__ void chain_count_kernel(int64_t n, const unsigned char* __restrict__ st_code,
                                   int* __restrict__ cntv) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) cntv[q] = (st_code[q] & 2) ? 1 : 2;
}

// break records (first node, zero coefficients) of the unlinked slots, and
// the pad record 0 (a node far outside the tree, zero coefficients)
__global__ void break_records_kernel(int64_t n, const int* __restrict__ st_elem,
                                     const unsigned char* __restrict__ st_code,
                                     const int* __restrict__ rbeg, const double* __restrict__ ex,
                                     const double* __restrict__ ey, const double* __restrict__ ea,
                                     const double* __restrict__ ec, const double* __restrict__ es,
                                     double2 pad, double* __restrict__ srec) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q == 0) {
    double2* o = reinterpret_cast<double2*>(srec);
    o[0] = pad;
    for (int f = 1; f < kRecStride / 2; ++f) o[f] = make_double2(0.0, 0.0);
  }
  if (q >= n) return;
  const unsigned char code = st_code[q];
  if (code & 2) return;
  double2* o = reinterpret_cast<double2*>(srec + (int64_t)rbeg[q] * kRecStride);
  o[0] = end_node(ex, ey, ea, ec, es, st_elem[q], code & 1);
  for (int f = 1; f < kRecStride / 2; ++f) o[f] = make_double2(0.0, 0.0);
}

// Record ranges of every P2P item: the item's window [item.z, item.w) of
// its leaf's concatenated U ranges, mapped to stream records (rbeg).  One
// entry per intersecting U range; the P2P kernel reads one int2 per range
// instead of chasing u_lo/u_hi -> rbeg -> records.
__global__ void item_rng_count(int nitems, const int4* __restrict__ items,
                               const int* __restrict__ u_off, const int* __restrict__ u_lo,
                               const int* __restrict__ u_hi, int* __restrict__ cnt) {
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it > nitems) return;
  if (it == nitems) {
    cnt[it] = 0;
    return;
  }
  const int4 item = items[it];
  int pos = 0, n = 0;
  for (int r = u_off[item.x], rend = u_off[item.x + 1]; r < rend && pos < item.w; ++r) {
    const int len = u_hi[r] - u_lo[r];
    const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
    if (b < e) ++n;
    pos += len;
  }
  cnt[it] = n;
}

__global__ void item_rng_fill(int nitems, const int4* __restrict__ items,
                              const int* __restrict__ u_off, const int* __restrict__ u_lo,
                              const int* __restrict__ u_hi, const int* __restrict__ rbeg,
                              const int* __restrict__ roff, int2* __restrict__ rng) {
  const int it = blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= nitems) return;
  const int4 item = items[it];
  int pos = 0, o = roff[it];
  for (int r = u_off[item.x], rend = u_off[item.x + 1]; r < rend && pos < item.w; ++r) {
    const int lo = u_lo[r], len = u_hi[r] - lo;
    const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
    if (b < e) rng[o++] = make_int2(rbeg[lo + b], rbeg[lo + e]);
    pos += len;
  }
}

// Per stream slot (every matvec): the element's record from its DDs,
//   B = (D_s + i D_n) e, r = conj(e)^2, Bh = B/2, Q' = -(r B + conj B),
//   P1 = Bh (r - 1), P2 = i Bh (r + 1)   (negated for a flipped element)
// and D gathered to sorted order for the upward pass.
__global__ void prep_stream(int64_t q_lo, int64_t n, const int2* __restrict__ hrng,
                            const int64_t* __restrict__ hpre, int nh, int ncomp,
                            const int* __restrict__ perm,
                            const int* __restrict__ st_elem,
                            const unsigned char* __restrict__ st_code,
                            const int* __restrict__ rbeg, const double* __restrict__ D,
                            const double* __restrict__ ex, const double* __restrict__ ey,
                            const double* __restrict__ ea, const double* __restrict__ ec,
                            const double* __restrict__ es, double* __restrict__ srec,
                            double* __restrict__ dsort) {
  int64_t q = q_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  if (hrng) {   // q numbers the slots of the merged halo ranges
    int lo = 0, hi = nh - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (hpre[mid] <= q) lo = mid; else hi = mid - 1;
    }
    q = hrng[lo].x + (q - hpre[lo]);
  }
  const int i = st_elem[q];
  const unsigned char code = st_code[q];
  const int j = perm ? perm[i] : i;
  const double ds = D[(int64_t)j * ncomp + 0];
  const double dn = D[(int64_t)j * ncomp + 1];
  if (dsort) {
    dsort[(int64_t)i * ncomp + 0] = ds;
    dsort[(int64_t)i * ncomp + 1] = dn;
  }
  const double c = ec[i], s = es[i];
  const double sg = (code & 1) ? -1.0 : 1.0;
  const double2 B = make_double2(ds * c - dn * s, ds * s + dn * c);
  const double2 r = make_double2(c * c - s * s, -2.0 * c * s);
  const double2 rB = cmul(r, B);
  const double2 Bh = make_double2(0.5 * sg * B.x, 0.5 * sg * B.y);
  const double2 P1 = cmul(Bh, make_double2(r.x - 1.0, r.y));
  const double2 T2 = cmul(Bh, make_double2(r.x + 1.0, r.y));
  double2* o = reinterpret_cast<double2*>(srec + (int64_t)(rbeg[q] + ((code & 2) ? 0 : 1)) * kRecStride);
  o[0] = end_node(ex, ey, ea, ec, es, i, (code & 1) ? 0 : 1);   // second node
#if DDM_REC_K
  // 2 (z - zc).x P1 + 2 (z - zc).y P2 = z.x P1' + z.y P2' - K with P1' = 2 P1,
  // P2' = 2 P2, K = zc.x P1' + zc.y P2' (zc = the element centre)
  const double2 P1d = make_double2(2.0 * P1.x, 2.0 * P1.y);
  const double2 P2d = make_double2(-2.0 * T2.y, 2.0 * T2.x);   // 2 P2 = 2 i Bh (r + 1)
  const double xc = ex[i], yc = ey[i];
  o[1] = P1d;
  o[2] = P2d;
  o[3] = Bh;
  o[4] = make_double2(-sg * (rB.x + B.x), -sg * (rB.y - B.y));   // Q'
  o[5] = make_double2(fma(xc, P1d.x, yc * P2d.x), fma(xc, P1d.y, yc * P2d.y));   // K
#else
  o[1] = P1;
  o[2] = make_double2(-T2.y, T2.x);   // P2 = i Bh (r + 1)
  o[3] = Bh;
  o[4] = make_double2(-sg * (rB.x + B.x), -sg * (rB.y - B.y));   // Q'
#endif
}

// Per target (z, with the carried reciprocal rp and offset wp of the
// previous record's node) and record {node, P1, P2, Bh, Q'}:
//   w = z - node, r = 1/w, I2 = r - rp, S = r + rp, d = w + wp = 2 (z - zc)
//   phi += Im(Bh I2),  psi += I2 [Q' + (d.x P1 + d.y P2) S]
// 29 fp64-pipe instructions + 1 MUFU.RCP64H per record.  With DDM_REC_K the
// record carries P1' = 2 P1, P2' = 2 P2 and K = zc.x P1' + zc.y P2', so
//   d.x P1 + d.y P2 = z.x P1' + z.y P2' - K
// (4 DFMA instead of 2 DADD + 2 DMUL + 2 DFMA, and no offset carry): 27, and
// 26 with the one-step reciprocal below.

// DDM_P2P_RCP2=1 (default): the near-field reciprocal takes ONE Newton step
// on the MUFU seed instead of fast_rcp's cubic refinement.  Measured
// (scripts/micro/rcp_probe.cu, x over 1e-12..1e12): seed 9.9e-7, one step
// 9.9e-13, cubic 2.2e-16 max relative error.  The FMM bar is 1e-8 (the
// direct mode keeps the cubic form for its 1e-12 bar); one DFMA fewer per
// pair: P2P 0.579 -> 0.564 ms, concurrent step 0.976 -> 0.957 ms (config 5).
#ifndef DDM_P2P_RCP2
#define DDM_P2P_RCP2 1
#endif
__device__ __forceinline__ double p2p_rcp(double x) {
#if DDM_P2P_RCP2
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return fma(r, fma(-x, r, 1.0), r);
#else
  return fast_rcp(x);
#endif
}

struct NodeCarry {
#if DDM_REC_K
  double rx, ry;
#else
  double rx, ry, wx, wy;
#endif
};

__device__ __forceinline__ void node_init(NodeCarry& n, double zx, double zy, const double* rec) {
  const double wx = zx - rec[0], wy = zy - rec[1];
  const double inv = p2p_rcp(fma(wx, wx, wy * wy));
  n.rx = wx * inv;
  n.ry = -wy * inv;
#if !DDM_REC_K
  n.wx = wx;
  n.wy = wy;
#endif
}


__device__ __forceinline__ void record_update(P2PAcc& acc, NodeCarry& n, double zx, double zy,
                                              const double* sp) {
  const double wx = zx - sp[0], wy = zy - sp[1];
  const double inv = p2p_rcp(fma(wx, wx, wy * wy));
  const double rx = wx * inv, ry = -wy * inv;
  const double I2x = rx - n.rx, I2y = ry - n.ry;
  const double Sx = rx + n.rx, Sy = ry + n.ry;
#if DDM_REC_K
  const double BXx = fma(zx, sp[2], fma(zy, sp[4], -sp[10]));
  const double BXy = fma(zx, sp[3], fma(zy, sp[5], -sp[11]));
#else
  const double dx = wx + n.wx, dy = wy + n.wy;
  const double BXx = fma(dx, sp[2], dy * sp[4]);
  const double BXy = fma(dx, sp[3], dy * sp[5]);
#endif
  const double Vx = fma(BXx, Sx, fma(-BXy, Sy, sp[8]));
  const double Vy = fma(BXx, Sy, fma(BXy, Sx, sp[9]));
  acc.psi.x = fma(I2x, Vx, fma(-I2y, Vy, acc.psi.x));
  acc.psi.y = fma(I2x, Vy, fma(I2y, Vx, acc.psi.y));
  acc.phi = fma(sp[6], I2y, fma(sp[7], I2x, acc.phi));
  n.rx = rx;
  n.ry = ry;
#if !DDM_REC_K
  n.wx = wx;
  n.wy = wy;
#endif
}

// One warp per work item (leaf k, group of nt <= kTgtGroup targets, interval
// [item.z, item.w) of the leaf's concatenated source-slot ranges, read as the
// item's record ranges it_rng[it_roff[it] .. it_roff[it+1])).  Each lane
// owns kTPL targets (independent chains sharing every record load); the
// tp = ceil(nt/kTPL) lane-target slots are replicated over S = 32 / tp source
// slices, and slice s takes the s-th contiguous part of each range's records
// (a node carry needs consecutive records), starting from the node of the
// record before it.  Records are read through L1 (the tp lanes of a slice
// broadcast one record).  The S slice partials are summed in a fixed order
// (deterministic results, independent of the rank count).
#ifndef DDM_P2P_WARPS
#define DDM_P2P_WARPS 4
#endif
constexpr int kP2PWarps = DDM_P2P_WARPS;
#ifndef DDM_P2P_MINB
#define DDM_P2P_MINB 6
#endif
#ifndef DDM_TPL
#define DDM_TPL 2
#endif
constexpr int kTPL = DDM_TPL;   // targets per lane (independent chains sharing each record load)
#ifndef DDM_P2P_UNROLL
#define DDM_P2P_UNROLL 2
#endif
constexpr int kP2PUnroll = DDM_P2P_UNROLL;

__device__ __forceinline__ void load_rec(double (&sp)[kRecStride], const double* rec) {
  const double2* g = reinterpret_cast<const double2*>(rec);
#pragma unroll
  for (int f = 0; f < kRecStride / 2; ++f) {
    const double2 v = __ldg(g + f);
    sp[2 * f] = v.x;
    sp[2 * f + 1] = v.y;
  }
}

__global__ void __launch_bounds__(kP2PWarps * 32, DDM_P2P_MINB)
p2p_kernel(int nown, const int* __restrict__ order, const int4* __restrict__ items,
           const int* __restrict__ leaves,
           const int* __restrict__ c_start, const int* __restrict__ c_count,
           const int* __restrict__ it_roff, const int2* __restrict__ it_rng,
           const double* __restrict__ srec,
           const double* __restrict__ ex, const double* __restrict__ ey,
           const double* __restrict__ ec, const double* __restrict__ es, double gc,
           double2* __restrict__ part) {
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
      const int e0 = __ldg(it_roff + it), e1 = __ldg(it_roff + it + 1);
      int2 rr = e0 < e1 ? __ldg(it_rng + e0) : make_int2(0, 0);
      for (int ei = e0; ei < e1; ++ei) {
        const int rb = rr.x, L = rr.y - rr.x;
        if (ei + 1 < e1) rr = __ldg(it_rng + ei + 1);   // next range's bounds in flight
        const int q0 = rb + (int)(((int64_t)L * slice) / S);
        const int q1 = rb + (int)(((int64_t)L * (slice + 1)) / S);
        if (q0 >= q1) continue;
        NodeCarry nc[kTPL];
        {
          double sp[kRecStride];
          load_rec(sp, srec + (int64_t)(q0 - 1) * kRecStride);
#pragma unroll
          for (int q = 0; q < kTPL; ++q) node_init(nc[q], zx[q], zy[q], sp);
        }
#pragma unroll kP2PUnroll
        for (int j = q0; j < q1; ++j) {
          double sp[kRecStride];
          load_rec(sp, srec + (int64_t)j * kRecStride);
#pragma unroll
          for (int q = 0; q < kTPL; ++q) record_update(acc[q], nc[q], zx[q], zy[q], sp);
        }
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

// ---------------------------------------------------------------- leaf blocks
// Near field with the source records staged in shared memory:
// one CTA (4 warps) per owned leaf B.  B's source records are the U(B) ranges
// of the node-sharing stream, contiguous in srec, so each range (with the
// record before it, which carries the previous node) is ONE 1-D bulk copy
// (cp.async.bulk on the TMA engine) into shared memory, completing on an
// mbarrier: warp 0 reads the leaf's range table, prefix-sums the staged sizes
// with shuffles and its lanes issue one copy each.  (A leaf whose ranges
// exceed the buffer is processed in chunks, built by thread 0.)  Every staged
// record is then read by all targets of the leaf: 2 targets per lane, tp =
// ceil(nt/2) lanes per slice, S slices (S <= 128/tp and about >= 16 records per
// slice), slice s taking the s-th contiguous part of the chunk's records (a
// node carry is re-initialised where a range starts).  Slice partials are
// summed in a fixed order: deterministic, independent of the rank count.
#ifndef DDM_LEAF_THREADS
#define DDM_LEAF_THREADS 128
#endif
constexpr int kLeafThreads = DDM_LEAF_THREADS;
#ifndef DDM_LEAF_TPL
#define DDM_LEAF_TPL 2
#endif
constexpr int kLT = DDM_LEAF_TPL;           // targets per lane
constexpr int kLeafMaxTg = 32 * kLT;        // targets per pass (tp <= 32: >= 4 slices)
constexpr int kLeafMaxPieces = 32;  // ranges per chunk
constexpr int kLeafMinRec = 16;     // records per slice (at least, where possible)
#ifndef DDM_LEAF_RMAX
#define DDM_LEAF_RMAX (DDM_REC_K ? 352 : 384)   // staged records per chunk (33 / 30 KB: 6 CTAs per SM)
#endif
#ifndef DDM_LEAF_MINB
#define DDM_LEAF_MINB 6
#endif

#ifndef DDM_LEAF_UNROLL
#define DDM_LEAF_UNROLL 2
#endif
constexpr int kLeafUnroll = DDM_LEAF_UNROLL;
__device__ __forceinline__ void load_rec_s(double (&sp)[kRecStride], const double* rec) {
  const double2* g = reinterpret_cast<const double2*>(rec);
#pragma unroll
  for (int f = 0; f < kRecStride / 2; ++f) {
    const double2 v = g[f];
    sp[2 * f] = v.x;
    sp[2 * f + 1] = v.y;
  }
}

__global__ void __launch_bounds__(kLeafThreads, DDM_LEAF_MINB)
p2p_leaf_kernel(int leaf_lo, const int* __restrict__ order, const int4* __restrict__ leaf_info,
                const int2* __restrict__ lr_rng,
                const double* __restrict__ srec, const double* __restrict__ ex,
                const double* __restrict__ ey, const double* __restrict__ ec,
                const double* __restrict__ es, double gc, int rmax, double* __restrict__ y_near) {
  extern __shared__ __align__(128) double recs[];   // [rmax][kRecStride]
  __shared__ __align__(8) unsigned long long bar;
  // pieces of the current chunk: (first staged record = the carry, first real
  // record in srec, real records, real-record prefix)
  __shared__ int4 pcs[kLeafMaxPieces];
  __shared__ int s_np, s_R, s_last, s_cur_r, s_cur_off;
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned bar_a = smem_u32(&bar);
  // (cs, nt, first range, end range) of the leaf
  const int4 li = __ldg(leaf_info + leaf_lo + (order ? __ldg(order + blockIdx.x) : (int)blockIdx.x));
  const int cs = li.x, nt = li.y, rg0 = li.z, rg1 = li.w;
  if (tid == 0) mbar_init(bar_a, 1);
  __syncthreads();
  unsigned phase = 0;
  for (int tg0 = 0; tg0 < nt; tg0 += kLeafMaxTg) {
    const int tg = min(kLeafMaxTg, nt - tg0);
    const int tp = (tg + kLT - 1) / kLT, Smax = kLeafThreads / tp;
    double zx[kLT], zy[kLT];
    P2PAcc acc[kLT];
    const int tl0 = tid % tp;
#pragma unroll
    for (int q = 0; q < kLT; ++q) {
      const int ti = cs + tg0 + min(kLT * tl0 + q, tg - 1);
      zx[q] = __ldg(ex + ti);
      zy[q] = __ldg(ey + ti);
    }
    int S = 1;
    bool first_chunk = true;
    if (tid == 0) {
      s_cur_r = rg0;
      s_cur_off = 0;
    }
    while (true) {
      // ---- stage the next chunk
      bool fast = false;
      if (first_chunk && tid < 32 && rg1 - rg0 <= 32) {
        // all ranges at once: lane r takes range rg0 + r
        const int nr = rg1 - rg0;
        int2 rg = make_int2(0, 0);
        if (lane < nr) rg = __ldg(lr_rng + rg0 + lane);
        const int L = rg.y - rg.x;
        int incl = lane < nr ? L + 1 : 0;   // staged records of range `lane` (with its carry)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int used = __shfl_sync(0xffffffffu, incl, 31);
        fast = used <= rmax;
        if (fast) {
          const int st0 = incl - (lane < nr ? L + 1 : 0);
          if (lane < nr) pcs[lane] = make_int4(st0, rg.x, L, st0 - lane);
          if (lane == 0) {
            s_np = nr;
            s_R = used - nr;
            s_last = 1;
            if (nr > 0) mbar_expect_tx(bar_a, (unsigned)used * kRecStride * 8u);
          }
          __syncwarp();
          if (lane < nr)
            bulk_g2s(smem_u32(recs + (size_t)st0 * kRecStride), srec + (int64_t)(rg.x - 1) * kRecStride,
                     (unsigned)(L + 1) * kRecStride * 8u, bar_a);
        }
      }
      fast = __syncthreads_or(fast);
      if (!fast && tid == 0) {   // general case: greedy chunk from the cursor
        int cur_r = s_cur_r, cur_off = s_cur_off;
        int np = 0, used = 0, R = 0;
        while (cur_r < rg1 && np < kLeafMaxPieces) {
          const int2 rg = __ldg(lr_rng + cur_r);
          const int L = rg.y - rg.x - cur_off;
          const int room = rmax - used - 1;
          if (room <= 0) break;
          const int take = min(L, room);
          pcs[np++] = make_int4(used, rg.x + cur_off, take, R);
          used += take + 1;
          R += take;
          if (take < L) {
            cur_off += take;
            break;
          }
          ++cur_r;
          cur_off = 0;
        }
        s_cur_r = cur_r;
        s_cur_off = cur_off;
        s_np = np;
        s_R = R;
        s_last = cur_r >= rg1;
        if (np > 0) {
          mbar_expect_tx(bar_a, (unsigned)used * kRecStride * 8u);
          for (int q = 0; q < np; ++q) {
            const int4 pc = pcs[q];
            bulk_g2s(smem_u32(recs + (size_t)pc.x * kRecStride), srec + (int64_t)(pc.y - 1) * kRecStride,
                     (unsigned)(pc.z + 1) * kRecStride * 8u, bar_a);
          }
        }
      }
      if (!fast) __syncthreads();
      const int np = s_np, R = s_R;
      const bool last = s_last;
      if (first_chunk) {   // slices: >= kLeafMinRec records each where the leaf allows
        S = max(1, min(Smax, R / kLeafMinRec));
        first_chunk = false;
      }
      if (np == 0) break;
      mbar_wait(bar_a, phase);
      phase ^= 1u;
      // each range's staged predecessor (its carry record) keeps its node and
      // gets zero coefficients: it then acts as a break record, and every
      // slice walks ONE contiguous run of staged records with a single node
      // carry initialised from the record before it (no branch per record)
      if (tid < np) {
        double* cr = recs + (size_t)pcs[tid].x * kRecStride;
#pragma unroll
        for (int f = 2; f < kRecStride; ++f) cr[f] = 0.0;
      }
      __syncthreads();
      // ---- evaluate: slice `slice` of the chunk's staged records 1 .. used-1
      const int used = R + np;   // staged records (the first, index 0, is a carry)
      const int slice = tid / tp, tl = tid - slice * tp;
      if (slice < S) {
        const int a = 1 + (int)(((int64_t)(used - 1) * slice) / S);
        const int b = 1 + (int)(((int64_t)(used - 1) * (slice + 1)) / S);
        if (a < b) {
          NodeCarry ncr[kLT];
          {
            double sp[kRecStride];
            load_rec_s(sp, recs + (size_t)(a - 1) * kRecStride);
#pragma unroll
            for (int q = 0; q < kLT; ++q) node_init(ncr[q], zx[q], zy[q], sp);
          }
#pragma unroll kLeafUnroll
          for (int j = a; j < b; ++j) {
            double sp[kRecStride];
            load_rec_s(sp, recs + (size_t)j * kRecStride);
#pragma unroll
            for (int q = 0; q < kLT; ++q) record_update(acc[q], ncr[q], zx[q], zy[q], sp);
          }
        }
      }
      __syncthreads();   // the buffer is free for the next chunk
      if (last) break;
    }
    // ---- slice partials -> per target, summed in slice order
    const int slice = tid / tp, tl = tid - slice * tp;
    double* red = recs;   // [S][kLT tp][3] (<= kLT * 128 entries)
    if (slice < S) {
#pragma unroll
      for (int q = 0; q < kLT; ++q) {
        double* o = red + ((size_t)slice * kLT * tp + kLT * tl + q) * 3;
        o[0] = acc[q].phi;
        o[1] = acc[q].psi.x;
        o[2] = acc[q].psi.y;
      }
    }
    __syncthreads();
    if (tid < tg) {
      P2PAcc tot;
      for (int s2 = 0; s2 < S; ++s2) {
        const double* o = red + ((size_t)s2 * kLT * tp + tid) * 3;
        tot.phi += o[0];
        tot.psi.x += o[1];
        tot.psi.y += o[2];
      }
      const int ti = cs + tg0 + tid;
      reinterpret_cast<double2*>(y_near)[ti] = acc_to_traction(tot, gc, ec[ti], es[ti]);
    }
    __syncthreads();
  }
}

// per leaf: (first sorted element, count, first U range, end U range)
__global__ void leaf_info_fill(int nleaves, const int* __restrict__ leaves,
                               const int* __restrict__ c_start, const int* __restrict__ c_count,
                               const int* __restrict__ u_off, int4* __restrict__ info) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int c = leaves[k];
  info[k] = make_int4(c_start[c], c_count[c], u_off[k], u_off[k + 1]);
}

// the record range of every U range (once per tree): lr_rng[r] = [rbeg[u_lo[r]], rbeg[u_hi[r]])
__global__ void leaf_rng_fill(int64_t nu, const int* __restrict__ u_lo, const int* __restrict__ u_hi,
                              const int* __restrict__ rbeg, int2* __restrict__ lr_rng) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < nu) lr_rng[r] = make_int2(rbeg[u_lo[r]], rbeg[u_hi[r]]);
}

// elastic FMM assembly: y = near (p2p_leaf_kernel) + far (L2P), sorted and/or user order
__global__ void finalize_near_kernel(int64_t e_lo, int64_t e_hi, const double2* __restrict__ y_near,
                                     const double2* __restrict__ y_far,
                                     const int* __restrict__ perm, double2* __restrict__ y_user,
                                     double2* __restrict__ y_sorted) {
  // a PDL-launched successor (the GMRES step's first CGS kernel) may start early;
  // it waits for this grid before reading anything
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t i = e_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= e_hi) return;
  const double2 a = y_near[i], b = y_far[i];
  const double2 t = make_double2(a.x + b.x, a.y + b.y);
  if (y_sorted) y_sorted[i] = t;
  if (y_user) y_user[perm[i]] = t;
}

__global__ void add_const_kernel(int64_t n, int v, int* __restrict__ a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] += v;
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
#ifndef DDM_P2P_IPW
#define DDM_P2P_IPW 1
#endif
  const unsigned nb = nblk(item_hi - item_lo, kP2PWarps * DDM_P2P_IPW);   // items per warp
  p2p_kernel<<<nb, kP2PWarps * 32, 0, s>>>(item_hi - item_lo, t->p2p_order, t->items,
                                           t->leaves, t->c_start, t->c_count,
                                           t->it_roff, t->it_rng, t->srec, t->ex, t->ey, t->ec,
                                           t->es, gc, t->part);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// Elastic near field, leaf blocks: owned leaves in Morton
// order (consecutive CTAs share source records in L2); writes y_near.
bool use_leaf_p2p() {
  static const bool on = [] {
    const char* e = getenv("DDM_P2P_LEAF");
    return !(e && e[0] == '0');
  }();
  return on;
}

int launch_p2p_leaf(ddm_ctx_s* ctx, ddm_tree_s* t, double gc, cudaStream_t s, bool use_x) {
  const int nlv = t->own_leaf_hi - t->own_leaf_lo;
  if (nlv <= 0) return DDM_OK;
  const int rmax = DDM_LEAF_RMAX;
  const size_t shm = (size_t)rmax * kRecStride * sizeof(double);
  static bool attr = false;
  if (!attr) {
    DDM_CUDA(ctx, cudaFuncSetAttribute(p2p_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)shm));
    attr = true;
  }
  const bool ux = use_x && t->nx > 0;
  p2p_leaf_kernel<<<nlv, kLeafThreads, shm, s>>>(t->own_leaf_lo, t->p2p_leaf_order,
                                                ux ? t->leaf_info_x : t->leaf_info,
                                                ux ? t->lr_rng_x : t->lr_rng, t->srec,
                                                t->ex, t->ey, t->ec, t->es, gc, rmax, t->y_near);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_finalize_near(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, double* y_user,
                         double* y_sorted, cudaStream_t s) {
  if (hi <= lo) return DDM_OK;
  finalize_near_kernel<<<nblk(hi - lo, 256), 256, 0, s>>>(
      lo, hi, reinterpret_cast<const double2*>(t->y_near),
      reinterpret_cast<const double2*>(t->y_far), t->perm, reinterpret_cast<double2*>(y_user),
      reinterpret_cast<double2*>(y_sorted));
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// Near-field source stream of the tree (once per tree, outside any capture)
int build_source_stream(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) {
  if (t->srec || t->n == 0) return DDM_OK;
  const int64_t n = t->n;
  int rc;
  int* cntv = nullptr;
  if ((rc = talloc(ctx, &t->st_elem, (size_t)n, s)) || (rc = talloc(ctx, &t->st_code, (size_t)n, s)) ||
      (rc = talloc(ctx, &t->rbeg, (size_t)n + 1, s)) || (rc = talloc(ctx, &cntv, (size_t)n + 1, s)))
    return rc;
  chain_order_kernel<<<nblk(t->nleaves, 64), 64, 0, s>>>(t->nleaves, t->leaves, t->c_start,
                                                         t->c_count, t->ex, t->ey, t->ea, t->ec,
                                                         t->es, t->st_elem, t->st_code);
  DDM_CUDA(ctx, cudaGetLastError());
  chain_count_kernel<<<nblk(n, 256), 256, 0, s>>>(n, t->st_code, cntv);
  DDM_CUDA(ctx, cudaMemsetAsync(cntv + n, 0, sizeof(int), s));
  int total = 0;
  if ((rc = exclusive_scan_i32(ctx, cntv, t->rbeg, (int)n + 1, &total, s))) return rc;
  cudaFreeAsync(cntv, s);
  // records: pad (0), then the slots' records; rbeg was counted from 0
  add_const_kernel<<<nblk(n + 1, 256), 256, 0, s>>>(n + 1, 1, t->rbeg);
  DDM_CUDA(ctx, cudaGetLastError());
  t->nrec = (int64_t)total + 1;
  if ((rc = talloc(ctx, &t->srec, (size_t)t->nrec * kRecStride, s))) return rc;
  const double2 pad = make_double2(t->x_min - 16.0 * t->W, t->y_min - 16.0 * t->W);
  break_records_kernel<<<nblk(n, 256), 256, 0, s>>>(n, t->st_elem, t->st_code, t->rbeg, t->ex,
                                                    t->ey, t->ea, t->ec, t->es, pad, t->srec);
  DDM_CUDA(ctx, cudaGetLastError());
  // record ranges of every P2P item
  const int ni = t->nitems;
  int* icnt = nullptr;
  if ((rc = talloc(ctx, &t->it_roff, (size_t)ni + 1, s)) || (rc = talloc(ctx, &icnt, (size_t)ni + 1, s)))
    return rc;
  item_rng_count<<<nblk(ni + 1, 128), 128, 0, s>>>(ni, t->items, t->u_off, t->u_lo, t->u_hi, icnt);
  DDM_CUDA(ctx, cudaGetLastError());
  int nr = 0;
  if ((rc = exclusive_scan_i32(ctx, icnt, t->it_roff, ni + 1, &nr, s))) return rc;
  cudaFreeAsync(icnt, s);
  if ((rc = talloc(ctx, &t->it_rng, (size_t)std::max(nr, 1), s))) return rc;
  item_rng_fill<<<nblk(ni, 128), 128, 0, s>>>(ni, t->items, t->u_off, t->u_lo, t->u_hi, t->rbeg,
                                              t->it_roff, t->it_rng);
  DDM_CUDA(ctx, cudaGetLastError());
  // record ranges of the U ranges (leaf-block near field)
  if ((rc = talloc(ctx, &t->lr_rng, (size_t)std::max<int64_t>(t->nu, 1), s))) return rc;
  if (t->nu > 0) {
    leaf_rng_fill<<<nblk(t->nu, 256), 256, 0, s>>>(t->nu, t->u_lo, t->u_hi, t->rbeg, t->lr_rng);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  if ((rc = talloc(ctx, &t->leaf_info, (size_t)t->nleaves, s))) return rc;
  leaf_info_fill<<<nblk(t->nleaves, 256), 256, 0, s>>>(t->nleaves, t->leaves, t->c_start, t->c_count,
                                                       t->u_off, t->leaf_info);
  DDM_CUDA(ctx, cudaGetLastError());
  // the same tables for U minus X (elastic series FMM with X lists)
  if (t->nx > 0) {
    if ((rc = talloc(ctx, &t->lr_rng_x, (size_t)std::max<int64_t>(t->nux, 1), s))) return rc;
    if (t->nux > 0) {
      leaf_rng_fill<<<nblk(t->nux, 256), 256, 0, s>>>(t->nux, t->ux_lo, t->ux_hi, t->rbeg,
                                                      t->lr_rng_x);
      DDM_CUDA(ctx, cudaGetLastError());
    }
    if ((rc = talloc(ctx, &t->leaf_info_x, (size_t)t->nleaves, s))) return rc;
    leaf_info_fill<<<nblk(t->nleaves, 256), 256, 0, s>>>(t->nleaves, t->leaves, t->c_start,
                                                         t->c_count, t->ux_off, t->leaf_info_x);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  return DDM_OK;
}

int launch_prep_stream(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D,
                       int ncomp, cudaStream_t s, bool halo) {
  // slots [halo_lo, halo_hi): every record the owned leaves' near field reads
  // (all slots on one rank)
  const bool h = halo && t->halo_rng;
  const int64_t q0 = 0, q1 = h ? t->halo_slots : (halo ? 0 : t->n);
  if (q1 <= q0) return DDM_OK;
  prep_stream<<<nblk(q1 - q0, 256), 256, 0, s>>>(q0, q1, h ? t->halo_rng : nullptr,
                                               h ? t->halo_pre : nullptr, t->nhalo, ncomp, perm_in,
                                               t->st_elem, t->st_code,
                                               t->rbeg, D, t->ex, t->ey, t->ea, t->ec, t->es,
                                               t->srec, perm_in ? t->d_sorted : nullptr);
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
