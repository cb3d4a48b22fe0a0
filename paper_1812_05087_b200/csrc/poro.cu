// Fully coupled poroelastic continuous-source kernel on the GPU (DESIGN.md
// §4.5; PAPER.md Eq.(int_sigs)-(int_pp) P:319-375, Eq.(final_sigs)-(final_pp)
// P:389-449).  Plane strain Biot theory, tension-positive stress, CS-convention
// DDs, physical pore pressure; the ABI sign map J = diag(1, 1, -1) is applied
// at the boundary of this file (source q and output p negated).
//
// Element influence = drained Kolosov–Muskhelishvili (closed form, nu)
//   + sigma^p = 2 eta (Phi_,ij - p delta_ij) and p, integrated along the
//     element with the fixed rule: panels graded away from the nearest point
//     (each <= max(r, sqrt(c tau)) / 4), 8-point Gauss–Legendre per panel,
//     E1 log singularity removed analytically when the target is on the
//     element; analytic far form when u_min = dist^2 / (4 c tau) > 40.
// Point kernels (per unit length, omega = w/|w|, u = |w|^2/(4 c tau)):
//   p       = Re(K ob^2) f2(u)/(4 c tau) + mu e^-u/(4 pi c tau) + q E1(u)/(4 pi kappa)
//   d2Phi   = K ob^4 g2(u)/(4 c tau) - e^-u Re(K ob^2) ob^2/(16 c tau)
//             - mu f2(u) ob^2/(16 pi c tau) - q h2(u) ob^2/(16 pi kappa)
//   K = -4 k_p i G C B e, B = (Ds + i Dn) e, mu = -(eta/S) Dn
//   T^p = sigma_n + i sigma_s = -eta p + e^{2 i bt} (-4 eta d2Phi)
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kcommon.cuh"

namespace ddm {
namespace {

__constant__ double c_gl_x[8];
__constant__ double c_gl_w[8];

constexpr double kUFar = 40.0;
constexpr double kPanelFraction = 0.25;
constexpr double kEulerGamma = 0.57721566490153286061;

struct PoroConst {
  double G, C, eta, kp, S, kappa, c, ct;   // ct = c tau
  double gc;                              // G C
};

// f2 = (1 - (1+u)e^-u)/u, g2 = (-1/4 - e^-u/2 + 3(1-e^-u)/(4u))/u, h2 = (1-e^-u)/u
// power-series coefficients (powers of u, ascending), filled by poro_init_tables:
//   f2 = sum_{k>=2} (-1)^k (k-1) u^(k-1)/k!,  g2 = sum_{k>=1} (-1)^k (1-2k) u^(k-1)/(4 (k+1)!),
//   h2 = sum_{k>=0} (-u)^k/(k+1)!
constexpr int kNSeries = 25;
__constant__ double c_f2[kNSeries];
__constant__ double c_g2[kNSeries];
__constant__ double c_h2[8];

__device__ __forceinline__ void fgh(double u, double& f2, double& g2, double& h2, double& eu) {
  eu = exp(-u);
  if (u < 1.0) {
    double sf = 0.0, sg = 0.0;
#pragma unroll
    for (int k = kNSeries - 1; k >= 0; --k) {
      sf = fma(sf, u, c_f2[k]);
      sg = fma(sg, u, c_g2[k]);
    }
    f2 = sf;
    g2 = sg;
  } else {
    f2 = (1.0 - (1.0 + u) * eu) / u;
    g2 = (-0.25 - 0.5 * eu + 0.75 * (-expm1(-u)) / u) / u;
  }
  if (u < 1e-3) {
    double s = 0.0;
#pragma unroll
    for (int k = 7; k >= 0; --k) s = fma(s, u, c_h2[k]);
    h2 = s;
  } else {
    h2 = -expm1(-u) / u;
  }
}

// Exponential integral E1 (Theis fluid-source kernel), table driven (no
// iterative continued fraction on the device):
//   u <= 2:        Ein(u) = E1(u) + gamma + ln u = sum_{k=1}^{25} (-1)^{k+1} u^k/(k k!)  (Horner)
//   2 < u <= 1024: h(u) = u e^u E1(u) by a 26-term Chebyshev series per octave
//                  [2^j, 2^{j+1}] (coefficients from a long-double continued
//                  fraction at start-up, poro_init_tables)
//   u > 1024:      h = 1 - 1/u + 2/u^2 - 6/u^3 + 24/u^4 - 120/u^5
// Max relative error vs a reference E1: 3.4e-15.
constexpr int kEinTerms = 25;
constexpr int kE1Oct = 9;        // octaves [2,4) .. [512,1024)
constexpr int kE1Cheb = 26;
__device__ double g_ein[kEinTerms];
__device__ double g_e1cheb[kE1Oct * kE1Cheb];

__device__ __forceinline__ double ein_poly(double u) {   // u <= 2
  double s = 0.0;
#pragma unroll
  for (int k = kEinTerms - 1; k >= 0; --k) s = fma(s, u, __ldg(g_ein + k));
  return s * u;
}

__device__ __forceinline__ double e1_h(double u) {   // u e^u E1(u), u > 2
  if (u > 1024.0) {
    const double iu = 1.0 / u;
    return 1.0 - iu * (1.0 - 2.0 * iu * (1.0 - 3.0 * iu * (1.0 - 4.0 * iu * (1.0 - 5.0 * iu))));
  }
  int j = ilogb(u) - 1;               // u in [2^(j+1), 2^(j+2))
  j = min(max(j, 0), kE1Oct - 1);
  const double a = ldexp(2.0, j), b = 2.0 * a;
  const double x = (2.0 * u - a - b) / (b - a);
  const double* c = g_e1cheb + j * kE1Cheb;
  double b1 = 0.0, b2 = 0.0;
#pragma unroll
  for (int k = kE1Cheb - 1; k >= 1; --k) {
    const double t = fma(2.0 * x, b1, __ldg(c + k) - b2);
    b2 = b1;
    b1 = t;
  }
  return fma(x, b1, __ldg(c) - b2);
}

// E1(u), u > 0
__device__ __forceinline__ double expint_e1(double u) {
  if (u <= 2.0) return ein_poly(u) - kEulerGamma - log(u);
  return e1_h(u) * exp(-u) / u;
}
// Ein(u) = E1(u) + gamma + ln u (the smooth part, for targets on the element)
__device__ __forceinline__ double expint_ein(double u) {
  if (u <= 2.0) return ein_poly(u);
  return e1_h(u) * exp(-u) / u + kEulerGamma + log(u);
}

// point kernel: adds w_q * (p, d2Phi) of the unit-length point source at offset w
__device__ __forceinline__ void point_add(double wx, double wy, double wq, const PoroConst& k,
                                          double2 K, double mu, double q, bool q_split,
                                          double& p_acc, double2& d2_acc) {
  const double r2 = fma(wx, wx, wy * wy);
  const double u = r2 / (4.0 * k.ct);
  const double ir = rsqrt(r2);
  // ob = conj(omega)
  const double obx = wx * ir, oby = -wy * ir;
  const double2 ob2 = make_double2(obx * obx - oby * oby, 2.0 * obx * oby);
  const double2 ob4 = cmul(ob2, ob2);
  double f2, g2, h2, eu;
  fgh(u, f2, g2, h2, eu);
  const double2 Kob2 = cmul(K, ob2);
  const double ReK = Kob2.x;
  double p = ReK * f2 / (4.0 * k.ct) + mu * eu / (4.0 * M_PI * k.ct);
  const double2 Kob4 = cmul(K, ob4);
  double2 d2 = make_double2(Kob4.x * g2 / (4.0 * k.ct), Kob4.y * g2 / (4.0 * k.ct));
  const double cb = eu * ReK / (16.0 * k.ct) + mu * f2 / (16.0 * M_PI * k.ct);
  d2.x -= cb * ob2.x;
  d2.y -= cb * ob2.y;
  if (q != 0.0) {
    const double e1 = q_split ? expint_ein(u) : expint_e1(u);
    p += q * e1 / (4.0 * M_PI * k.kappa);
    const double cq = q * h2 / (16.0 * M_PI * k.kappa);
    d2.x -= cq * ob2.x;
    d2.y -= cq * ob2.y;
  }
  p_acc = fma(wq, p, p_acc);
  d2_acc.x = fma(wq, d2.x, d2_acc.x);
  d2_acc.y = fma(wq, d2.y, d2_acc.y);
}

// point_add for the three unit source columns at once (near-field block
// builds): column 0 = unit D_s (K0 = -4 k_p i G C e^2), column 1 = unit D_n
// (K1 = i K0, mu = -eta/S), column 2 = unit q_ABI (q_formula = -1).  The
// kernel functions of the node (f2, g2, h2, e^-u, E1) are evaluated once.
__device__ __forceinline__ void point_add3(double wx, double wy, double wq, const PoroConst& k,
                                           double2 K0, double mu1, bool q_split, double* p_acc,
                                           double2* d2_acc) {
  const double r2 = fma(wx, wx, wy * wy);
  const double u = r2 / (4.0 * k.ct);
  const double ir = rsqrt(r2);
  const double obx = wx * ir, oby = -wy * ir;
  const double2 ob2 = make_double2(obx * obx - oby * oby, 2.0 * obx * oby);
  const double2 ob4 = cmul(ob2, ob2);
  double f2, g2, h2, eu;
  fgh(u, f2, g2, h2, eu);
  const double c4 = 1.0 / (4.0 * k.ct), c16 = 1.0 / (16.0 * k.ct);
  const double2 Kob2 = cmul(K0, ob2), Kob4 = cmul(K0, ob4);
  // column 0
  {
    const double ReK = Kob2.x;
    const double p = ReK * f2 * c4;
    const double cb = eu * ReK * c16;
    p_acc[0] = fma(wq, p, p_acc[0]);
    d2_acc[0].x = fma(wq, Kob4.x * g2 * c4 - cb * ob2.x, d2_acc[0].x);
    d2_acc[0].y = fma(wq, Kob4.y * g2 * c4 - cb * ob2.y, d2_acc[0].y);
  }
  // column 1: K1 ob^2 = i K0 ob^2, K1 ob^4 = i K0 ob^4
  {
    const double ReK = -Kob2.y;
    const double p = ReK * f2 * c4 + mu1 * eu / (4.0 * M_PI * k.ct);
    const double cb = eu * ReK * c16 + mu1 * f2 / (16.0 * M_PI * k.ct);
    p_acc[1] = fma(wq, p, p_acc[1]);
    d2_acc[1].x = fma(wq, -Kob4.y * g2 * c4 - cb * ob2.x, d2_acc[1].x);
    d2_acc[1].y = fma(wq, Kob4.x * g2 * c4 - cb * ob2.y, d2_acc[1].y);
  }
  // column 2: q = -1
  {
    const double e1 = q_split ? expint_ein(u) : expint_e1(u);
    const double cq = h2 / (16.0 * M_PI * k.kappa);
    p_acc[2] = fma(wq, -e1 / (4.0 * M_PI * k.kappa), p_acc[2]);
    d2_acc[2].x = fma(wq, cq * ob2.x, d2_acc[2].x);
    d2_acc[2].y = fma(wq, cq * ob2.y, d2_acc[2].y);
  }
}

// integral of (-gamma - ln(s^2/(4 c tau))) ds over [s0, s1], 0 <= s0 < s1
__device__ __forceinline__ double e1_log_part(double s0, double s1, double ct) {
  auto prim = [&](double s) {
    if (s == 0.0) return 0.0;
    return -kEulerGamma * s - (2.0 * (s * log(s) - s) - s * log(4.0 * ct));
  };
  return prim(s1) - prim(s0);
}

}  // namespace

// Poroelastic influence of one source element on one target (tension-positive
// traction T = sigma_n + i sigma_s and physical p, CS-convention DDs):
// the sigma^p + p part only (the drained part is added by the caller).
__device__ void poro_element(double2 zt, double2 zc, double2 e, double a, double Ds, double Dn,
                             double q, const PoroConst& k, double2 e2t, double2& T, double& p) {
  const double lt = sqrt(k.ct);
  const double rx = zt.x - zc.x, ry = zt.y - zc.y;
  const double sstar = rx * e.x + ry * e.y;          // Re((zt - zc) conj(e))
  const double dperp = fabs(-rx * e.y + ry * e.x);   // |Im(...)|
  const double dist = (fabs(sstar) <= a) ? dperp : hypot(dperp, fabs(sstar) - a);
  const double2 B = make_double2(Ds * e.x - Dn * e.y, Ds * e.y + Dn * e.x);
  const double mu = -(k.eta / k.S) * Dn;
  if (dist * dist / (4.0 * k.ct) > kUFar) {
    // analytic far form: Phi^p = 2 eta k_p Phi^D, Psi^p = 2 eta k_p 2 i G C B Ibar3
    //   + (eta mu/pi + eta q c tau/(pi kappa)) conj(e) I2 + 48 eta k_p c tau i G C B I4
    const double2 z1 = make_double2(zc.x - a * e.x, zc.y - a * e.y);
    const double2 z2 = make_double2(zc.x + a * e.x, zc.y + a * e.y);
    const double2 w1 = make_double2(zt.x - z1.x, zt.y - z1.y);
    const double2 w2 = make_double2(zt.x - z2.x, zt.y - z2.y);
    auto inv = [](double2 w) {
      const double n = fma(w.x, w.x, w.y * w.y);
      return make_double2(w.x / n, -w.y / n);
    };
    const double2 r1 = inv(w1), r2 = inv(w2);
    const double2 I2 = csub(r2, r1);
    const double2 r12 = cmul(r1, r1), r22 = cmul(r2, r2);
    const double2 I3 = cscale(csub(r22, r12), 0.5);
    const double2 I4 = cscale(csub(cmul(r22, r2), cmul(r12, r1)), 1.0 / 3.0);
    const double2 rr = make_double2(e.x * e.x - e.y * e.y, -2.0 * e.x * e.y);   // conj(e)^2
    const double2 dz = make_double2(zt.x - zc.x, zt.y - zc.y);
    double2 X = make_double2(zc.x, -zc.y);
    cmac(X, rr, dz);
    const double2 I3b = csub(cmul(X, I3), cmul(rr, I2));
    const double2 iGC = make_double2(0.0, k.gc);
    const double2 iGCB = cmul(iGC, B);
    const double ekp = 2.0 * k.eta * k.kp;
    const double2 PhiD = cmul(iGCB, I2);
    const double2 Phi = cscale(PhiD, ekp);
    const double2 dPhi = cscale(cmul(iGCB, I3), -2.0 * ekp);
    const double wm = k.eta * mu / M_PI + k.eta * q * k.ct / (M_PI * k.kappa);
    double2 Psi = cscale(cmul(iGCB, I3b), 2.0 * ekp);
    cmac(Psi, cscale(make_double2(e.x, -e.y), wm), I2);
    cmac(Psi, cscale(iGCB, 48.0 * k.eta * k.kp * k.ct), I4);
    double2 Wv = Psi;
    cmac(Wv, make_double2(zt.x, -zt.y), dPhi);
    const double2 t2 = cmul(e2t, Wv);
    T = make_double2(2.0 * Phi.x + t2.x, t2.y);
    p = -k.kp * 4.0 * PhiD.x;
    return;
  }
  // near rule
  const double2 K = cscale(cmul(make_double2(0.0, k.gc), cmul(B, e)), -4.0 * k.kp);
  const bool on_line = (dperp == 0.0) && (fabs(sstar) < a);
  const double s0c = fmin(fmax(sstar, -a), a);
  double pacc = 0.0;
  double2 d2acc = make_double2(0.0, 0.0);
  for (int side = 0; side < 2; ++side) {
    const double other = side ? a : -a;
    const double sign = side ? 1.0 : -1.0;
    if ((other - s0c) * sign <= 0.0) continue;
    double s = s0c;
    int guard = 0;
    while ((other - s) * sign > 0.0 && guard++ < 4096) {
      const double r = hypot(dperp, s - sstar);
      double snext = s + sign * kPanelFraction * fmax(r, lt);
      if ((other - snext) * sign <= 0.0) snext = other;
      const double mid = 0.5 * (s + snext), half = 0.5 * fabs(snext - s);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const double sq = mid + half * c_gl_x[g];
        const double wx = zt.x - (zc.x + sq * e.x), wy = zt.y - (zc.y + sq * e.y);
        point_add(wx, wy, half * c_gl_w[g], k, K, mu, q, on_line, pacc, d2acc);
      }
      s = snext;
    }
    if (on_line && q != 0.0) {
      const double len = fabs(other - sstar);
      pacc += q * e1_log_part(0.0, len, k.ct) / (4.0 * M_PI * k.kappa);
    }
  }
  p = pacc;
  const double2 t2 = cmul(e2t, make_double2(-4.0 * k.eta * d2acc.x, -4.0 * k.eta * d2acc.y));
  T = make_double2(-k.eta * pacc + t2.x, t2.y);
}

// Is the pair (target zt, source element) in the near-rule regime of
// poro_element at this c tau?  (dist^2 / (4 c tau) <= 40)
__device__ __forceinline__ bool poro_is_near(double2 zt, double2 zc, double2 e, double a,
                                             double ct) {
  const double rx = zt.x - zc.x, ry = zt.y - zc.y;
  const double sstar = rx * e.x + ry * e.y;
  const double dperp = fabs(-rx * e.y + ry * e.x);
  const double dist = (fabs(sstar) <= a) ? dperp : hypot(dperp, fabs(sstar) - a);
  return !(dist * dist / (4.0 * ct) > kUFar);
}

// Warp-cooperative near rule of poro_element (same panels, nodes and weights:
// panels graded away from the nearest point, each <= max(r, sqrt(c tau))/4,
// 8-point Gauss–Legendre; analytic E1 log part on the element).  Lanes 0 and
// 1 generate the panel breakpoints of the two sides (sequential recurrence)
// into shared memory, then all 32 lanes evaluate the quadrature points; the
// sums are reduced across the warp.  All lanes must call it with the same
// arguments; every lane returns (T, p).
constexpr int kCoopPanels = 64;   // panels per side per round (shared memory)
__device__ void poro_near_coop(double2 zt, double2 zc, double2 e, double a, double Ds, double Dn,
                               double q, const PoroConst& k, double2 e2t, double* sh, int lane,
                               double2& T, double& p) {
  const double lt = sqrt(k.ct);
  const double rx = zt.x - zc.x, ry = zt.y - zc.y;
  const double sstar = rx * e.x + ry * e.y;
  const double dperp = fabs(-rx * e.y + ry * e.x);
  const double2 B = make_double2(Ds * e.x - Dn * e.y, Ds * e.y + Dn * e.x);
  const double mu = -(k.eta / k.S) * Dn;
  const double2 K = cscale(cmul(make_double2(0.0, k.gc), cmul(B, e)), -4.0 * k.kp);
  const bool on_line = (dperp == 0.0) && (fabs(sstar) < a);
  const double s0c = fmin(fmax(sstar, -a), a);
  // sh layout: [2 sides][kCoopPanels + 1] breakpoints, [2] counts (as doubles), [2] done flags
  double* bp = sh;
  double* cnt = sh + 2 * (kCoopPanels + 1);
  double pacc = 0.0;
  double2 d2acc = make_double2(0.0, 0.0);
  double cur = s0c;          // lane 0/1: current position of its side
  bool done = false;         // lane 0/1: side finished
  int guard = 0;
  if (lane < 2) {
    const double other = lane ? a : -a;
    const double sign = lane ? 1.0 : -1.0;
    done = !((other - s0c) * sign > 0.0);
  }
  for (;;) {
    if (lane < 2) {
      const double other = lane ? a : -a;
      const double sign = lane ? 1.0 : -1.0;
      double* b = bp + lane * (kCoopPanels + 1);
      int np = 0;
      b[0] = cur;
      while (!done && np < kCoopPanels) {
        if (!((other - cur) * sign > 0.0) || guard++ >= 4096) {
          done = true;
          break;
        }
        const double r = hypot(dperp, cur - sstar);
        double snext = cur + sign * kPanelFraction * fmax(r, lt);
        if ((other - snext) * sign <= 0.0) snext = other;
        b[++np] = snext;
        cur = snext;
        if (!((other - cur) * sign > 0.0)) done = true;
      }
      cnt[lane] = (double)np;
    }
    __syncwarp();
    const int n0 = (int)cnt[0], n1 = (int)cnt[1];
    const int npts = 8 * (n0 + n1);
    for (int t = lane; t < npts; t += 32) {
      const int pan = t >> 3, g = t & 7;
      const int side = pan < n0 ? 0 : 1;
      const int pi = side ? pan - n0 : pan;
      const double* b = bp + side * (kCoopPanels + 1);
      const double s = b[pi], snext = b[pi + 1];
      const double mid = 0.5 * (s + snext), half = 0.5 * fabs(snext - s);
      const double sq = mid + half * c_gl_x[g];
      const double wx = zt.x - (zc.x + sq * e.x), wy = zt.y - (zc.y + sq * e.y);
      point_add(wx, wy, half * c_gl_w[g], k, K, mu, q, on_line, pacc, d2acc);
    }
    const unsigned more = __ballot_sync(0xffffffffu, lane < 2 && !done);
    __syncwarp();
    if (!more) break;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    pacc += __shfl_xor_sync(0xffffffffu, pacc, o);
    d2acc.x += __shfl_xor_sync(0xffffffffu, d2acc.x, o);
    d2acc.y += __shfl_xor_sync(0xffffffffu, d2acc.y, o);
  }
  if (on_line && q != 0.0) {
    for (int side = 0; side < 2; ++side) {
      const double other = side ? a : -a;
      const double sign = side ? 1.0 : -1.0;
      if ((other - s0c) * sign <= 0.0) continue;
      const double len = fabs(other - sstar);
      pacc += q * e1_log_part(0.0, len, k.ct) / (4.0 * M_PI * k.kappa);
    }
  }
  p = pacc;
  const double2 t2 = cmul(e2t, make_double2(-4.0 * k.eta * d2acc.x, -4.0 * k.eta * d2acc.y));
  T = make_double2(-k.eta * pacc + t2.x, t2.y);
}

// Far form of the poroelastic part, affine in tau: F(tau) = F0 + tau F1 (the
// analytic branch of poro_element).  Returns F0(D0) + tau1 F1(D1) for two
// source triples (formula convention), used by the fast history sum where
// sum_{j <= j0} F(j dt) E_j = F0(sum E_j) + dt F1(sum j E_j).
__device__ void poro_far_split(double2 zt, double2 zc, double2 e, double a, double Ds0, double Dn0,
                               double Ds1, double Dn1, double q1, double tau1, const PoroConst& k,
                               double2 e2t, double2& T, double& p) {
  const double2 B0 = make_double2(Ds0 * e.x - Dn0 * e.y, Ds0 * e.y + Dn0 * e.x);
  const double2 B1 = make_double2(Ds1 * e.x - Dn1 * e.y, Ds1 * e.y + Dn1 * e.x);
  const double mu0 = -(k.eta / k.S) * Dn0;
  const double2 z1 = make_double2(zc.x - a * e.x, zc.y - a * e.y);
  const double2 z2 = make_double2(zc.x + a * e.x, zc.y + a * e.y);
  const double2 w1 = make_double2(zt.x - z1.x, zt.y - z1.y);
  const double2 w2 = make_double2(zt.x - z2.x, zt.y - z2.y);
  auto inv = [](double2 w) {
    const double n = fma(w.x, w.x, w.y * w.y);
    return make_double2(w.x / n, -w.y / n);
  };
  const double2 r1 = inv(w1), r2 = inv(w2);
  const double2 I2 = csub(r2, r1);
  const double2 r12 = cmul(r1, r1), r22 = cmul(r2, r2);
  const double2 I3 = cscale(csub(r22, r12), 0.5);
  const double2 I4 = cscale(csub(cmul(r22, r2), cmul(r12, r1)), 1.0 / 3.0);
  const double2 rr = make_double2(e.x * e.x - e.y * e.y, -2.0 * e.x * e.y);   // conj(e)^2
  const double2 dz = make_double2(zt.x - zc.x, zt.y - zc.y);
  double2 X = make_double2(zc.x, -zc.y);
  cmac(X, rr, dz);
  const double2 I3b = csub(cmul(X, I3), cmul(rr, I2));
  const double2 iGC = make_double2(0.0, k.gc);
  const double2 iGCB0 = cmul(iGC, B0), iGCB1 = cmul(iGC, B1);
  const double ekp = 2.0 * k.eta * k.kp;
  const double2 PhiD = cmul(iGCB0, I2);
  const double2 Phi = cscale(PhiD, ekp);
  const double2 dPhi = cscale(cmul(iGCB0, I3), -2.0 * ekp);
  const double ct1 = k.c * tau1;
  const double wm0 = k.eta * mu0 / M_PI;
  const double wm1 = k.eta * q1 * ct1 / (M_PI * k.kappa);
  double2 Psi = cscale(cmul(iGCB0, I3b), 2.0 * ekp);
  cmac(Psi, cscale(make_double2(e.x, -e.y), wm0 + wm1), I2);
  cmac(Psi, cscale(iGCB1, 48.0 * k.eta * k.kp * ct1), I4);
  double2 Wv = Psi;
  cmac(Wv, make_double2(zt.x, -zt.y), dPhi);
  const double2 t2 = cmul(e2t, Wv);
  T = make_double2(2.0 * Phi.x + t2.x, t2.y);
  p = -k.kp * 4.0 * PhiD.x;
}

namespace {

// drained elastic KM influence (tension-positive traction T = sigma_n + i sigma_s)
__device__ __forceinline__ double2 drained_traction(double2 zt, double2 zc, double2 e, double a,
                                                    double Ds, double Dn, double gc, double2 e2t) {
  const double2 B = make_double2(Ds * e.x - Dn * e.y, Ds * e.y + Dn * e.x);
  const double2 rr = make_double2(e.x * e.x - e.y * e.y, -2.0 * e.x * e.y);
  const double2 Q = csub(cmul(rr, B), make_double2(B.x, -B.y));
  const double2 z1 = make_double2(zc.x - a * e.x, zc.y - a * e.y);
  const double2 z2 = make_double2(zc.x + a * e.x, zc.y + a * e.y);
  const double2 w1 = make_double2(zt.x - z1.x, zt.y - z1.y);
  const double2 w2 = make_double2(zt.x - z2.x, zt.y - z2.y);
  const double n1 = fma(w1.x, w1.x, w1.y * w1.y), n2 = fma(w2.x, w2.x, w2.y * w2.y);
  const double2 r1 = make_double2(w1.x / n1, -w1.y / n1), r2 = make_double2(w2.x / n2, -w2.y / n2);
  const double2 I2 = csub(r2, r1);
  const double2 I3 = cscale(csub(cmul(r2, r2), cmul(r1, r1)), 0.5);
  const double2 dz = make_double2(zt.x - zc.x, zt.y - zc.y);
  double2 X = make_double2(zc.x, -zc.y);
  cmac(X, rr, dz);
  const double2 I3b = csub(cmul(X, I3), cmul(rr, I2));
  const double2 iGC = make_double2(0.0, gc);
  const double2 Phi = cmul(iGC, cmul(B, I2));
  const double2 dPhi = cscale(cmul(iGC, cmul(B, I3)), -2.0);
  double2 Psi = cmul(Q, I2);
  cmac(Psi, cscale(B, 2.0), I3b);
  Psi = cmul(iGC, Psi);
  double2 Wv = Psi;
  cmac(Wv, make_double2(zt.x, -zt.y), dPhi);
  const double2 t2 = cmul(e2t, Wv);
  return make_double2(2.0 * Phi.x + t2.x, t2.y);
}

// full 3x3 action of one source (Ds, Dn, q ABI) on one target: adds
// (sigma_s, sigma_n, p) in ABI convention
__device__ __forceinline__ void poro_pair(double2 zt, double2 e2t, const double* sp,
                                          const PoroConst& k, double& os, double& on,
                                          double& op) {
  const double2 zc = make_double2(sp[0], sp[1]);
  const double2 e = make_double2(sp[2], sp[3]);
  const double a = sp[4];
  const double Ds = sp[5], Dn = sp[6], q = -sp[7];   // J: q_formula = -q_ABI
  const double2 Td = drained_traction(zt, zc, e, a, Ds, Dn, k.gc, e2t);
  double2 Tp;
  double p;
  poro_element(zt, zc, e, a, Ds, Dn, q, k, e2t, Tp, p);
  os += Td.y + Tp.y;
  on += Td.x + Tp.x;
  op -= p;                                             // J: p_ABI = -p_formula
}

// drained part + (far-form poroelastic part unless the pair is in the near-rule
// regime); returns true if the near-rule part is still to be added
__device__ __forceinline__ bool poro_pair_split(double2 zt, double2 e2t, const double* sp,
                                                const PoroConst& k, double& os, double& on,
                                                double& op) {
  const double2 zc = make_double2(sp[0], sp[1]);
  const double2 e = make_double2(sp[2], sp[3]);
  const double a = sp[4];
  const double Ds = sp[5], Dn = sp[6], q = -sp[7];   // J: q_formula = -q_ABI
  const double2 Td = drained_traction(zt, zc, e, a, Ds, Dn, k.gc, e2t);
  os += Td.y;
  on += Td.x;
  if (poro_is_near(zt, zc, e, a, k.ct)) return true;
  double2 Tp;
  double p;
  poro_element(zt, zc, e, a, Ds, Dn, q, k, e2t, Tp, p);   // analytic far form
  os += Tp.y;
  on += Tp.x;
  op -= p;                                                 // J: p_ABI = -p_formula
  return false;
}

constexpr int kPoroStride = 8;   // {zc, e, a, Ds, Dn, q}
constexpr int kQueue = 64;       // per-warp queue of near-rule pairs (flushed at >= 32)

// per-warp near-rule queue: entries (target slot, source, lag) evaluated one
// at a time by the whole warp (poro_near_coop); sums per target slot in
// queue order (deterministic)
constexpr int kBatchQ = 16;   // queue entries whose panels are generated in parallel
constexpr int kBP = 32;       // panel breakpoints per side kept for a batched entry
struct NearQueue {
  int t[kQueue], s[kQueue], j[kQueue];
  double acc[3][kTgtGroup];
  double coop[2 * (kCoopPanels + 1) + 2];   // fallback (entries with > kBP panels a side)
  double bp[kBatchQ][2][kBP + 1];
  int np[kBatchQ][2];                       // panels per side, -1 = more than kBP
};

// the default sink of a flushed entry: add (T, p) to its target slot in ABI
// convention (sigma_s, sigma_n, p): J: p_ABI = -p_formula
struct AccSink {
  NearQueue* Q;
  __device__ void operator()(int qi, double2 T, double p) const {
    const int slot = Q->t[qi];
    Q->acc[0][slot] += T.y;
    Q->acc[1][slot] += T.x;
    Q->acc[2][slot] -= p;
  }
};

// One queued near-rule evaluation: target (zt, e2t), source element (zc, e,
// a), source strengths (formula convention) and c tau.
struct NearDesc {
  double2 zt, e2t, zc, e;
  double a, Ds, Dn, q, ct;
};

// Phase A of a queue flush: graded panel breakpoints of entries [base,
// base + ng), lane = (entry, side).
template <class Desc>
__device__ void near_queue_panels(NearQueue& Q, int base, int ng, int lane, const Desc& desc) {
  {  // phase A: panel breakpoints, lane = (entry, side)
    const int ei = lane >> 1, side = lane & 1;
    if (ei < ng) {
      const NearDesc d = desc(base + ei);
      const double lt = sqrt(d.ct);
      const double rx = d.zt.x - d.zc.x, ry = d.zt.y - d.zc.y;
      const double sstar = rx * d.e.x + ry * d.e.y;
      const double dperp = fabs(-rx * d.e.y + ry * d.e.x);
      const double s0c = fmin(fmax(sstar, -d.a), d.a);
      const double other = side ? d.a : -d.a;
      const double sign = side ? 1.0 : -1.0;
      double* b = Q.bp[ei][side];
      double cur = s0c;
      int np = 0;
      b[0] = cur;
      bool over = false;
      if ((other - s0c) * sign > 0.0) {
        while ((other - cur) * sign > 0.0) {
          if (np == kBP) {
            over = true;
            break;
          }
          const double r = hypot(dperp, cur - sstar);
          double snext = cur + sign * kPanelFraction * fmax(r, lt);
          if ((other - snext) * sign <= 0.0) snext = other;
          b[++np] = snext;
          cur = snext;
        }
      }
      Q.np[ei][side] = over ? -1 : np;
    }
  }
}

// Flush the queue: entries in batches of kBatchQ; lanes 2i, 2i+1 generate the
// graded panels of entry i's two sides in parallel (the sequential recurrence
// of poro_element), then the warp integrates the entries one at a time (32
// lanes over the 8 x panels Gauss–Legendre nodes) and lane 0 adds the result
// to the entry's target slot -- in queue order (deterministic).  desc(qi)
// returns entry qi's NearDesc.
template <class Desc, class Sink>
__device__ void near_queue_flush(NearQueue& Q, int qn, int lane, const PoroConst& k0,
                                 const Desc& desc, const Sink& sink) {
  __syncwarp();
  for (int base = 0; base < qn; base += kBatchQ) {
    const int ng = min(kBatchQ, qn - base);
    near_queue_panels(Q, base, ng, lane, desc);
    __syncwarp();
    for (int ei = 0; ei < ng; ++ei) {   // phase B: the warp integrates entry ei
      const NearDesc d = desc(base + ei);
      PoroConst k = k0;
      k.ct = d.ct;
      double2 T;
      double p;
      const int n0 = Q.np[ei][0], n1 = Q.np[ei][1];
      if (n0 < 0 || n1 < 0) {
        poro_near_coop(d.zt, d.zc, d.e, d.a, d.Ds, d.Dn, d.q, k, d.e2t, Q.coop, lane, T, p);
      } else {
        const double rx = d.zt.x - d.zc.x, ry = d.zt.y - d.zc.y;
        const double sstar = rx * d.e.x + ry * d.e.y;
        const double dperp = fabs(-rx * d.e.y + ry * d.e.x);
        const double2 B = make_double2(d.Ds * d.e.x - d.Dn * d.e.y, d.Ds * d.e.y + d.Dn * d.e.x);
        const double mu = -(k.eta / k.S) * d.Dn;
        const double2 K = cscale(cmul(make_double2(0.0, k.gc), cmul(B, d.e)), -4.0 * k.kp);
        const bool on_line = (dperp == 0.0) && (fabs(sstar) < d.a);
        const double s0c = fmin(fmax(sstar, -d.a), d.a);
        double pacc = 0.0;
        double2 d2acc = make_double2(0.0, 0.0);
        const int npts = 8 * (n0 + n1);
        for (int t = lane; t < npts; t += 32) {
          const int pan = t >> 3, g = t & 7;
          const int side = pan < n0 ? 0 : 1;
          const int pi = side ? pan - n0 : pan;
          const double* b = Q.bp[ei][side];
          const double s0 = b[pi], s1 = b[pi + 1];
          const double mid = 0.5 * (s0 + s1), half = 0.5 * fabs(s1 - s0);
          const double sq = mid + half * c_gl_x[g];
          const double wx = d.zt.x - (d.zc.x + sq * d.e.x), wy = d.zt.y - (d.zc.y + sq * d.e.y);
          point_add(wx, wy, half * c_gl_w[g], k, K, mu, d.q, on_line, pacc, d2acc);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
          pacc += __shfl_xor_sync(0xffffffffu, pacc, o);
          d2acc.x += __shfl_xor_sync(0xffffffffu, d2acc.x, o);
          d2acc.y += __shfl_xor_sync(0xffffffffu, d2acc.y, o);
        }
        if (on_line && d.q != 0.0) {
          for (int side = 0; side < 2; ++side) {
            const double other = side ? d.a : -d.a;
            const double sign = side ? 1.0 : -1.0;
            if ((other - s0c) * sign <= 0.0) continue;
            const double len = fabs(other - sstar);
            pacc += d.q * e1_log_part(0.0, len, k.ct) / (4.0 * M_PI * k.kappa);
          }
        }
        p = pacc;
        const double2 t2 =
            cmul(d.e2t, make_double2(-4.0 * k.eta * d2acc.x, -4.0 * k.eta * d2acc.y));
        T = make_double2(-k.eta * pacc + t2.x, t2.y);
      }
      if (lane == 0) sink(base + ei, T, p);
      __syncwarp();
    }
  }
}

// near_queue_flush for the three unit source columns of each entry (near-
// field block builds, §4.5b/§4.6b): one quadrature pass per entry gives all
// three columns (point_add3); sink(qi, T[3], p[3]).  desc(qi) supplies the
// geometry and c tau (its strengths are ignored).
template <class Desc, class Sink>
__device__ void near_queue_flush3(NearQueue& Q, int qn, int lane, const PoroConst& k0,
                                  const Desc& desc, const Sink& sink) {
  __syncwarp();
  for (int base = 0; base < qn; base += kBatchQ) {
    const int ng = min(kBatchQ, qn - base);
    near_queue_panels(Q, base, ng, lane, desc);
    __syncwarp();
    for (int ei = 0; ei < ng; ++ei) {
      const NearDesc d = desc(base + ei);
      PoroConst k = k0;
      k.ct = d.ct;
      double2 T[3];
      double p[3];
      const int n0 = Q.np[ei][0], n1 = Q.np[ei][1];
      if (n0 < 0 || n1 < 0) {   // long panel lists: the per-column cooperative rule
        for (int c = 0; c < 3; ++c)
          poro_near_coop(d.zt, d.zc, d.e, d.a, c == 0 ? 1.0 : 0.0, c == 1 ? 1.0 : 0.0,
                         c == 2 ? -1.0 : 0.0, k, d.e2t, Q.coop, lane, T[c], p[c]);
      } else {
        const double rx = d.zt.x - d.zc.x, ry = d.zt.y - d.zc.y;
        const double sstar = rx * d.e.x + ry * d.e.y;
        const double dperp = fabs(-rx * d.e.y + ry * d.e.x);
        const double2 K0 = cscale(cmul(make_double2(0.0, k.gc), cmul(d.e, d.e)), -4.0 * k.kp);
        const double mu1 = -(k.eta / k.S);
        const bool on_line = (dperp == 0.0) && (fabs(sstar) < d.a);
        const double s0c = fmin(fmax(sstar, -d.a), d.a);
        double pacc[3] = {0.0, 0.0, 0.0};
        double2 d2acc[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
        const int npts = 8 * (n0 + n1);
        for (int t = lane; t < npts; t += 32) {
          const int pan = t >> 3, g = t & 7;
          const int side = pan < n0 ? 0 : 1;
          const int pi = side ? pan - n0 : pan;
          const double* b = Q.bp[ei][side];
          const double s0 = b[pi], s1 = b[pi + 1];
          const double mid = 0.5 * (s0 + s1), half = 0.5 * fabs(s1 - s0);
          const double sq = mid + half * c_gl_x[g];
          const double wx = d.zt.x - (d.zc.x + sq * d.e.x), wy = d.zt.y - (d.zc.y + sq * d.e.y);
          point_add3(wx, wy, half * c_gl_w[g], k, K0, mu1, on_line, pacc, d2acc);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            pacc[c] += __shfl_xor_sync(0xffffffffu, pacc[c], o);
            d2acc[c].x += __shfl_xor_sync(0xffffffffu, d2acc[c].x, o);
            d2acc[c].y += __shfl_xor_sync(0xffffffffu, d2acc[c].y, o);
          }
        if (on_line) {   // analytic log part of E1 on the element, column 2 (q = -1)
          for (int side = 0; side < 2; ++side) {
            const double other = side ? d.a : -d.a;
            const double sign = side ? 1.0 : -1.0;
            if ((other - s0c) * sign <= 0.0) continue;
            const double len = fabs(other - sstar);
            pacc[2] -= e1_log_part(0.0, len, k.ct) / (4.0 * M_PI * k.kappa);
          }
        }
        for (int c = 0; c < 3; ++c) {
          p[c] = pacc[c];
          const double2 t2 =
              cmul(d.e2t, make_double2(-4.0 * k.eta * d2acc[c].x, -4.0 * k.eta * d2acc[c].y));
          T[c] = make_double2(-k.eta * pacc[c] + t2.x, t2.y);
        }
      }
      if (lane == 0) sink(base + ei, T, p);
      __syncwarp();
    }
  }
}

__global__ void poro_prep(int64_t n, const int* __restrict__ perm, const double* __restrict__ D,
                          const double* __restrict__ ex, const double* __restrict__ ey,
                          const double* __restrict__ ea, const double* __restrict__ ec,
                          const double* __restrict__ es, double* __restrict__ src,
                          double* __restrict__ dsort) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm ? perm[i] : (int)i;
  double* o = src + i * kPoroStride;
  o[0] = ex[i];
  o[1] = ey[i];
  o[2] = ec[i];
  o[3] = es[i];
  o[4] = ea[i];
  const double d0 = D[(int64_t)j * 3 + 0], d1 = D[(int64_t)j * 3 + 1], d2 = D[(int64_t)j * 3 + 2];
  o[5] = d0;
  o[6] = d1;
  o[7] = d2;
  if (dsort) {   // D gathered into sorted order for the upward pass
    dsort[i * 3 + 0] = d0;
    dsort[i * 3 + 1] = d1;
    dsort[i * 3 + 2] = d2;
  }
}

// near field: warp per item (<= kTgtGroup targets); lane = (target, slice).
// The cheap parts (drained closed form, far-form poroelastic part) run per
// lane; pairs in the near-rule regime go to a per-warp queue and are
// integrated by all 32 lanes together (poro_near_coop), so the quadrature does
// not serialise a warp on a few divergent lanes.
__global__ void __launch_bounds__(128)
poro_p2p_kernel(int nown, const int* __restrict__ order, const int4* __restrict__ items,
                const int* __restrict__ u_off, const int* __restrict__ u_lo,
                const int* __restrict__ u_hi, const int* __restrict__ leaves,
                const int* __restrict__ c_start, const int* __restrict__ c_count,
                const double* __restrict__ src, const double* __restrict__ ex,
                const double* __restrict__ ey, const double* __restrict__ ec,
                const double* __restrict__ es, PoroConst k, int G, double* __restrict__ gpart,
                double* __restrict__ part3) {
  __shared__ double red[4][3][32];
  __shared__ NearQueue nq[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  NearQueue& Q = nq[w];
  const unsigned lt_mask = (1u << lane) - 1u;
  // warp task = (owned item oi, source group grp of G): the item's rounds of S
  // sources are dealt round-robin to the groups; G > 1 writes per-group
  // partials gpart[grp][oi][t][3] (summed in order by poro_hist_reduce)
  for (int task = blockIdx.x * 4 + w; task < nown * G; task += gridDim.x * 4) {
    const int oi = task / G, grp = task - oi * G;
    const int it = order[oi];
    const int4 item = items[it];
    const int kk = item.x;
    const int c = leaves[kk];
    const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
    const int S = 32 / nt;
    const int tl = lane % nt, slice = lane / nt;
    const bool active = slice < S;
    const int ti = item.y + tl;
    const double2 zt = make_double2(ex[ti], ey[ti]);
    const double ctg = ec[ti], stg = es[ti];
    const double2 e2t = make_double2(ctg * ctg - stg * stg, 2.0 * ctg * stg);
    for (int e = lane; e < 3 * kTgtGroup; e += 32) (&Q.acc[0][0])[e] = 0.0;
    int qn = 0;
    double os = 0.0, on = 0.0, op = 0.0;
    auto desc = [&](int qi) {
      const int tg = item.y + Q.t[qi];
      const double cq = ec[tg], sq = es[tg];
      const double* sp = src + (int64_t)Q.s[qi] * kPoroStride;
      NearDesc d;
      d.zt = make_double2(ex[tg], ey[tg]);
      d.e2t = make_double2(cq * cq - sq * sq, 2.0 * cq * sq);
      d.zc = make_double2(sp[0], sp[1]);
      d.e = make_double2(sp[2], sp[3]);
      d.a = sp[4];
      d.Ds = sp[5];
      d.Dn = sp[6];
      d.q = -sp[7];   // J: q_formula = -q_ABI
      d.ct = k.ct;
      return d;
    };
    auto flush = [&]() {
      near_queue_flush(Q, qn, lane, k, desc, AccSink{&Q});
      qn = 0;
    };
    int pos = 0;
    for (int r = u_off[kk], rend = u_off[kk + 1]; r < rend && pos < item.w; ++r) {
      const int lo = u_lo[r], len = u_hi[r] - lo;
      const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
      for (int jb = b; jb < e; jb += S) {
        if (G > 1 && ((pos + jb - item.z) / S) % G != grp) continue;   // another warp's round
        const int j = jb + slice;
        bool near = false;
        if (active && j < e)
          near = poro_pair_split(zt, e2t, src + (int64_t)(lo + j) * kPoroStride, k, os, on, op);
        const unsigned m = __ballot_sync(0xffffffffu, near);
        if (near) {
          const int idx = qn + __popc(m & lt_mask);
          Q.t[idx] = tl;
          Q.s[idx] = lo + j;
        }
        qn += __popc(m);
        if (qn >= 32) flush();
      }
      pos += len;
    }
    flush();
    if (active) {
      red[w][0][lane] = os;
      red[w][1][lane] = on;
      red[w][2][lane] = op;
    }
    __syncwarp();
    if (lane < kTgtGroup) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      if (lane < nt) {
        for (int q = 0; q < S; ++q) {
          s0 += red[w][0][lane + q * nt];
          s1 += red[w][1][lane + q * nt];
          s2 += red[w][2][lane + q * nt];
        }
        s0 += Q.acc[0][lane];
        s1 += Q.acc[1][lane];
        s2 += Q.acc[2][lane];
      }
      double* o = G > 1 ? gpart + (((int64_t)grp * nown + oi) * kTgtGroup + lane) * 3
                        : part3 + ((int64_t)it * kTgtGroup + lane) * 3;
      o[0] = s0;
      o[1] = s1;
      o[2] = s2;
    }
    __syncwarp();
  }
}

__global__ void poro_direct_kernel(int64_t n, int64_t t_lo, int64_t t_hi,
                                   const double* __restrict__ src, const double* __restrict__ ex,
                                   const double* __restrict__ ey, const double* __restrict__ ec,
                                   const double* __restrict__ es, PoroConst k,
                                   const int* __restrict__ perm, double* __restrict__ y_user,
                                   double* __restrict__ y_sorted) {
  const int64_t ti = t_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ti >= t_hi) return;
  const double2 zt = make_double2(ex[ti], ey[ti]);
  const double ct = ec[ti], st = es[ti];
  const double2 e2t = make_double2(ct * ct - st * st, 2.0 * ct * st);
  double os = 0.0, on = 0.0, op = 0.0;
  for (int64_t j = 0; j < n; ++j) poro_pair(zt, e2t, src + j * kPoroStride, k, os, on, op);
  if (y_sorted) {
    y_sorted[ti * 3] = os;
    y_sorted[ti * 3 + 1] = on;
    y_sorted[ti * 3 + 2] = op;
  }
  if (y_user) {
    const int j = perm[ti];
    y_user[(int64_t)j * 3] = os;
    y_user[(int64_t)j * 3 + 1] = on;
    y_user[(int64_t)j * 3 + 2] = op;
  }
}

// ---------------------------------------------------------------- near cache
// Near-field matrix cache.  Inside GMRES (and any repeated
// matvec at one elapsed time) the near-field influence blocks are the same at
// every iteration, and the poroelastic ones are expensive (graded quadrature
// with E1).  The 3x3 block of every owned near pair is evaluated once, with
// the same functions as poro_p2p_kernel (per-lane drained + far form, the
// warp-cooperative near rule for near-rule pairs, one unit source component
// at a time), and each later matvec applies the blocks (9 FMA and 72 B per
// pair: HBM bound).  Layout per item: block (jpos, t) at
// nc_off[item] + (jpos kTgtGroup + t) 9, row r = (sigma_s, sigma_n, p), column c =
// (Ds, Dn, q), ABI convention.
constexpr int kBuildGroups = 8;   // warps per item in the block builds

__global__ void __launch_bounds__(128)
poro_near_build_kernel(int nown, const int* __restrict__ order, const int4* __restrict__ items,
                       int item_lo, const int* __restrict__ u_off, const int* __restrict__ u_lo,
                       const int* __restrict__ u_hi, const int* __restrict__ leaves,
                       const int* __restrict__ c_start, const int* __restrict__ c_count,
                       const double* __restrict__ ex, const double* __restrict__ ey,
                       const double* __restrict__ ea, const double* __restrict__ ec,
                       const double* __restrict__ es, PoroConst k, int drained, int lstride,
                       int lidx, const int64_t* __restrict__ ioff, double* __restrict__ cache) {
  __shared__ NearQueue nq[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  NearQueue& Q = nq[w];
  const unsigned lt_mask = (1u << lane) - 1u;
  // warp task = (owned item, source group grp of kBuildGroups): the item's
  // rounds of S sources are dealt round-robin to its groups (the blocks of a
  // pair are written by exactly one warp: disjoint, no ordering needed)
  for (int task = blockIdx.x * 4 + w; task < nown * kBuildGroups; task += gridDim.x * 4) {
    const int oi = task / kBuildGroups, grp = task - oi * kBuildGroups;
    const int it = order[oi];
    const int4 item = items[it];
    const int kk = item.x;
    const int c = leaves[kk];
    const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
    const int S = 32 / nt;
    const int tl = lane % nt, slice = lane / nt;
    const bool active = slice < S;
    const int ti = item.y + tl;
    const double2 zt = make_double2(ex[ti], ey[ti]);
    const double ctg = ec[ti], stg = es[ti];
    const double2 e2t = make_double2(ctg * ctg - stg * stg, 2.0 * ctg * stg);
    // block (jpos, t) of lag slot lidx: ((jpos lstride + lidx) kTgtGroup + t) 9
    double* blk0 = cache + ioff[it - item_lo] * lstride + (int64_t)lidx * kTgtGroup * 9;
    const int64_t jstride = (int64_t)lstride * kTgtGroup * 9;
    int qn = 0;
    // queue entry: t = target slot, s = source element, j = jpos (all three
    // unit columns of the pair integrated together, near_queue_flush3)
    auto desc = [&](int qi) {
      const int tg = item.y + Q.t[qi];
      const int sj = Q.s[qi];
      const double cq = ec[tg], sq = es[tg];
      NearDesc d;
      d.zt = make_double2(ex[tg], ey[tg]);
      d.e2t = make_double2(cq * cq - sq * sq, 2.0 * cq * sq);
      d.zc = make_double2(ex[sj], ey[sj]);
      d.e = make_double2(ec[sj], es[sj]);
      d.a = ea[sj];
      d.Ds = d.Dn = d.q = 0.0;   // unused by near_queue_flush3
      d.ct = k.ct;
      return d;
    };
    auto sink = [&](int qi, const double2* T, const double* p) {
      double* b = blk0 + (int64_t)Q.j[qi] * jstride + Q.t[qi] * 9;
      for (int comp = 0; comp < 3; ++comp) {
        b[comp] += T[comp].y;
        b[3 + comp] += T[comp].x;
        b[6 + comp] -= p[comp];   // J: p_ABI = -p_formula
      }
    };
    int pos = 0;
    for (int r = u_off[kk], rend = u_off[kk + 1]; r < rend && pos < item.w; ++r) {
      const int lo = u_lo[r], len = u_hi[r] - lo;
      const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
      for (int jb = b; jb < e; jb += S) {
        if (((pos + jb - item.z) / S) % kBuildGroups != grp) continue;   // another warp's round
        const int j = jb + slice;
        const bool have = active && j < e;
        const int jpos = pos + j - item.z;
        double sp[kPoroStride];
        if (have) {
          sp[0] = ex[lo + j];
          sp[1] = ey[lo + j];
          sp[2] = ec[lo + j];
          sp[3] = es[lo + j];
          sp[4] = ea[lo + j];
        }
        bool near = false;
        if (have) {
          const double2 zc = make_double2(sp[0], sp[1]), e = make_double2(sp[2], sp[3]);
          near = poro_is_near(zt, zc, e, sp[4], k.ct);
          double* bb = blk0 + jpos * jstride + tl * 9;
          for (int comp = 0; comp < 3; ++comp) {
            const double Ds = comp == 0 ? 1.0 : 0.0, Dn = comp == 1 ? 1.0 : 0.0;
            double os = 0.0, on = 0.0, op = 0.0;
            if (drained) {
              const double2 Td = drained_traction(zt, zc, e, sp[4], Ds, Dn, k.gc, e2t);
              os += Td.y;
              on += Td.x;
            }
            if (!near) {   // analytic far form of the poroelastic part
              double2 Tp;
              double pp;
              poro_element(zt, zc, e, sp[4], Ds, Dn, comp == 2 ? -1.0 : 0.0, k, e2t, Tp, pp);
              os += Tp.y;
              on += Tp.x;
              op -= pp;   // J: p_ABI = -p_formula
            }
            bb[comp] = os;
            bb[3 + comp] = on;
            bb[6 + comp] = op;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, near);
        if (near) {
          const int idx = qn + __popc(m & lt_mask);
          Q.t[idx] = tl;
          Q.s[idx] = lo + j;
          Q.j[idx] = jpos;
        }
        qn += __popc(m);
        if (qn >= 32) {
          near_queue_flush3(Q, qn, lane, k, desc, sink);
          qn = 0;
        }
      }
      pos += len;
    }
    near_queue_flush3(Q, qn, lane, k, desc, sink);
    __syncwarp();
  }
}

// y_near = blocks x D per owned item: block per item, its kApplyWarps warps
// take interleaved groups of the source positions, lane = (target, slice);
// partials reduced in a fixed order (deterministic).  Same partial layout as
// poro_p2p_kernel.
constexpr int kApplyWarps = 8;

// DDM_NC_STREAM=1: the near-field matrix cache (134 MB on config 3, read once
// per matvec) is read with the streaming (evict-first) cache hint, so it does
// not push the GMRES Krylov basis out of L2 between Arnoldi steps
#ifndef DDM_NC_STREAM
#define DDM_NC_STREAM 1
#endif
__device__ __forceinline__ double nc_ld(const double* p) {
#if DDM_NC_STREAM
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

__global__ void __launch_bounds__(kApplyWarps * 32)
poro_near_apply_kernel(const int* __restrict__ order, const int4* __restrict__ items,
                       int item_lo, const int* __restrict__ u_off, const int* __restrict__ u_lo,
                       const int* __restrict__ u_hi, const int* __restrict__ leaves,
                       const int* __restrict__ c_start, const int* __restrict__ c_count,
                       const double* __restrict__ src, const int64_t* __restrict__ ioff,
                       const double* __restrict__ cache, double* __restrict__ part3) {
  __shared__ double red[kApplyWarps][3][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int it = order[blockIdx.x];
  const int4 item = items[it];
  const int kk = item.x;
  const int c = leaves[kk];
  const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
  const int S = 32 / nt;
  const int tl = lane % nt, slice = lane / nt;
  const bool active = slice < S;
  const double* blk0 = cache + ioff[it - item_lo];
  double os = 0.0, on = 0.0, op = 0.0;
  if (active) {
    int pos = 0;
    for (int r = u_off[kk], rend = u_off[kk + 1]; r < rend && pos < item.w; ++r) {
      const int lo = u_lo[r], len = u_hi[r] - lo;
      const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
#pragma unroll 2
      for (int j = b + slice + S * w; j < e; j += S * kApplyWarps) {
        const int jpos = pos + j - item.z;
        const double* bb = blk0 + ((int64_t)jpos * kTgtGroup + tl) * 9;
        const double* d = src + (int64_t)(lo + j) * kPoroStride + 5;
        const double d0 = __ldg(d), d1 = __ldg(d + 1), d2 = __ldg(d + 2);
        os = fma(nc_ld(bb + 0), d0, fma(nc_ld(bb + 1), d1, fma(nc_ld(bb + 2), d2, os)));
        on = fma(nc_ld(bb + 3), d0, fma(nc_ld(bb + 4), d1, fma(nc_ld(bb + 5), d2, on)));
        op = fma(nc_ld(bb + 6), d0, fma(nc_ld(bb + 7), d1, fma(nc_ld(bb + 8), d2, op)));
      }
      pos += len;
    }
  }
  red[w][0][lane] = os;
  red[w][1][lane] = on;
  red[w][2][lane] = op;
  __syncthreads();
  if (w == 0 && lane < kTgtGroup) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (lane < nt)
      for (int ww = 0; ww < kApplyWarps; ++ww)
        for (int q = 0; q < S; ++q) {
          s0 += red[ww][0][lane + q * nt];
          s1 += red[ww][1][lane + q * nt];
          s2 += red[ww][2][lane + q * nt];
        }
    double* o = part3 + ((int64_t)it * kTgtGroup + lane) * 3;
    o[0] = s0;
    o[1] = s1;
    o[2] = s2;
  }
}

// History near field from the lag cache:
//   r_near(t) = sum_s sum_{j=1}^{h+1} K^p_ts(j dt) E_j(s),  E_j = D^(h+1-j) - D^(h-j)
// with the cached blocks of every lag (the drained part cancels, sum_j E_j = 0).
// Lags are stored in chunks of kLagChunk: in a chunk the blocks of one pair's
// successive lags are adjacent ([item][jpos][lag][t][9]), so a lane streams
// through contiguous memory and a warp touches few pages.  Warp per item,
// lane = (target, source slice); per (pair, lag) 9 FMA on a 72-B block (HBM
// bound).  Same partial layout as poro_hist_near_kernel.
constexpr int kLagChunk = 16;
constexpr int kHistWarps = 8;   // warps per (item, lag chunk) block, splitting the sources

// grid (owned item i, lag chunk q): the block sums lags 16q+1 .. 16q+16 of
// every pair of item order[i] (its warps take interleaved source groups) and
// writes its per-target partial to hpart[q][i][t][3]; poro_hist_reduce sums
// the chunks in order (deterministic).
__global__ void __launch_bounds__(kHistWarps * 32)
poro_hist_cached_kernel(const int* __restrict__ order, const int4* __restrict__ items,
                        int item_lo, int nown, const int* __restrict__ u_off,
                        const int* __restrict__ u_lo, const int* __restrict__ u_hi,
                        const int* __restrict__ leaves, const int* __restrict__ c_start,
                        const int* __restrict__ c_count, const double* __restrict__ Hs, int h,
                        const int64_t* __restrict__ ioff, const double* const* __restrict__ chunks,
                        double* __restrict__ hpart) {
  __shared__ double red[kHistWarps][3][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hs = (h + 2) * 3;
  const int oi = blockIdx.x, q = blockIdx.y;
  const int it = order[oi];
  const int4 item = items[it];
  const int kk = item.x;
  const int c = leaves[kk];
  const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
  const int S = 32 / nt;
  const int tl = lane % nt, slice = lane / nt;
  const bool active = slice < S;
  const int l0 = q * kLagChunk;
  const int ln = min(kLagChunk, h + 1 - l0);
  const double* ch = chunks[q] + ioff[it - item_lo] * kLagChunk;
  double os = 0.0, on = 0.0, op = 0.0;
  if (active) {
    int pos = 0;
    for (int r = u_off[kk], rend = u_off[kk + 1]; r < rend && pos < item.w; ++r) {
      const int lo = u_lo[r], len = u_hi[r] - lo;
      const int b = max(item.z - pos, 0), e = min(item.w - pos, len);
      for (int j = b + slice + S * w; j < e; j += S * kHistWarps) {
        const double* bb0 = ch + ((int64_t)(pos + j - item.z) * kLagChunk * kTgtGroup + tl) * 9;
        // lags l = l0+1 .. l0+ln: E_l = D^(h+1-l) - D^(h-l) = H[h+2-l] - H[h+1-l]
        const double* H = Hs + (int64_t)(lo + j) * hs + (h + 1 - l0) * 3;
        double dp0 = __ldg(H), dp1 = __ldg(H + 1), dp2 = __ldg(H + 2);
#pragma unroll 4
        for (int li = 0; li < ln; ++li) {
          const double* Db = H - 3 * (li + 1);
          const double d0 = __ldg(Db), d1 = __ldg(Db + 1), d2 = __ldg(Db + 2);
          const double e0 = dp0 - d0, e1 = dp1 - d1, e2 = dp2 - d2;
          dp0 = d0;
          dp1 = d1;
          dp2 = d2;
          const double* bb = bb0 + li * (kTgtGroup * 9);
          os = fma(__ldg(bb + 0), e0, fma(__ldg(bb + 1), e1, fma(__ldg(bb + 2), e2, os)));
          on = fma(__ldg(bb + 3), e0, fma(__ldg(bb + 4), e1, fma(__ldg(bb + 5), e2, on)));
          op = fma(__ldg(bb + 6), e0, fma(__ldg(bb + 7), e1, fma(__ldg(bb + 8), e2, op)));
        }
      }
      pos += len;
    }
  }
  red[w][0][lane] = os;
  red[w][1][lane] = on;
  red[w][2][lane] = op;
  __syncthreads();
  if (w == 0 && lane < kTgtGroup) {   // fixed order: warps, then slices
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (lane < nt)
      for (int ww = 0; ww < kHistWarps; ++ww)
        for (int sl = 0; sl < S; ++sl) {
          s0 += red[ww][0][lane + sl * nt];
          s1 += red[ww][1][lane + sl * nt];
          s2 += red[ww][2][lane + sl * nt];
        }
    double* o = hpart + (((int64_t)q * nown + oi) * kTgtGroup + lane) * 3;
    o[0] = s0;
    o[1] = s1;
    o[2] = s2;
  }
}

// part3[item order[i]][t] = sum over the lag chunks q (in order) of hpart[q][i][t]
__global__ void poro_hist_reduce(int nown, int nch, const int* __restrict__ order,
                                 const double* __restrict__ hpart, double* __restrict__ part3) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // (i, t, comp)
  if (e >= (int64_t)nown * kTgtGroup * 3) return;
  const int i = (int)(e / (kTgtGroup * 3));
  const int rem = (int)(e - (int64_t)i * kTgtGroup * 3);
  double s = 0.0;
  for (int q = 0; q < nch; ++q) s += hpart[(int64_t)q * nown * kTgtGroup * 3 + e];
  part3[(int64_t)order[i] * kTgtGroup * 3 + rem] = s;
}

// ---------------------------------------------------------------- fast history (f1)
// D_hist [h][n][3] (user order, ABI) -> Hs[i][k'][3] (sorted element i,
// k' = 0..h+1 holds D^(k'-1), D^-1 = D^h = 0) and Cs[i][k][3] = sum_{k''<k} D^k''
// (k = 0..h).  Thread per (element, component).
__global__ void hist_gather(int64_t n, int h, const int* __restrict__ perm,
                            const double* __restrict__ Dh, double* __restrict__ Hs,
                            double* __restrict__ Cs, double* __restrict__ Ctot) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * 3) return;
  const int64_t i = t / 3;
  const int c = (int)(t - i * 3);
  const int64_t j = perm[i];
  double* H = Hs + i * (int64_t)(h + 2) * 3 + c;
  double* C = Cs + i * (int64_t)(h + 1) * 3 + c;
  H[0] = 0.0;
  double acc = 0.0;
  C[0] = 0.0;
  for (int k = 0; k < h; ++k) {
    const double d = Dh[((int64_t)k * n + j) * 3 + c];
    H[(k + 1) * 3] = d;
    acc += d;
    C[(k + 1) * 3] = acc;
  }
  H[(h + 1) * 3] = 0.0;
  Ctot[i * 3 + c] = acc;   // C[h] = sum_{k<h} D^k: source of the far pass (sorted)
}

// Near field of the history sum, one launch for all lags:
//   r = sum_{j=1}^{h+1} K(j dt) E_j,  E_j = D^(h+1-j) - D^(h-j)
// The drained part of K is tau independent and sum_j E_j = 0, so only the
// poroelastic part is summed.  Per pair, lags j <= j0 (the far-form lags of
// poro_element: dist^2 / (4 c j dt) > 40, the same decision as a per-lag
// matvec) collapse to F0(S0) + dt F1(S1) with S0 = sum_{j<=j0} E_j = -D^(h-j0)
// and S1 = sum_{j<=j0} j E_j = C[h] - C[h+1-j0] - j0 D^(h-j0); the remaining
// lags use the near rule at tau = j dt.
__global__ void __launch_bounds__(128)
poro_hist_near_kernel(int nown, const int* __restrict__ order, const int4* __restrict__ items,
                      const int* __restrict__ u_off, const int* __restrict__ u_lo,
                      const int* __restrict__ u_hi, const int* __restrict__ leaves,
                      const int* __restrict__ c_start, const int* __restrict__ c_count,
                      const double* __restrict__ src, const double* __restrict__ Hs,
                      const double* __restrict__ Cs, int h, double dt,
                      const double* __restrict__ ex, const double* __restrict__ ey,
                      const double* __restrict__ ec, const double* __restrict__ es, PoroConst k,
                      int G, double* __restrict__ gpart, double* __restrict__ part3) {
  __shared__ double red[4][3][32];
  __shared__ NearQueue nq[4];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  NearQueue& Q = nq[w];
  const unsigned lt_mask = (1u << lane) - 1u;
  const int hs = (h + 2) * 3, cst = (h + 1) * 3;
  // warp task = (owned item oi, source group grp of G), as poro_p2p_kernel
  for (int task = blockIdx.x * 4 + w; task < nown * G; task += gridDim.x * 4) {
    const int oi = task / G, grp = task - oi * G;
    const int it = order[oi];
    const int4 item = items[it];
    const int kk = item.x;
    const int c = leaves[kk];
    const int nt = min(kTgtGroup, c_start[c] + c_count[c] - item.y);
    const int S = 32 / nt;
    const int tl = lane % nt, slice = lane / nt;
    const bool active = slice < S;
    const int ti = item.y + tl;
    const double2 zt = make_double2(ex[ti], ey[ti]);
    const double ctg = ec[ti], stg = es[ti];
    const double2 e2t = make_double2(ctg * ctg - stg * stg, 2.0 * ctg * stg);
    for (int e = lane; e < 3 * kTgtGroup; e += 32) (&Q.acc[0][0])[e] = 0.0;
    int qn = 0;
    double os = 0.0, on = 0.0, op = 0.0;
    auto desc = [&](int qi) {
      const int tg = item.y + Q.t[qi], sidx = Q.s[qi], j = Q.j[qi];
      const double cq = ec[tg], sq = es[tg];
      const double* sp = src + (int64_t)sidx * kPoroStride;
      const double* Da = Hs + (int64_t)sidx * hs + (h + 2 - j) * 3;   // D^(h+1-j)
      const double* Db = Da - 3;                                       // D^(h-j)
      NearDesc d;
      d.zt = make_double2(ex[tg], ey[tg]);
      d.e2t = make_double2(cq * cq - sq * sq, 2.0 * cq * sq);
      d.zc = make_double2(sp[0], sp[1]);
      d.e = make_double2(sp[2], sp[3]);
      d.a = sp[4];
      d.Ds = Da[0] - Db[0];
      d.Dn = Da[1] - Db[1];
      d.q = -(Da[2] - Db[2]);   // J: q_formula = -q_ABI
      d.ct = k.c * (j * dt);
      return d;
    };
    auto flush = [&]() {
      near_queue_flush(Q, qn, lane, k, desc, AccSink{&Q});
      qn = 0;
    };
    int pos = 0;
    for (int r = u_off[kk], rend = u_off[kk + 1]; r < rend && pos < item.w; ++r) {
      const int lo = u_lo[r], len = u_hi[r] - lo;
      const int b = max(item.z - pos, 0), e_ = min(item.w - pos, len);
      for (int jb = b; jb < e_; jb += S) {
        if (G > 1 && ((pos + jb - item.z) / S) % G != grp) continue;   // another warp's round
        const int jj = jb + slice;
        const bool valid = active && jj < e_;
        const int sidx = lo + (valid ? jj : 0);
        int j0 = 0;
        if (valid) {
          const double* sp = src + (int64_t)sidx * kPoroStride;
          const double2 zc = make_double2(sp[0], sp[1]);
          const double2 e = make_double2(sp[2], sp[3]);
          const double a = sp[4];
          const double* H = Hs + (int64_t)sidx * hs;
          const double* C = Cs + (int64_t)sidx * cst;
          // distance of the target to the segment (as poro_element)
          const double rx = zt.x - zc.x, ry = zt.y - zc.y;
          const double sstar = rx * e.x + ry * e.y;
          const double dperp = fabs(-rx * e.y + ry * e.x);
          const double dist = (fabs(sstar) <= a) ? dperp : hypot(dperp, fabs(sstar) - a);
          const double d2 = dist * dist;
          // j0 = number of leading far-form lags (monotone in j; same test as poro_element)
          auto is_far = [&](int j) { return d2 / (4.0 * (k.c * (j * dt))) > kUFar; };
          j0 = (int)fmin((double)(h + 1), floor(d2 / (4.0 * kUFar * k.c * dt)));
          j0 = max(j0, 0);
          while (j0 < h + 1 && is_far(j0 + 1)) ++j0;
          while (j0 > 0 && !is_far(j0)) --j0;
          if (j0 > 0) {
            // S0 = -D^(h-j0) (k' = h-j0+1), S1 = C[h] - C[h+1-j0] - j0 D^(h-j0)
            const double* Dj = H + (h - j0 + 1) * 3;
            const double* Ch = C + h * 3;
            const double* Cl = C + (h + 1 - j0) * 3;
            const double s0s = -Dj[0], s0n = -Dj[1];
            const double s1s = Ch[0] - Cl[0] - j0 * Dj[0];
            const double s1n = Ch[1] - Cl[1] - j0 * Dj[1];
            const double s1q = Ch[2] - Cl[2] - j0 * Dj[2];
            double2 T;
            double p;
            poro_far_split(zt, zc, e, a, s0s, s0n, s1s, s1n, -s1q, dt, k, e2t, T, p);
            os += T.y;
            on += T.x;
            op -= p;   // J: p_ABI = -p_formula
          }
        }
        // near-rule lags j0+1 .. h+1 of this pair -> queue
        int jn = j0 + 1, rem = valid ? h + 1 - j0 : 0;
        for (;;) {
          const bool has = rem > 0;
          const unsigned m = __ballot_sync(0xffffffffu, has);
          if (!m) break;
          if (has) {
            const int idx = qn + __popc(m & lt_mask);
            Q.t[idx] = tl;
            Q.s[idx] = sidx;
            Q.j[idx] = jn;
            ++jn;
            --rem;
          }
          qn += __popc(m);
          if (qn >= 32) flush();
        }
      }
      pos += len;
    }
    flush();
    if (active) {
      red[w][0][lane] = os;
      red[w][1][lane] = on;
      red[w][2][lane] = op;
    }
    __syncwarp();
    if (lane < kTgtGroup) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      if (lane < nt) {
        for (int q = 0; q < S; ++q) {
          s0 += red[w][0][lane + q * nt];
          s1 += red[w][1][lane + q * nt];
          s2 += red[w][2][lane + q * nt];
        }
        s0 += Q.acc[0][lane];
        s1 += Q.acc[1][lane];
        s2 += Q.acc[2][lane];
      }
      double* o = G > 1 ? gpart + (((int64_t)grp * nown + oi) * kTgtGroup + lane) * 3
                        : part3 + ((int64_t)it * kTgtGroup + lane) * 3;
      o[0] = s0;
      o[1] = s1;
      o[2] = s2;
    }
    __syncwarp();
  }
}

// Self blocks of the poroelastic influence (block-Jacobi preconditioner):
// blk[i][r][c] = (sigma_s, sigma_n, p)_r at element i from a unit ABI
// component c (D_s, D_n, q) on element i (sorted order).
__global__ void poro_self_blocks(int64_t n, const double* __restrict__ ex,
                                 const double* __restrict__ ey, const double* __restrict__ ea,
                                 const double* __restrict__ ec, const double* __restrict__ es,
                                 PoroConst k, double* __restrict__ blk) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 zt = make_double2(ex[i], ey[i]);
  const double ct = ec[i], st = es[i];
  const double2 e2t = make_double2(ct * ct - st * st, 2.0 * ct * st);
  for (int col = 0; col < 3; ++col) {
    const double sp[kPoroStride] = {ex[i], ey[i], ct, st, ea[i], col == 0 ? 1.0 : 0.0,
                                    col == 1 ? 1.0 : 0.0, col == 2 ? 1.0 : 0.0};
    double os = 0.0, on = 0.0, op = 0.0;
    poro_pair(zt, e2t, sp, k, os, on, op);
    blk[i * 9 + 0 * 3 + col] = os;
    blk[i * 9 + 1 * 3 + col] = on;
    blk[i * 9 + 2 * 3 + col] = op;
  }
}

// dense diagonal blocks of the leaf-block Jacobi preconditioner (gmres.cu):
// CTA per chunk of <= kPcChunk consecutive sorted elements; entry
// (3 i + r, 3 j + c) = response r at element e0+i to a unit component c on
// element e0+j (the exact direct-mode pair kernel)
__global__ void poro_chunk_blocks(const int2* __restrict__ chunks, const int64_t* __restrict__ off,
                                  const double* __restrict__ ex, const double* __restrict__ ey,
                                  const double* __restrict__ ea, const double* __restrict__ ec,
                                  const double* __restrict__ es, PoroConst k,
                                  double* __restrict__ blk) {
  const int2 ch = chunks[blockIdx.x];
  const int e0 = ch.x, ne = ch.y, d = 3 * ne;
  double* B = blk + off[blockIdx.x];
  for (int idx = threadIdx.x; idx < ne * ne * 3; idx += blockDim.x) {
    const int col = idx % 3, pr = idx / 3, i = e0 + pr / ne, j = e0 + pr % ne;
    const double2 zt = make_double2(ex[i], ey[i]);
    const double ct = ec[i], st = es[i];
    const double2 e2t = make_double2(ct * ct - st * st, 2.0 * ct * st);
    const double sp[kPoroStride] = {ex[j], ey[j], ec[j], es[j], ea[j], col == 0 ? 1.0 : 0.0,
                                    col == 1 ? 1.0 : 0.0, col == 2 ? 1.0 : 0.0};
    double os = 0.0, on = 0.0, op = 0.0;
    poro_pair(zt, e2t, sp, k, os, on, op);
    const int r0 = 3 * (i - e0), c0 = 3 * (j - e0) + col;
    B[(size_t)(r0 + 0) * d + c0] = os;
    B[(size_t)(r0 + 1) * d + c0] = on;
    B[(size_t)(r0 + 2) * d + c0] = op;
  }
}

}  // namespace

static PoroConst to_const(const PoroParams& P) {
  PoroConst k;
  k.G = P.G; k.C = P.C; k.eta = P.eta; k.kp = P.kp; k.S = P.S; k.kappa = P.kappa; k.c = P.c;
  k.ct = P.ct; k.gc = P.G * P.C;
  return k;
}

int launch_poro_chunk_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, int nchunks,
                             const int2* chunks, const int64_t* off, double* blk, cudaStream_t s) {
  if (nchunks <= 0) return DDM_OK;
  poro_chunk_blocks<<<nchunks, 128, 0, s>>>(chunks, off, t->ex, t->ey, t->ea, t->ec, t->es,
                                            to_const(P), blk);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

PoroParams poro_params(const ddm_material* m, double tau) {
  PoroParams P;
  const double G = m->G, nu = m->nu, nuu = m->nu_u, al = m->alpha;
  const double M = 2 * G * (nuu - nu) / (al * al * (1 - 2 * nuu) * (1 - 2 * nu));
  P.S = al * al * (1 - 2 * nu) / (2 * G * (1 - nu)) + 1.0 / M;
  P.c = m->kappa / P.S;
  P.eta = al * (1 - 2 * nu) / (2 * (1 - nu));
  P.kp = al * (1 - 2 * nu) / (2 * G * P.S);
  P.kappa = m->kappa;
  P.G = G;
  P.C = 1.0 / (4.0 * M_PI * (1.0 - nu));
  P.ct = P.c * tau;
  return P;
}

int poro_init_tables(ddm_ctx_s* ctx) {
  // 8-point Gauss–Legendre nodes/weights on [-1, 1] by Newton on P_8
  double x[8], wts[8];
  const int n = 8;
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        const double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      const double z1 = z;
      z = z1 - p1 / pp;
      if (fabs(z - z1) < 1e-16) break;
    }
    x[i] = z;
    wts[i] = 2.0 / ((1.0 - z * z) * pp * pp);
  }
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_gl_x, x, sizeof(x)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_gl_w, wts, sizeof(wts)));
  double f2[kNSeries] = {}, g2[kNSeries] = {}, h2[8] = {};
  double fact = 1.0;                       // k!
  for (int k = 1; k <= kNSeries + 1; ++k) {
    fact *= k;
    const double sgn = (k & 1) ? -1.0 : 1.0;
    if (k >= 2 && k - 1 < kNSeries) f2[k - 1] = sgn * (k - 1) / fact;
    if (k - 1 < kNSeries) g2[k - 1] = sgn * (1 - 2 * k) / (4.0 * fact * (k + 1));
  }
  fact = 1.0;
  for (int k = 0; k < 8; ++k) {
    fact *= (k + 1);                       // (k+1)!
    h2[k] = ((k & 1) ? -1.0 : 1.0) / fact;
  }
  {
    // E1 tables: Ein series coefficients and per-octave Chebyshev series of
    // h(u) = u e^u E1(u), evaluated in long double by the backward continued
    // fraction E1(u) e^u = 1/(u+1- 1/(u+3- 4/(u+5- ...)))
    double ein[kEinTerms];
    long double kf = 1.0L;
    for (int k = 1; k <= kEinTerms; ++k) {
      kf *= k;
      ein[k - 1] = (double)(((k & 1) ? 1.0L : -1.0L) / (k * kf));
    }
    auto h_ld = [](long double u) {
      const int M = 4000;
      long double f = u + 2.0L * M + 1.0L;
      for (int k = M; k >= 1; --k) f = u + 2.0L * k - 1.0L - (long double)k * k / f;
      return u / f;
    };
    std::vector<double> cheb(kE1Oct * kE1Cheb);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < kE1Oct; ++j) {
      const long double a = ldexpl(2.0L, j), b = 2.0L * a;
      const long double mid = 0.5L * (a + b), half = 0.5L * (b - a);
      long double hv[kE1Cheb];
      for (int i = 0; i < kE1Cheb; ++i)
        hv[i] = h_ld(mid + half * cosl(pi * (i + 0.5L) / kE1Cheb));
      for (int k = 0; k < kE1Cheb; ++k) {
        long double sum = 0.0L;
        for (int i = 0; i < kE1Cheb; ++i) sum += hv[i] * cosl(pi * k * (i + 0.5L) / kE1Cheb);
        cheb[j * kE1Cheb + k] = (double)(sum * 2.0L / kE1Cheb / (k == 0 ? 2.0L : 1.0L));
      }
    }
    DDM_CUDA(ctx, cudaMemcpyToSymbol(g_ein, ein, sizeof(ein)));
    DDM_CUDA(ctx, cudaMemcpyToSymbol(g_e1cheb, cheb.data(), cheb.size() * sizeof(double)));
  }
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_f2, f2, sizeof(f2)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_g2, g2, sizeof(g2)));
  DDM_CUDA(ctx, cudaMemcpyToSymbol(c_h2, h2, sizeof(h2)));
  return DDM_OK;
}


int launch_poro_prep(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D,
                     cudaStream_t s) {
  poro_prep<<<nblk(t->n, 256), 256, 0, s>>>(t->n, perm_in, D, t->ex, t->ey, t->ea, t->ec, t->es,
                                             t->src, perm_in ? t->d_sorted : nullptr);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

static void const_key(const PoroConst& k, double* key) {
  const double v[9] = {k.G, k.C, k.eta, k.kp, k.S, k.kappa, k.c, k.ct, k.gc};
  for (int i = 0; i < 9; ++i) key[i] = v[i];
}
static bool key_eq(const double* a, const double* b) {
  return std::memcmp(a, b, 9 * sizeof(double)) == 0;
}

// Block offsets of the owned P2P items (window length x kTgtGroup x 9
// doubles each), shared by the near-field cache and the history lag cache.
static int item_block_offsets(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) {
  if (t->nc_off) return DDM_OK;
  const int nown = t->item_hi_owned - t->item_lo_owned;
  std::vector<int4> it((size_t)nown);
  DDM_CUDA(ctx, cudaMemcpyAsync(it.data(), t->items + t->item_lo_owned, nown * sizeof(int4),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  std::vector<int64_t> off((size_t)nown);
  int64_t tot = 0;
  for (int i = 0; i < nown; ++i) {
    off[i] = tot;
    tot += (int64_t)(it[i].w - it[i].z) * kTgtGroup * 9;
  }
  int rc;
  if ((rc = dalloc(ctx, &t->nc_off, (size_t)nown))) return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->nc_off, off.data(), nown * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  t->nc_n = tot;
  return DDM_OK;
}

// Near-field cache bookkeeping, called by fmm_matvec before any graph capture:
// the blocks for these parameters are built on the second consecutive
// poroelastic FMM matvec with them (a single matvec never pays the build),
// if they fit in half the free device memory (DDM_NEAR_CACHE=0 disables).
int poro_near_cache_update(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, cudaStream_t s) {
  static const bool off = [] {
    const char* e = getenv("DDM_NEAR_CACHE");
    return e && e[0] == '0';
  }();
  const int nown = t->item_hi_owned - t->item_lo_owned;
  if (off || nown <= 0) return DDM_OK;
  const PoroConst k = to_const(P);
  double key[9];
  const_key(k, key);
  if (t->nc_valid && key_eq(key, t->nc_key)) return DDM_OK;
  const bool repeat = t->nc_seen_set && key_eq(key, t->nc_seen);
  std::memcpy(t->nc_seen, key, sizeof(key));
  t->nc_seen_set = true;
  if (!repeat) return DDM_OK;
  int rc;
  if ((rc = item_block_offsets(ctx, t, s))) return rc;
  if (!t->nc) {
    size_t fr = 0, total = 0;
    DDM_CUDA(ctx, cudaMemGetInfo(&fr, &total));
    if ((size_t)t->nc_n * sizeof(double) > fr / 2) return DDM_OK;   // does not fit: on the fly
    if ((rc = dalloc(ctx, &t->nc, (size_t)t->nc_n))) return rc;
  }
  t->nc_valid = false;
  // graphs captured against the previous blocks (another elapsed time) would
  // replay the apply kernel on the blocks rebuilt here
  drop_graphs(t);
  poro_near_build_kernel<<<nblk((int64_t)nown * kBuildGroups, 4), 128, 0, s>>>(
      nown, t->p2p_order, t->items, t->item_lo_owned, t->u_off, t->u_lo, t->u_hi, t->leaves,
      t->c_start, t->c_count, t->ex, t->ey, t->ea, t->ec, t->es, k, 1, 1, 0, t->nc_off, t->nc);
  DDM_CUDA(ctx, cudaGetLastError());
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  std::memcpy(t->nc_key, key, sizeof(key));
  t->nc_valid = true;
  return DDM_OK;
}

// per-tree buffer of the per-group partials of the on-the-fly near-field
// kernels (grown with cudaMalloc; a first-use cudaMallocAsync pool growth
// cost ~20 ms)
static int group_partials(ddm_ctx_s* ctx, ddm_tree_s* t, size_t doubles, double** out) {
  if (t->gpart_n < (int64_t)doubles) {
    drop_graphs(t);   // captured on-the-fly graphs hold the old buffer
    if (t->gpart) cudaFree(t->gpart);
    t->gpart = nullptr;
    t->gpart_n = 0;
    int rc;
    if ((rc = dalloc(ctx, &t->gpart, doubles))) return rc;
    t->gpart_n = (int64_t)doubles;
  }
  *out = t->gpart;
  return DDM_OK;
}

int launch_poro_p2p(ddm_ctx_s* ctx, ddm_tree_s* t, int item_lo, int item_hi, const PoroParams& P,
                    cudaStream_t s) {
  if (item_hi <= item_lo) return DDM_OK;
  const PoroConst k = to_const(P);
  double key[9];
  const_key(k, key);
  if (t->nc_valid && key_eq(key, t->nc_key) && item_lo == t->item_lo_owned &&
      item_hi == t->item_hi_owned) {
    poro_near_apply_kernel<<<item_hi - item_lo, kApplyWarps * 32, 0, s>>>(
        t->p2p_order, t->items, t->item_lo_owned, t->u_off, t->u_lo, t->u_hi,
        t->leaves, t->c_start, t->c_count, t->src, t->nc_off, t->nc,
        reinterpret_cast<double*>(t->part));
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }
  // source groups per item (the near-rule work of an item is large and
  // uneven; one warp per item left 181 warps for config 4's 181 items)
  const int nown = item_hi - item_lo;
  static const int g_env = [] {
    const char* e = getenv("DDM_PORO_GROUPS");
    return e ? atoi(e) : 0;
  }();
  // measured (DDM_NEAR_CACHE=0): config 4 0.59 -> 0.15 ms, config 3 0.93 -> 0.81 ms at G = 8
  const int G = g_env > 0 ? g_env : 8;
  double* gpart = nullptr;
  if (G > 1) {
    int rc;
    // sized for at least the history kernels' 8 groups, so a later history
    // call never reallocates the buffer under a captured matvec graph
    if ((rc = group_partials(ctx, t, (size_t)std::max(G, 8) * nown * kTgtGroup * 3, &gpart)))
      return rc;
  }
  poro_p2p_kernel<<<nblk((int64_t)nown * G, 4), 128, 0, s>>>(
      nown, t->p2p_order, t->items, t->u_off, t->u_lo, t->u_hi, t->leaves, t->c_start, t->c_count,
      t->src, t->ex, t->ey, t->ec, t->es, to_const(P), G, gpart, reinterpret_cast<double*>(t->part));
  DDM_CUDA(ctx, cudaGetLastError());
  if (G > 1) {
    const int64_t ne = (int64_t)nown * kTgtGroup * 3;
    poro_hist_reduce<<<nblk(ne, 256), 256, 0, s>>>(nown, G, t->p2p_order, gpart,
                                                   reinterpret_cast<double*>(t->part));
    DDM_CUDA(ctx, cudaGetLastError());
  }
  return DDM_OK;
}

// History lag cache bookkeeping (fmm_history, outside any capture): for the
// (material, dt) of a history sum requested twice in a row, the blocks of
// lags 1..h+1 are built (missing lags only, as the history grows) while the
// device keeps a quarter of its memory free; returns true when every lag the
// call needs is cached.  DDM_HIST_CACHE=0 disables.
bool poro_hist_cache_update(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                            int h, cudaStream_t s, int* rc_out) {
  *rc_out = DDM_OK;
  static const bool off = [] {
    const char* e = getenv("DDM_HIST_CACHE");
    return e && e[0] == '0';
  }();
  const int nown = t->item_hi_owned - t->item_lo_owned;
  if (off || nown <= 0 || h < 1) return false;
  double key[9];
  const_key(to_const(poro_params(mat, dt)), key);
  if (!(t->hc_valid && key_eq(key, t->hc_key))) {
    const bool repeat = t->hc_seen_set && key_eq(key, t->hc_seen);
    std::memcpy(t->hc_seen, key, sizeof(key));
    t->hc_seen_set = true;
    if (!repeat) return false;
    for (double* p : t->hc_alloc) cudaFree(p);
    t->hc_alloc.clear();
    t->hc_lag.clear();
    t->hc_nlags = 0;
    // chunk budget, fixed at creation (no memory queries while the history
    // grows): chunks that keep a quarter of the device memory free
    int rc;
    if ((rc = item_block_offsets(ctx, t, s))) {
      *rc_out = rc;
      return false;
    }
    size_t fr = 0, total = 0;
    DDM_CUDA(ctx, cudaMemGetInfo(&fr, &total));
    const size_t cbytes = (size_t)t->nc_n * kLagChunk * sizeof(double);
    t->hc_max_chunks = fr > total / 4 && cbytes > 0 ? (int)((fr - total / 4) / cbytes) : 0;
    // DDM_HIST_CHUNKS=k caps the budget at k chunks (tests of the fallback;
    // read whenever a cache is keyed, so a test can change it in-process)
    const char* cap_env = getenv("DDM_HIST_CHUNKS");
    if (cap_env && cap_env[0]) t->hc_max_chunks = std::min(t->hc_max_chunks, atoi(cap_env));
    std::memcpy(t->hc_key, key, sizeof(key));
    t->hc_valid = true;
    t->hc_capped = false;
  }
  if (t->hc_nlags < h + 1 && !t->hc_capped) {
    int rc;
    while (t->hc_nlags < h + 1) {
      const int j = t->hc_nlags + 1;
      const int ci = (j - 1) / kLagChunk;
      if (ci == (int)t->hc_lag.size()) {
        if (ci >= t->hc_max_chunks) {   // memory budget reached: on the fly from here on
          t->hc_capped = true;
          break;
        }
        // plain cudaMalloc (~4 ms at any size; growing the stream-ordered
        // pool by a chunk stalled the host for 10-800 ms, scripts/micro/alloc.cu),
        // as many chunks as already exist (doubling: O(log) allocations)
        const int k = std::min(std::max(1, (int)t->hc_lag.size()), t->hc_max_chunks - ci);
        double* blk = nullptr;
        if (dalloc(ctx, &blk, (size_t)t->nc_n * kLagChunk * k)) {
          // out of memory while growing: keep the lags built so far and
          // evaluate this and later history sums on the fly (not an error)
          ctx->err.clear();
          t->hc_capped = true;
          break;
        }
        t->hc_alloc.push_back(blk);
        for (int q = 0; q < k; ++q) t->hc_lag.push_back(blk + (size_t)q * t->nc_n * kLagChunk);
      }
      poro_near_build_kernel<<<nblk((int64_t)nown * kBuildGroups, 4), 128, 0, s>>>(
          nown, t->p2p_order, t->items, t->item_lo_owned, t->u_off, t->u_lo, t->u_hi, t->leaves,
          t->c_start, t->c_count, t->ex, t->ey, t->ea, t->ec, t->es,
          to_const(poro_params(mat, j * dt)), 0, kLagChunk, (j - 1) % kLagChunk, t->nc_off,
          t->hc_lag[ci]);
      DDM_CUDA(ctx, cudaGetLastError());
      t->hc_nlags = j;
    }
    if (t->hc_ptrs_n < (int)t->hc_lag.size()) {
      if (t->hc_ptrs) cudaFree(t->hc_ptrs);
      t->hc_ptrs = nullptr;
      t->hc_ptrs_n = 0;
      const int cap = std::max(2 * (int)t->hc_lag.size(), 64);
      if (dalloc(ctx, &t->hc_ptrs, (size_t)cap)) {
        ctx->err.clear();
        t->hc_capped = true;
        return false;
      }
      t->hc_ptrs_n = cap;
    }
    DDM_CUDA(ctx, cudaMemcpyAsync(t->hc_ptrs, t->hc_lag.data(), t->hc_lag.size() * sizeof(double*),
                                  cudaMemcpyHostToDevice, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
  }
  return t->hc_nlags >= h + 1;
}

int launch_poro_hist_cached(ddm_ctx_s* ctx, ddm_tree_s* t, int h, const double* Hs,
                            cudaStream_t s) {
  const int nown = t->item_hi_owned - t->item_lo_owned;
  if (nown <= 0) return DDM_OK;
  const int nch = (h + 1 + kLagChunk - 1) / kLagChunk;
  double* hpart = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&hpart, (size_t)nch * nown * kTgtGroup * 3 * sizeof(double),
                                s));
  poro_hist_cached_kernel<<<dim3(nown, nch), kHistWarps * 32, 0, s>>>(
      t->p2p_order, t->items, t->item_lo_owned, nown, t->u_off, t->u_lo, t->u_hi, t->leaves,
      t->c_start, t->c_count, Hs, h, t->nc_off, t->hc_ptrs, hpart);
  DDM_CUDA(ctx, cudaGetLastError());
  const int64_t ne = (int64_t)nown * kTgtGroup * 3;
  poro_hist_reduce<<<nblk(ne, 256), 256, 0, s>>>(nown, nch, t->p2p_order, hpart,
                                                 reinterpret_cast<double*>(t->part));
  DDM_CUDA(ctx, cudaGetLastError());
  cudaFreeAsync(hpart, s);
  return DDM_OK;
}

int launch_poro_direct(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi,
                       const PoroParams& P, double* y_user, double* y_sorted, cudaStream_t s) {
  if (hi <= lo) return DDM_OK;
  poro_direct_kernel<<<nblk(hi - lo, 64), 64, 0, s>>>(t->n, lo, hi, t->src, t->ex, t->ey, t->ec,
                                                      t->es, to_const(P), t->perm, y_user,
                                                      y_sorted);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_poro_hist_gather(ddm_ctx_s* ctx, ddm_tree_s* t, int h, const double* D_hist,
                            double* Hs, double* Cs, double* Ctot, cudaStream_t s) {
  hist_gather<<<nblk(t->n * 3, 256), 256, 0, s>>>(t->n, h, t->perm, D_hist, Hs, Cs, Ctot);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_poro_hist_near(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, int h, double dt,
                          const double* Hs, const double* Cs, cudaStream_t s) {
  const int nown = t->item_hi_owned - t->item_lo_owned;
  if (nown <= 0) return DDM_OK;
  constexpr int G = 8;   // source groups per item (as launch_poro_p2p)
  double* gpart = nullptr;
  {
    int rc;
    if ((rc = group_partials(ctx, t, (size_t)G * nown * kTgtGroup * 3, &gpart))) return rc;
  }
  poro_hist_near_kernel<<<nblk((int64_t)nown * G, 4), 128, 0, s>>>(
      nown, t->p2p_order, t->items, t->u_off, t->u_lo, t->u_hi, t->leaves, t->c_start,
      t->c_count, t->src, Hs, Cs, h, dt, t->ex, t->ey, t->ec, t->es, to_const(P), G, gpart,
      reinterpret_cast<double*>(t->part));
  DDM_CUDA(ctx, cudaGetLastError());
  const int64_t ne = (int64_t)nown * kTgtGroup * 3;
  poro_hist_reduce<<<nblk(ne, 256), 256, 0, s>>>(nown, G, t->p2p_order, gpart,
                                                 reinterpret_cast<double*>(t->part));
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int launch_poro_self_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, double* blk,
                            cudaStream_t s) {
  poro_self_blocks<<<nblk(t->n, 64), 64, 0, s>>>(t->n, t->ex, t->ey, t->ea, t->ec, t->es,
                                                 to_const(P), blk);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

}  // namespace ddm
