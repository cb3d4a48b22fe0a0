"""ORACLE (test infrastructure only) — fully coupled poroelastic kernel.

What it computes: the continuous-source influence of a constant element
carrying (D_s, D_n, q) (shear DD, normal DD, fluid-source rate per unit length)
switched on at elapsed time 0 and held, on the traction (sigma_s, sigma_n) and
pore pressure p at a target element centre, elapsed time tau later — the
coefficients A_xx .. A_pq of Eq.(final_sigs)-(final_pp), time
integrated over "continuous impulses".  The paper prints none of
these kernels (it cites Carvalho 1991 / Cleary 1977); the
derivation below (DESIGN.md §2 R17) is from Biot /
Rice–Cleary theory, plane strain, tension-positive stress, CS-convention DDs,
physical pore pressure:

  constants  M = 2G(nu_u-nu)/(alpha^2 (1-2nu_u)(1-2nu)),
             S = alpha^2 (1-2nu)/(2G(1-nu)) + 1/M,  c = kappa/S,
             eta = alpha (1-2nu)/(2(1-nu)),  k_p = alpha (1-2nu)/(2 G S)
  split      u = u^D + (eta/G) grad Phi,  lap Phi = p,
             sigma = sigma^D(nu) + 2 eta (Phi_,ij - p delta_ij)
  pressure   p(0+) = -(alpha/S) eps^D_kk,reg -> diffuses with c for tau > 0.
             For a point DD: order-2 part p2 = Re(K/w^2) F(u) plus, for the
             normal DD, a monopole mu e^-u/(4 pi c tau), mu = -(eta/S) D_n,
             K = -4 k_p i G C B e, B = (D_s + i D_n) e, u = |w|^2/(4 c tau),
             F(u) = 1 - (1+u) e^-u.  Fluid source: Theis q E1(u)/(4 pi kappa).
  potential  d^2 Phi/dw^2 (order 2) = K conj(w)^... written with
             omega = w/|w|:  K omegab^4 g2(u)/(4 c tau)
                             - e^-u Re(K omegab^2) omegab^2/(16 c tau)
             monopole:  -mu f2(u) omegab^2 / (16 pi c tau)
             fluid:     -q h2(u) omegab^2 / (16 pi kappa)
             f2 = F/u, g2 = (-1/4 - e^-u/2 + 3(1-e^-u)/(4u))/u, h2 = (1-e^-u)/u
             (stable series for small u).
  traction   T = sigma_n + i sigma_s = (sigma_kk)/2 + e^{2i b_t}(sigma_yy - sigma_xx + 2i sigma_xy)/2
             sigma^p part: T^p = -eta p + e^{2 i b_t} (-4 eta d^2Phi/dw^2)
The element influence = drained Crouch–Starfield (oracle/elastic.py, nu) +
integral along the element of (T^p, p) by the fixed composite Gauss–Legendre
rule of DESIGN.md R17, §4.5 (8 nodes per panel, panels graded away from the nearest point, each <= max(r, sqrt(c tau))/4,
split at the foot of the perpendicular when the target lies on the element,
where the log singularity of E1 is integrated analytically).  Beyond
u_min = dist^2/(4 c tau) > 40 the transient terms are below 1e-17 and the
far form is integrated analytically.

ABI mapping (R2): DDs opening-positive and stresses
compression-positive flip together, the pressure and the fluid source keep
their physical sign, hence A_ABI = J A J with J = diag(1, 1, -1).

Pins (tests/test_oracle_poro.py): tau -> 0+ gives Crouch–Starfield with nu_u
(undrained, full tensor) and Skempton's pore pressure; tau -> inf gives
Crouch–Starfield with nu and p -> 0; the fluid source reduces to Theis; every
pressure field satisfies the diffusion equation (finite differences); the
stresses are in equilibrium; alpha -> 0 decouples; the element rule agrees
with adaptive quadrature and with the analytic far form where they overlap.
"""
from __future__ import annotations

import math

import numpy as np
from scipy import special

from . import elastic as E

GL_NODES, GL_WEIGHTS = np.polynomial.legendre.leggauss(8)
U_FAR = 40.0
PANEL_FRACTION = 0.25


def constants(G, nu, nu_u, alpha, kappa):
    M = 2 * G * (nu_u - nu) / (alpha ** 2 * (1 - 2 * nu_u) * (1 - 2 * nu))
    S = alpha ** 2 * (1 - 2 * nu) / (2 * G * (1 - nu)) + 1.0 / M
    c = kappa / S
    eta = alpha * (1 - 2 * nu) / (2 * (1 - nu))
    kp = alpha * (1 - 2 * nu) / (2 * G * S)
    B_sk = 3 * (nu_u - nu) / (alpha * (1 - 2 * nu) * (1 + nu_u))
    return dict(M=M, S=S, c=c, eta=eta, kp=kp, kappa=kappa, B_sk=B_sk, G=G, nu=nu, nu_u=nu_u,
                alpha=alpha, C=1.0 / (4 * np.pi * (1 - nu)))


def _series(u, coef):
    out = np.zeros_like(u)
    for cf in reversed(coef):
        out = out * u + cf
    return out


# power-series coefficients (in u) of f2 = F/u, g2 = g1/u, h2 = (1-e^-u)/u
_NS = 24
_F2 = [0.0] + [((-1) ** k) * (k - 1) / math.factorial(k) for k in range(2, _NS + 2)]  # u^(k-1)
_G2 = [((-1) ** k) * (1 - 2 * k) / (4 * math.factorial(k + 1)) for k in range(1, _NS + 1)]   # u^(k-1)
_H2 = [((-1) ** k) / math.factorial(k + 1) for k in range(0, _NS)]                     # u^k


def f2(u):
    u = np.asarray(u, dtype=np.float64)
    small = u < 1.0
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        direct = (1.0 - (1.0 + u) * np.exp(-u)) / u
    return np.where(small, _series(u, _F2), direct)


def g2(u):
    u = np.asarray(u, dtype=np.float64)
    small = u < 1.0
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        e = np.exp(-u)
        direct = (-0.25 - 0.5 * e + 0.75 * (-np.expm1(-u)) / u) / u
    return np.where(small, _series(u, _G2), direct)


def h2(u):
    u = np.asarray(u, dtype=np.float64)
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        direct = -np.expm1(-u) / u
    return np.where(u < 1e-3, _series(u, _H2), direct)


def point_kernel(w, tau, k, e, Ds, Dn, q):
    """sigma^p traction pieces and pressure at offsets w (complex array) from a
    unit-length point source carrying (Ds, Dn, q) with direction e.  Returns
    (p, d2Phi) so that T^p = -eta p + e^{2 i b_t} (-4 eta d2Phi)."""
    c = k["c"]
    ct = c * tau
    r2 = (w * np.conj(w)).real
    u = r2 / (4 * ct)
    om = w / np.sqrt(r2)
    ob2 = np.conj(om) ** 2
    B = (Ds + 1j * Dn) * e
    K = -4 * k["kp"] * 1j * k["G"] * k["C"] * B * e
    mu = -(k["eta"] / k["S"]) * Dn
    ReK = (K * ob2).real
    p = ReK * f2(u) / (4 * ct) + mu * np.exp(-u) / (4 * np.pi * ct)
    d2 = K * ob2 * ob2 * g2(u) / (4 * ct) - np.exp(-u) * ReK * ob2 / (16 * ct)
    d2 = d2 - mu * f2(u) * ob2 / (16 * np.pi * ct)
    if np.any(q != 0):
        p = p + q * special.exp1(u) / (4 * np.pi * k["kappa"])
        d2 = d2 - q * h2(u) * ob2 / (16 * np.pi * k["kappa"])
    return p, d2


def _far_element(z, zc, e, a, tau, k, Ds, Dn, q):
    """Analytic far form (u > U_FAR over the element) of the sigma^p traction
    pieces and p: Phi^p = 2 eta k_p Phi^D, Psi^p = 2 eta k_p (2 i G C B Ibar3)
    + (eta mu/pi + eta q c tau/(pi kappa)) ebar I2 + 48 eta k_p c tau i G C B I4,
    p = -k_p 4 Re Phi^D.  Returns (Phi, dPhi, Psi, p)."""
    z1 = zc - a * e
    z2 = zc + a * e
    r = np.conj(e) ** 2
    I2 = 1 / (z - z2) - 1 / (z - z1)
    I3 = 0.5 * (1 / (z - z2) ** 2 - 1 / (z - z1) ** 2)
    I4 = (1 / (z - z2) ** 3 - 1 / (z - z1) ** 3) / 3
    I3b = (np.conj(zc) + r * (z - zc)) * I3 - r * I2
    B = (Ds + 1j * Dn) * e
    iGC = 1j * k["G"] * k["C"]
    ekp = 2 * k["eta"] * k["kp"]
    mu = -(k["eta"] / k["S"]) * Dn
    ct = k["c"] * tau
    PhiD = iGC * B * I2
    Phi = ekp * PhiD
    dPhi = ekp * (-2 * iGC * B * I3)
    Psi = (ekp * 2 * iGC * B * I3b + (k["eta"] * mu / np.pi + k["eta"] * q * ct / (np.pi * k["kappa"]))
           * np.conj(e) * I2 + 48 * k["eta"] * k["kp"] * ct * iGC * B * I4)
    p = -k["kp"] * 4 * PhiD.real
    return Phi, dPhi, Psi, p


def _e1_line_integral(s0, s1, cscale):
    """Integral of E1(s^2/(4 c tau)) ds over [s0, s1] with 0 <= s0 < s1, where
    the log singularity at s = 0 is removed analytically:
    E1(u) = -gamma - ln u + Ein(u), Ein smooth."""
    # analytic part: int (-gamma - ln(s^2/(4ct))) ds
    def prim(s):
        if s == 0.0:
            return 0.0
        return -np.euler_gamma * s - (2 * (s * np.log(s) - s) - s * np.log(4 * cscale))
    return prim(s1) - prim(s0)


def _graded_edges(s0, s1, sfrom, sstar, dperp, lt):
    """Panel edges on [s0, s1] graded away from the nearest point sfrom: each
    panel is at most half of max(distance of its near end to the target,
    sqrt(c tau)) times PANEL_FRACTION long (R17, §4.5)."""
    pts = [sfrom]
    s = sfrom
    other = s1 if sfrom == s0 else s0
    sign = 1.0 if other > sfrom else -1.0
    while (other - s) * sign > 0:
        r = math.hypot(dperp, s - sstar)
        step = PANEL_FRACTION * max(r, lt)
        s = s + sign * step
        if (other - s) * sign <= 0:
            s = other
        pts.append(s)
        if len(pts) > 4097:
            raise RuntimeError("element rule: too many panels")
    pts = np.array(pts)
    return pts if sign > 0 else pts[::-1]


def element_integral(zt, zc, e, a, tau, k, Ds, Dn, q):
    """sigma^p traction pieces and p at target zt from the element (zc, e, a)
    by the fixed rule.  Returns (Tp_kk2 = -eta p ..., pieces) as (p, d2) totals."""
    ct = k["c"] * tau
    lt = math.sqrt(ct)
    L = 2 * a
    rel = (zt - zc) * np.conj(e)
    sstar, dperp = rel.real, abs(rel.imag)
    if abs(sstar) <= a:
        dist = dperp
    else:
        dist = math.hypot(dperp, abs(sstar) - a)
    if dist * dist / (4 * ct) > U_FAR:
        Phi, dPhi, Psi, p = _far_element(zt, zc, e, a, tau, k, Ds, Dn, q)
        return ("far", Phi, dPhi, Psi, p)
    on_line = dperp == 0.0 and abs(sstar) < a
    s0c = min(max(sstar, -a), a)          # nearest point of the segment
    p_tot = 0.0
    d2_tot = 0.0 + 0.0j
    for s0, s1 in ((-a, s0c), (s0c, a)):
        if s1 <= s0:
            continue
        edges = _graded_edges(s0, s1, s0c, sstar, dperp, lt)
        mid = 0.5 * (edges[:-1] + edges[1:])
        half = 0.5 * (edges[1:] - edges[:-1])
        s = (mid[:, None] + half[:, None] * GL_NODES[None, :]).ravel()
        wq = (half[:, None] * GL_WEIGHTS[None, :]).ravel()
        w = zt - (zc + s * e)
        if on_line and q != 0.0:
            p, d2 = point_kernel(w, tau, k, e, Ds, Dn, 0.0)
            # fluid source: smooth part by the rule, log part analytically
            u = (w * np.conj(w)).real / (4 * ct)
            ein = special.exp1(u) + np.euler_gamma + np.log(u)
            p = p + q * ein / (4 * np.pi * k["kappa"])
            d2 = d2 - q * h2(u) * (np.conj(w / np.abs(w)) ** 2) / (16 * np.pi * k["kappa"])
            lo, hi = s0 - sstar, s1 - sstar
            a0, a1 = (abs(hi), abs(lo)) if hi <= 0 else (lo, hi)
            logpart = _e1_line_integral(min(abs(a0), abs(a1)), max(abs(a0), abs(a1)), ct)
            p_tot += q * logpart / (4 * np.pi * k["kappa"])
        else:
            p, d2 = point_kernel(w, tau, k, e, Ds, Dn, q)
        p_tot += np.sum(wq * p)
        d2_tot += np.sum(wq * d2)
    return ("near", p_tot, d2_tot)


def influence(zt, bt, zc, bs, a, tau, k, Ds, Dn, q):
    """Traction (sigma_s, sigma_n) (tension positive) and pore pressure at the
    target from one source element with CS-convention (Ds, Dn) and fluid q."""
    e = np.exp(1j * bs)
    # drained elastic part (real-variable Crouch–Starfield)
    sxx, syy, sxy = E.global_stress(zt.real, zt.imag, zc.real, zc.imag, a, bs, Ds, Dn,
                                    k["G"], k["nu"])
    ss, sn = E.project_traction(sxx, syy, sxy, bt)
    e2 = np.exp(2j * bt)
    res = element_integral(zt, zc, e, a, tau, k, Ds, Dn, q)
    if res[0] == "far":
        _, Phi, dPhi, Psi, p = res
        T = 2 * Phi.real + e2 * (np.conj(zt) * dPhi + Psi)
    else:
        _, p, d2 = res
        T = -k["eta"] * p + e2 * (-4 * k["eta"] * d2)
    return float(ss + T.imag), float(sn + T.real), float(np.real(p))


_UNIT = ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0))
_J = np.array([1.0, 1.0, -1.0])


def row_blocks(geom, k, tau, i):
    """3x3 influence blocks of every source on target i, ABI convention:
    returns [N, 3 (rows s, n, p), 3 (cols D_s, D_n, q)].  The far sources
    (u_min > U_FAR) are evaluated in vectorised analytic form, the others one
    by one with the element rule."""
    n = geom.n
    zc = geom.xc + 1j * geom.yc
    zt = zc[i]
    bt = geom.beta[i]
    e = np.exp(1j * geom.beta)
    a = geom.half_len
    ct = k["c"] * tau
    out = np.zeros((n, 3, 3))
    # drained elastic part, vectorised
    A_ss, A_sn, A_ns, A_nn = E.influence_blocks(zt.real, zt.imag, bt, geom.xc, geom.yc, a,
                                                geom.beta, k["G"], k["nu"])
    out[:, 0, 0], out[:, 0, 1], out[:, 1, 0], out[:, 1, 1] = A_ss, A_sn, A_ns, A_nn
    # distance of the target to every element
    rel = (zt - zc) * np.conj(e)
    sstar, dperp = rel.real, np.abs(rel.imag)
    dist = np.where(np.abs(sstar) <= a, dperp, np.hypot(dperp, np.abs(sstar) - a))
    far = dist * dist / (4 * ct) > U_FAR
    e2 = np.exp(2j * bt)
    jf = np.nonzero(far)[0]
    for col, (Ds, Dn, q) in enumerate(_UNIT):
        if jf.size:
            Phi, dPhi, Psi, p = _far_element(zt, zc[jf], e[jf], a[jf], tau, k, Ds, Dn, q)
            T = 2 * Phi.real + e2 * (np.conj(zt) * dPhi + Psi)
            out[jf, 0, col] += T.imag
            out[jf, 1, col] += T.real
            out[jf, 2, col] += p
        for j in np.nonzero(~far)[0]:
            res = element_integral(zt, zc[j], e[j], a[j], tau, k, Ds, Dn, q)
            _, p, d2 = res
            T = -k["eta"] * p + e2 * (-4 * k["eta"] * d2)
            out[j, 0, col] += T.imag
            out[j, 1, col] += T.real
            out[j, 2, col] += p.real if np.iscomplexobj(p) else p
    return out * _J[None, :, None] * _J[None, None, :]


def assemble_dense(geom, mat, tau):
    """Dense 3N x 3N matrix K^c(tau) at elapsed time tau, ABI convention (DOF
    3i+c, c = 0 D_s, 1 D_n, 2 q; rows sigma_s, sigma_n, p), A_ABI = J A_CS J."""
    k = constants(mat["G"], mat["nu"], mat["nu_u"], mat["alpha"], mat["kappa"])
    n = geom.n
    A = np.zeros((3 * n, 3 * n))
    for i in range(n):
        A[3 * i:3 * i + 3, :] = row_blocks(geom, k, tau, i).transpose(1, 0, 2).reshape(3, 3 * n)
    return A


def matvec_rows(geom, mat, tau, D, rows):
    """(K^c(tau) D)[rows] row by row (sampled parity at large N); D [N, 3]."""
    k = constants(mat["G"], mat["nu"], mat["nu_u"], mat["alpha"], mat["kappa"])
    out = np.zeros((len(rows), 3))
    for r, i in enumerate(rows):
        blk = row_blocks(geom, k, tau, int(i))
        out[r] = np.einsum("jrc,jc->r", blk, D)
    return out
