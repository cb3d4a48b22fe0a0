"""Pins of the poroelastic oracle (oracle/poro.py) against limits and
identities fixed by Biot theory, not against itself.  CPU only."""
import math

import numpy as np
import pytest
from scipy import integrate, special

from oracle import elastic as E
from oracle import poro as P
from synth.geometry import Geometry

from ._quad import element_integral_ts

MAT = dict(G=6e9, nu=0.2, nu_u=0.33, alpha=0.8, kappa=1e-15)     # BASELINE configs[2]
WESTERLY = dict(G=15e9, nu=0.25, nu_u=0.331, alpha=0.449, kappa=4e-19 / 1e-3)
K3 = P.constants(**MAT)
A, BS, ZC = 0.5, 0.3, 0.1 + 0.2j


def _targets():
    for ang in np.linspace(0.1, 6.0, 7):
        for r in (1.5, 3.0, 8.0):
            yield ZC + r * np.exp(1j * ang), 1.1


def test_constants_match_closed_forms():
    # c = kappa / S equals the Rice-Cleary diffusivity; Skempton B identity
    k = K3
    G, nu, nuu, al, kap = MAT["G"], MAT["nu"], MAT["nu_u"], MAT["alpha"], MAT["kappa"]
    B = k["B_sk"]
    c_rc = 2 * kap * G * (1 - nu) * (nuu - nu) / (al ** 2 * (1 - 2 * nu) ** 2 * (1 - nuu))
    assert abs(k["c"] / c_rc - 1) < 1e-14
    # undrained factor identity 1 + 2 eta k_p = (1 - nu)/(1 - nu_u)
    assert abs(1 + 2 * k["eta"] * k["kp"] - (1 - nu) / (1 - nuu)) < 1e-14
    assert abs(B - 0.61090) < 1e-5          # SURVEY App. B config-3 value


@pytest.mark.parametrize("mat", [MAT, WESTERLY])
def test_undrained_limit_is_crouch_starfield_nu_u_and_skempton(mat):
    k = P.constants(**mat)
    tau = 1e-10 * A * A / k["c"]
    for zt, bt in _targets():
        for Ds, Dn in ((1.0, 0.0), (0.0, 1.0)):
            ss, sn, p = P.influence(zt, bt, ZC, BS, A, tau, k, Ds, Dn, 0.0)
            sxx, syy, sxy = E.global_stress(zt.real, zt.imag, ZC.real, ZC.imag, A, BS, Ds, Dn,
                                            mat["G"], mat["nu_u"])
            s2, n2 = E.project_traction(sxx, syy, sxy, bt)
            sc = max(abs(s2), abs(n2))
            assert abs(ss - s2) <= 1e-9 * sc and abs(sn - n2) <= 1e-9 * sc
            pu = -(k["B_sk"] / 3) * (1 + mat["nu_u"]) * (sxx + syy)   # Skempton, tension +
            assert abs(p - pu) <= 1e-10 * abs(pu)


def test_drained_limit_is_crouch_starfield_nu():
    k = K3
    tau = 1e12 * A * A / k["c"]          # approach to drained is O(r^2 / (c tau))
    for zt, bt in _targets():
        for Ds, Dn in ((1.0, 0.0), (0.0, 1.0)):
            ss, sn, p = P.influence(zt, bt, ZC, BS, A, tau, k, Ds, Dn, 0.0)
            sxx, syy, sxy = E.global_stress(zt.real, zt.imag, ZC.real, ZC.imag, A, BS, Ds, Dn,
                                            MAT["G"], MAT["nu"])
            s2, n2 = E.project_traction(sxx, syy, sxy, bt)
            sc = max(abs(s2), abs(n2))
            assert abs(ss - s2) <= 1e-8 * sc and abs(sn - n2) <= 1e-8 * sc
            assert abs(p) <= 1e-7 * sc


def test_near_rule_continuous_with_analytic_far_form():
    zt, bt = ZC + 2.0 * np.exp(0.7j), 0.4
    e = np.exp(1j * BS)
    rel = (zt - ZC) * np.conj(e)
    dist = abs(rel.imag) if abs(rel.real) <= A else math.hypot(rel.imag, abs(rel.real) - A)
    tau = dist ** 2 / (4 * K3["c"] * 36.0)
    for Ds, Dn, q in ((1, 0, 0), (0, 1, 0), (0, 0, 1)):
        _, pn, d2 = P.element_integral(zt, ZC, e, A, tau, K3, Ds, Dn, q)
        Phi, dPhi, Psi, pf = P._far_element(zt, ZC, e, A, tau, K3, Ds, Dn, q)
        Tf = 2 * Phi.real + np.exp(2j * bt) * (np.conj(zt) * dPhi + Psi)
        Tn = -K3["eta"] * pn + np.exp(2j * bt) * (-4 * K3["eta"] * d2)
        assert abs(Tn - Tf) <= 1e-13 * abs(Tf)
        if q == 0:
            assert abs(pn - pf) <= 1e-13 * abs(pf)


def _point_field(z, tau, k, Ds, Dn, q, bt):
    p, d2 = P.point_kernel(np.array([z]), tau, k, np.exp(1j * BS), Ds, Dn, q)
    return p[0], d2[0]


def test_fluid_source_is_theis():
    # point source: p = q E1(r^2 / 4 c tau) / (4 pi kappa)
    k = K3
    tau = 50.0
    for r in (0.01, 0.05, 0.2):
        p, _ = _point_field(r + 0j, tau, k, 0.0, 0.0, 1.0, 0.0)
        theis = special.exp1(r * r / (4 * k["c"] * tau)) / (4 * np.pi * k["kappa"])
        assert abs(p / theis - 1) < 1e-14
    # decoupling alpha -> 0 at fixed M: q -> p is Theis with S = 1/M, no stresses
    G, nu = MAT["G"], MAT["nu"]
    M = K3["M"]
    alpha = 1e-4
    # choose nu_u so that M stays the same: M = 2G(nu_u-nu)/(alpha^2 (1-2nu_u)(1-2nu))
    x = M * alpha ** 2 * (1 - 2 * nu) / (2 * G)
    nuu = (nu + x) / (1 + 2 * x)                         # solves nu_u - nu = x (1 - 2 nu_u)
    kd = P.constants(G, nu, nuu, alpha, MAT["kappa"])
    assert abs(kd["M"] / M - 1) < 1e-6
    z, tau = 0.07 + 0.02j, 30.0
    p, d2 = _point_field(z, tau, kd, 0.0, 0.0, 1.0, 0.0)
    u = abs(z) ** 2 * kd["S"] / (4 * MAT["kappa"] * tau)
    assert abs(p / (special.exp1(u) / (4 * np.pi * MAT["kappa"])) - 1) < 1e-6
    # the DD -> p coupling vanishes with alpha (order alpha)
    pD, _ = _point_field(z, tau, kd, 0.0, 1.0, 0.0, 0.0)
    assert abs(pD) < 1e-3 * abs(_point_field(z, tau, K3, 0.0, 1.0, 0.0, 0.0)[0])
    # ... and so does the q -> sigma coupling: the fluid source induces no
    # stress (SURVEY §8c.3 pin 5), for the point kernel and for an element
    def tq(kk, zz):
        p, d2 = _point_field(zz, tau, kk, 0.0, 0.0, 1.0, 0.0)
        return -kk["eta"] * p + np.exp(0.6j) * (-4 * kk["eta"] * d2)
    for zz in (z, 0.3 - 0.1j, 2.0 + 1.0j):
        assert abs(tq(kd, zz)) <= 1e-3 * abs(tq(K3, zz))
    ss_d, sn_d, _ = P.influence(ZC + 0.04j, 0.6, ZC, BS, 0.02, tau, kd, 0.0, 0.0, 1.0)
    ss_c, sn_c, _ = P.influence(ZC + 0.04j, 0.6, ZC, BS, 0.02, tau, K3, 0.0, 0.0, 1.0)
    assert math.hypot(ss_d, sn_d) <= 1e-3 * math.hypot(ss_c, sn_c)


@pytest.mark.parametrize("src", [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)])
def test_pressure_satisfies_diffusion(src):
    # d p / d tau = c lap p off the source, for the element fields
    k = K3
    e = np.exp(1j * BS)
    a = 0.05
    tau = 40.0                                # sqrt(c tau) ~ 0.018 m
    ell = math.sqrt(k["c"] * tau)
    h = 0.04 * ell
    dt = 1e-3 * tau
    for zt in (ZC + 0.04j * e, ZC + 0.1 * np.exp(1j * (BS + 2.0)), ZC + (0.08 + 0.03j) * e):
        f = lambda z, t: P.element_integral(z, ZC, e, a, t, k, *src)[1].real
        # 4th-order central differences in x, y and 2nd order in tau
        lap = 0.0
        pmax = 0.0
        for d in (1.0, 1j):
            v = [f(zt + m * h * d, tau) for m in (-2, -1, 0, 1, 2)]
            pmax = max(pmax, max(abs(x) for x in v))
            lap += (-v[0] + 16 * v[1] - 30 * v[2] + 16 * v[3] - v[4]) / (12 * h * h)
        pt = (f(zt, tau + dt) - f(zt, tau - dt)) / (2 * dt)
        scale = k["c"] * pmax / ell ** 2
        assert abs(pt - k["c"] * lap) <= 1e-4 * scale     # FD truncation ~ (h/ell)^4


def _tensor(zt, tau, k, src):
    """Full tension-positive stress tensor from tractions on faces b = 0, pi/2."""
    ss0, sn0, _ = P.influence(zt, 0.0, ZC, BS, 0.05, tau, k, *src)
    ss9, sn9, _ = P.influence(zt, np.pi / 2, ZC, BS, 0.05, tau, k, *src)
    return sn9, sn0, ss0          # sxx, syy, sxy


@pytest.mark.parametrize("src", [(1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)])
def test_stress_equilibrium(src):
    k = K3
    tau = 40.0
    ell = math.sqrt(k["c"] * tau)
    h = 0.04 * ell
    e = np.exp(1j * BS)

    def d1(fn, z, d):   # 4th-order central first derivative along direction d
        return (-fn(z + 2 * h * d) + 8 * fn(z + h * d) - 8 * fn(z - h * d)
                + fn(z - 2 * h * d)) / (12 * h)

    for zt in (ZC + 0.04j * e, ZC + 0.1 * np.exp(1j * (BS + 2.0))):
        sx = lambda z: np.array(_tensor(z, tau, k, src))
        gx = d1(sx, zt, 1.0)
        gy = d1(sx, zt, 1j)
        divx = gx[0] + gy[2]
        divy = gx[2] + gy[1]
        scale = np.abs(sx(zt)).max() / ell
        assert abs(divx) <= 1e-5 * scale and abs(divy) <= 1e-5 * scale


@pytest.mark.parametrize("where", ["self", "near_off_line", "collinear", "close_parallel"])
def test_element_rule_matches_double_exponential_quadrature(where):
    """The fixed element rule (graded Gauss-Legendre, oracle/poro.py
    element_integral) against a converged tanh-sinh integral of the point
    kernel over the element, split at the foot of the perpendicular and at a
    few distances from it.  The reference is converged when steps h = 1/16
    and 1/32 agree; the offsets are formed as (rel - s) e, so nodes next to
    the target keep their relative accuracy."""
    k = K3
    e = np.exp(1j * BS)
    a = 0.025
    tau = 100.0
    zt = {"self": ZC, "near_off_line": ZC + 0.03 * np.exp(1j * (BS + 1.2)),
          "collinear": ZC + 0.05 * e, "close_parallel": ZC + 0.01 * e + 0.02j * e}[where]
    for src in ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)):
        _, p, d2 = P.element_integral(zt, ZC, e, a, tau, k, *src)
        ref = [element_integral_ts(zt, ZC, e, a, tau, k, *src, h=h) for h in (1 / 16, 1 / 32)]
        (p16, d16, mag), (p32, d32, _) = ref
        floor = 1e-12 * k["G"] * a      # rounding floor of fields that vanish by symmetry
        # the reference is converged ...
        assert abs(p16 - p32) <= 1e-14 * mag and abs(d16 - d32) <= 1e-14 * mag
        # ... and the element rule reproduces it (measured <= 3e-16 of mag)
        assert abs(p.real - p32) <= 1e-13 * mag + floor, (where, src)
        assert abs(d2 - d32) <= 1e-13 * mag + floor, (where, src)


def test_abi_matrix_convention_and_undrained_block():
    # A_ABI = J A_CS J; at tau -> 0 the DD block is Crouch-Starfield(nu_u)
    n = 6
    t = np.linspace(-1, 1, n + 1)
    xc = 0.5 * (t[1:] + t[:-1])
    g = Geometry(xc, 0.3 * xc ** 2, np.full(n, 1.0 / n), np.full(n, 0.2), np.zeros(n, int),
                 np.array([[0, n - 1]]))
    tau = 1e-8 * (1.0 / n) ** 2 / K3["c"]     # undrained limit approached linearly in tau
    A = P.assemble_dense(g, MAT, tau)
    Au = E.assemble_dense(g, MAT["G"], MAT["nu_u"])
    dd = np.ix_([3 * i + c for i in range(n) for c in (0, 1)],
                [3 * j + c for j in range(n) for c in (0, 1)])
    assert np.abs(A[dd] - Au).max() <= 1e-7 * np.abs(Au).max()
    # an opening DD raises the pore pressure around it, undrained (p compression +)
    for i in range(n):
        assert A[3 * i + 2, 3 * i + 1] > 0


def test_history_sum_pins():
    from oracle import history as H
    n = 3
    g = Geometry(np.array([0.0, 0.3, -0.2]), np.array([0.0, 0.1, 0.25]), np.array([0.05, 0.04, 0.06]),
                 np.array([0.1, 0.9, 2.0]), np.zeros(n, int), np.zeros((1, 2), int))
    mat = dict(MAT, kind=1)
    dt = 100.0
    # h = 0: empty sum; elastic: lag kernels vanish identically
    assert not H.history_sum(g, mat, dt, np.zeros((0, n, 3))).any()
    el = dict(kind=0, G=MAT["G"], nu=MAT["nu"])
    Dh = np.random.default_rng(1).normal(size=(4, n, 3))
    assert not H.history_sum(g, el, dt, Dh).any()
    # telescoping: a source held constant since t = 0 is the continuous-source
    # kernel at the total elapsed time, A^(0) D + sum_m A^(m) D = K((h+1) dt) D
    D = np.random.default_rng(2).normal(size=(n, 3))
    h = 4
    lhs = H.lag_matrix(g, mat, dt, 0) @ D.reshape(-1) + H.history_sum(
        g, mat, dt, np.repeat(D[None], h, axis=0)).reshape(-1)
    rhs = P.assemble_dense(g, MAT, (h + 1) * dt) @ D.reshape(-1)
    assert np.abs(lhs - rhs).max() <= 1e-10 * np.abs(rhs).max()
    # causality / linearity in the history: r_h depends only on D^0..D^(h-1)
    r1 = H.history_sum(g, mat, dt, Dh)
    Dh2 = Dh.copy()
    Dh2[0] *= 2.0
    r2 = H.history_sum(g, mat, dt, Dh2)
    r0 = H.history_sum(g, mat, dt, np.concatenate([Dh[:1], 0 * Dh[1:]]))
    assert np.allclose(r2 - r1, r0, rtol=1e-12, atol=1e-12 * np.abs(r1).max())


# --- reciprocity (SURVEY §8c.3 pin 4) ------------------------------------------
#
# Poroelastic reciprocal theorem (Laplace domain, zero initial state, sources
# switched on at t = 0 and held; tension-positive stress, CS-convention DD
# D = u(0-) - u(0+), q = fluid volume rate per unit length).  From the
# constitutive law sigma = 2G eps + lambda eps_kk I - alpha p I and
# zeta = alpha eps_kk + p/M, s zeta - kappa lap p = gamma:
#     int sigma1:eps2 + p1 gamma2 / s  =  int sigma2:eps1 + p2 gamma1 / s .
# State 1 = a held unit DD at x1 (no fluid source), state 2 = a held unit
# source at x2 (no DD): int sigma2:eps1 = t2(x1) . D (the cut's two faces),
# int sigma1:eps2 = 0, so with p1 = K_pD(s)/s, t2 = K_tq(s)/s ... in the time
# domain
#     sigma_(n|s)(x1, tau | q at x2)  =  int_0^tau p(x2, t | D_(n|s) at x1) dt
# (the q -> traction kernel is the time integral of the DD -> pressure
# kernel).  Dimensionally: the pressure pairs with the injected volume.
# Neither side's formula appears in the other (DD -> p: order-2 part f2 and the
# Gaussian monopole; q -> sigma: h2 and E1), so a dropped term, a wrong sign or
# factor in either fails this.

def _pD_point(w, t, e, Ds, Dn):
    p, _ = P.point_kernel(np.array([w]), t, K3, e, Ds, Dn, 0.0)
    return p[0].real


def _tq_point(w, tau, bt):
    p, d2 = P.point_kernel(np.array([w]), tau, K3, np.exp(1j * bt), 0.0, 0.0, 1.0)
    return -K3["eta"] * p[0] + np.exp(2j * bt) * (-4 * K3["eta"] * d2[0])


def _time_integral(f, tau):
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", integrate.IntegrationWarning)
        return integrate.quad(f, 0.0, tau, epsabs=0, epsrel=1e-13, limit=400,
                              points=[tau * 1e-6, tau * 1e-4, tau * 1e-2])[0]


@pytest.mark.parametrize("x2", [0.03 + 0.02j, -0.01 + 0.05j, 0.1 - 0.02j])
def test_reciprocity_point_kernels(x2):
    b1 = 0.37
    e1 = np.exp(1j * b1)
    x1 = 0.0 + 0.0j
    for tau in (10.0, 100.0, 1000.0):
        T = _tq_point(x1 - x2, tau, b1)
        for Ds, Dn, comp in ((0.0, 1.0, T.real), (1.0, 0.0, T.imag)):
            lhs = _time_integral(lambda t: _pD_point(x2 - x1, t, e1, Ds, Dn), tau)
            assert abs(lhs - comp) <= 1e-12 * abs(comp)


@pytest.mark.parametrize("x2", [0.03 + 0.02j, 0.01 + 0.012j])
def test_reciprocity_element_rule(x2):
    # element level: the pressure at x2 from a DD element (the oracle's fixed
    # element rule, near rule and analytic far form over the time range),
    # time-integrated, equals the traction from a point source at x2
    # integrated along the element (adaptive quadrature of the point kernel)
    b1, a = 0.37, 0.02
    e1 = np.exp(1j * b1)

    def p_elem(t, Ds, Dn):
        r = P.element_integral(x2, 0j, e1, a, t, K3, Ds, Dn, 0.0)
        return (r[1] if r[0] == "near" else r[4]).real

    for tau in (20.0, 200.0):
        for Ds, Dn in ((0.0, 1.0), (1.0, 0.0)):
            lhs = _time_integral(lambda t: p_elem(t, Ds, Dn), tau)
            part = (lambda T: T.real) if Dn else (lambda T: T.imag)
            rhs = integrate.quad(lambda s: part(_tq_point(s * e1 - x2, tau, b1)), -a, a,
                                 epsabs=0, epsrel=1e-13, limit=200)[0]
            assert abs(lhs - rhs) <= 1e-12 * abs(rhs)


def test_fluid_source_far_field_is_centre_of_dilatation():
    # outside the diffusion length the source's
    # potential is V ln r / (2 pi), V = Q tau / S, so sigma^p = 2 eta Phi_,ij =
    # (eta V / pi) d_ij ln r and the face traction is
    #   T = sigma_n + i sigma_s = e^{2 i b_t} (eta V / pi) conj(w)^2 / |w|^4
    # (d_ij ln r is trace-free; sigma_yy - sigma_xx + 2i sigma_xy = 2 conj(w)^2/|w|^4).
    tau = 50.0
    ell = math.sqrt(K3["c"] * tau)
    V = tau / K3["S"]
    for w in (25 * ell * np.exp(0.3j), 40 * ell * np.exp(2.2j), 60 * ell * np.exp(-1.0j)):
        for bt in (0.0, 0.8, 2.5):
            T = _tq_point(w, tau, bt)
            ref = np.exp(2j * bt) * (K3["eta"] * V / np.pi) * np.conj(w) ** 2 / abs(w) ** 4
            assert abs(T - ref) <= 1e-12 * abs(ref)
    # element far form (analytic, u_min > 40) against the same exterior field
    # integrated along the element
    a, bs = 0.3, 0.4
    e = np.exp(1j * bs)
    for zt in (ZC + 40 * ell * np.exp(0.5j), ZC + 70 * ell * np.exp(-2.0j)):
        for bt in (0.2, 1.3):
            Phi, dPhi, Psi, p = P._far_element(zt, ZC, e, a, tau, K3, 0.0, 0.0, 1.0)
            Tf = 2 * Phi.real + np.exp(2j * bt) * (np.conj(zt) * dPhi + Psi)

            # conj(w)^2 / |w|^4 = 1 / w^2 and dw/ds = -e, so the integral over
            # the element is closed-form: (1/e) [1/w(a) - 1/w(-a)]
            wa, wb = zt - (ZC + a * e), zt - (ZC - a * e)
            ref = np.exp(2j * bt) * (K3["eta"] * V / np.pi) * (1 / wa - 1 / wb) / e
            assert abs(Tf - ref) <= 1e-12 * abs(ref)
            assert p == 0.0 or abs(p) <= 1e-30
