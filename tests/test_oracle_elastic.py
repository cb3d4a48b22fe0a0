"""Pins of the elastic oracle against what the paper and the mathematics fix
(not against itself).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import elastic as E
from oracle import sif as S
from oracle.gmres import gmres
from synth import make_config, random_dd
from synth.geometry import Geometry

G0, NU0, E0 = 8e9, 0.25, 20e9
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _one(xc, yc, a, b):
    return Geometry(np.array([xc]), np.array([yc]), np.array([a]), np.array([b]),
                    np.array([0]), np.array([[0, 0]]))


@pytest.fixture(scope="module")
def cfg1():
    g = make_config(1)
    return g, E.assemble_dense(g, G0, NU0)


@pytest.fixture(scope="module")
def cfg2():
    g = make_config(2)
    return g, E.assemble_dense(g, G0, NU0)


def test_self_term_closed_form():
    # s_yy(0,0) = G / (pi (1 - nu) a) per unit D_y (Crouch-Starfield self term)
    for a in (0.005, 1.0, 3.7):
        A = E.assemble_dense(_one(0.3, -2.0, a, 0.7), G0, NU0)
        ref = G0 / (np.pi * (1 - NU0) * a)
        assert abs(A[1, 1] - ref) <= 1e-14 * ref
        assert abs(A[0, 0] - ref) <= 1e-14 * ref          # shear self term, same value
        assert abs(A[0, 1]) <= 1e-14 * ref and abs(A[1, 0]) <= 1e-14 * ref


def test_sneddon_opening(cfg1):
    # BASELINE configs[0]: w = 4 (1 - nu^2) p / E sqrt(a^2 - x^2)
    g, A = cfg1
    b = np.zeros((g.n, 2))
    b[:, 1] = 1e6
    x = np.linalg.solve(A, b.reshape(-1)).reshape(-1, 2)
    w = E.sneddon_opening(g.xc, 1.0, 1e6, E0, NU0)
    c = g.n // 2
    assert abs(x[c, 1] / w[c] - 1) < 0.01
    inner = slice(1, g.n - 1)
    rms = np.sqrt(np.mean(((x[inner, 1] - w[inner]) / w[inner]) ** 2))
    assert rms < 0.02
    assert np.abs(x[:, 0]).max() < 1e-12 * np.abs(x[:, 1]).max()   # no shear under pressure
    # SIF: K_I(Eq.SIF) / (p sqrt(pi a)) -- 0.806 corrects the tip overshoot
    KI, _ = S.sif(x[-1, 1], 0.0, g.half_len[-1], E0, NU0)
    assert abs(KI / (1e6 * np.sqrt(np.pi)) - 1.0095) < 0.01


def test_straight_crack_symmetric_toeplitz(cfg1):
    g, A = cfg1
    assert np.array_equal(A, A.T)
    assert np.abs(A[0::2, 1::2]).max() == 0.0 and np.abs(A[1::2, 0::2]).max() == 0.0
    Ann = A[1::2, 1::2]
    for k in (0, 1, 5, 50):
        d = np.diagonal(Ann, k)
        assert np.abs(d - d[0]).max() <= 1e-12 * abs(d[0])


def test_displacement_jump_equals_D():
    a, Dx, Dy = 1.3, 0.7, -0.4
    x = np.linspace(-1.2, 1.2, 9)
    up = E.cs_local_disp(x, 1e-12, a, Dx, Dy, NU0)
    dn = E.cs_local_disp(x, -1e-12, a, Dx, Dy, NU0)
    assert np.allclose(dn[0] - up[0], Dx, atol=1e-9)
    assert np.allclose(dn[1] - up[1], Dy, atol=1e-9)


def test_hooke_and_equilibrium_finite_differences():
    # stresses must equal Hooke's law (plane strain) applied to the displacement
    # field, and be divergence free (independent of the stress formulas)
    rng = np.random.default_rng(7)
    a, Dx, Dy = 1.0, 0.3, -0.8
    lam = 2 * G0 * NU0 / (1 - 2 * NU0)
    h = 1e-5
    for _ in range(20):
        x, y = rng.uniform(-3, 3), rng.uniform(0.2, 3) * rng.choice([-1, 1])
        ux = lambda X, Y: E.cs_local_disp(X, Y, a, Dx, Dy, NU0)[0]
        uy = lambda X, Y: E.cs_local_disp(X, Y, a, Dx, Dy, NU0)[1]
        exx = (ux(x + h, y) - ux(x - h, y)) / (2 * h)
        eyy = (uy(x, y + h) - uy(x, y - h)) / (2 * h)
        exy = 0.5 * ((ux(x, y + h) - ux(x, y - h)) + (uy(x + h, y) - uy(x - h, y))) / (2 * h)
        sxx, syy, sxy = E.cs_local_stress(x, y, a, Dx, Dy, G0, NU0)
        scale = max(abs(sxx), abs(syy), abs(sxy))
        assert abs(2 * G0 * exx + lam * (exx + eyy) - sxx) < 1e-6 * scale
        assert abs(2 * G0 * eyy + lam * (exx + eyy) - syy) < 1e-6 * scale
        assert abs(2 * G0 * exy - sxy) < 1e-6 * scale
        s = lambda X, Y: E.cs_local_stress(X, Y, a, Dx, Dy, G0, NU0)
        divx = (s(x + h, y)[0] - s(x - h, y)[0]) / (2 * h) + (s(x, y + h)[2] - s(x, y - h)[2]) / (2 * h)
        divy = (s(x + h, y)[2] - s(x - h, y)[2]) / (2 * h) + (s(x, y + h)[1] - s(x, y - h)[1]) / (2 * h)
        assert abs(divx) < 1e-5 * scale and abs(divy) < 1e-5 * scale


def test_additivity_of_split_elements():
    # a constant element of half-length a equals two halves at +-a/2 (exact integral)
    rng = np.random.default_rng(3)
    for _ in range(50):
        a = rng.uniform(0.1, 2)
        x, y = rng.uniform(-4, 4, 2)
        if abs(y) < 1e-3:
            continue
        Dx, Dy = rng.normal(size=2)
        full = np.array(E.cs_local_stress(x, y, a, Dx, Dy, G0, NU0))
        half = (np.array(E.cs_local_stress(x - a / 2, y, a / 2, Dx, Dy, G0, NU0)) +
                np.array(E.cs_local_stress(x + a / 2, y, a / 2, Dx, Dy, G0, NU0)))
        assert np.abs(full - half).max() <= 1e-10 * np.abs(full).max()


def test_r_minus_2_decay():
    for ang in (0.3, 1.1, 2.0):
        r = np.array([100.0, 200.0, 400.0])
        vals = E.cs_local_stress(r * np.cos(ang), r * np.sin(ang), 0.5, 0.2, 1.0, G0, NU0)[1]
        slope = np.log(abs(vals[2] / vals[1])) / np.log(2.0)
        assert abs(slope + 2) < 1e-3


def test_rotation_invariance(cfg2):
    g, A = cfg2
    th = 0.6180339887
    c, s = np.cos(th), np.sin(th)
    g2 = Geometry(c * g.xc - s * g.yc + 13.0, s * g.xc + c * g.yc - 7.0, g.half_len,
                  g.beta + th, g.frac_id, g.tips)
    A2 = E.assemble_dense(g2, G0, NU0)
    assert np.abs(A2 - A).max() <= 1e-9 * np.abs(A).max()
    D = random_dd(g.n, 2, 102)
    y, y2 = E.matvec_dense(A, D), E.matvec_dense(A2, D)
    assert np.linalg.norm(y2 - y) <= 1e-12 * np.linalg.norm(y)


def _km_matvec(g, D, G, nu):
    """Independent formula family: Kolosov-Muskhelishvili potentials of a
    constant DD element, summed over all sources."""
    C = 1 / (4 * np.pi * (1 - nu))
    e = np.exp(1j * g.beta)
    zc = g.xc + 1j * g.yc
    z1, z2 = zc - g.half_len * e, zc + g.half_len * e
    B = (D[:, 0] + 1j * D[:, 1]) * e
    r = np.exp(-2j * g.beta)
    Q = r * B - np.conj(B)
    out = np.empty((g.n, 2))
    for i in range(g.n):
        z = zc[i]
        I2 = 1 / (z - z2) - 1 / (z - z1)
        I3 = 0.5 * (1 / (z - z2) ** 2 - 1 / (z - z1) ** 2)
        I3b = (np.conj(zc) + r * (z - zc)) * I3 - r * I2
        Phi = 1j * G * C * np.sum(B * I2)
        dPhi = -2j * G * C * np.sum(B * I3)
        Psi = 1j * G * C * np.sum(Q * I2 + 2 * B * I3b)
        T = 2 * Phi.real + np.exp(2j * g.beta[i]) * (np.conj(z) * dPhi + Psi)
        out[i] = (T.imag, T.real)
    return out


def test_complex_variable_family_agrees(cfg2):
    g, A = cfg2
    D = random_dd(g.n, 2, 102)
    y = E.matvec_dense(A, D)
    yk = _km_matvec(g, D, G0, NU0)
    assert np.linalg.norm(yk - y) <= 1e-12 * np.linalg.norm(y)
    # row-sampled matrix-free path equals the dense one
    rows = np.arange(0, g.n, 37)
    yr = E.matvec_rows(g, G0, NU0, D, rows)
    assert np.linalg.norm(yr - y[rows]) <= 1e-14 * np.linalg.norm(y[rows])


def test_farfield_load_resolution():
    # beta = 0 -> (0, sh); beta = pi/2 -> (0, sH); isotropic -> no shear
    g = Geometry(np.zeros(3), np.zeros(3), np.ones(3), np.array([0.0, np.pi / 2, 0.4]),
                 np.arange(3), np.zeros((3, 2), int))
    load = {"p_f": 0.0, "sH": 58.60e6, "sh": 55.15e6, "p0": 0.0, "mode": "absolute"}
    b = E.farfield_rhs(g, load)
    assert abs(b[0, 0]) < 1e-6 and abs(b[0, 1] + 55.15e6) < 1e-6
    assert abs(b[1, 0]) < 1e-6 and abs(b[1, 1] + 58.60e6) < 1e-6
    iso = dict(load, sH=40e6, sh=40e6)
    assert np.abs(E.farfield_rhs(g, iso)[:, 0]).max() < 1e-6


def test_inclined_crack_sliding_sign():
    # Pins the sign of the shear load: under a positive resolved shear the +n
    # face slides along +t by 4(1-nu^2) tau/E sqrt(a^2-x^2) (Griffith mode II),
    # and the opening follows Sneddon with the net normal pressure.
    beta = np.pi / 6
    n = 200
    k = (np.arange(n) + 0.5) / n
    t = -1 + 2 * k
    g = Geometry(t * np.cos(beta), t * np.sin(beta), np.full(n, 1.0 / n), np.full(n, beta),
                 np.zeros(n, int), np.array([[0, n - 1]]))
    sH, sh = 30e6, 25e6
    snff = sH * np.sin(beta) ** 2 + sh * np.cos(beta) ** 2
    load = {"p_f": snff + 1e6, "sH": sH, "sh": sh, "p0": 0.0, "mode": "absolute"}
    A = E.assemble_dense(g, G0, NU0)
    x = np.linalg.solve(A, E.farfield_rhs(g, load).reshape(-1)).reshape(-1, 2)
    tau = (sH - sh) * np.sin(beta) * np.cos(beta)      # tension-positive t.sigma.n
    c = n // 2
    assert abs(x[c, 0] / E.sneddon_opening(t[c], 1.0, tau, E0, NU0) - 1) < 0.01
    assert abs(x[c, 1] / E.sneddon_opening(t[c], 1.0, 1e6, E0, NU0) - 1) < 0.01
    # and directly from the displacement field: u(+n) - u(-n) along t = D_s
    e_t = np.array([np.cos(beta), np.sin(beta)])
    e_n = np.array([-np.sin(beta), np.cos(beta)])
    P = 0.003 * e_t
    du = np.zeros(2)
    for side, sgn in ((1e-9, 1), (-1e-9, -1)):
        q = P + side * e_n
        u = np.zeros(2)
        for j in range(n):
            dx, dy = q[0] - g.xc[j], q[1] - g.yc[j]
            xl = dx * np.cos(beta) + dy * np.sin(beta)
            yl = -dx * np.sin(beta) + dy * np.cos(beta)
            # ABI DDs are minus the CS DDs
            ul = E.cs_local_disp(xl, yl, g.half_len[j], -x[j, 0], -x[j, 1], NU0)
            u += ul[0] * e_t + ul[1] * e_n
        du += sgn * u
    assert du @ e_t > 0 and abs(du @ e_t / x[c, 0] - 1) < 0.02
    assert du @ e_n > 0


def test_sif_golden_value():
    gv = GOLD["sif_example"]
    Ey = 2 * gv["G"] * (1 + gv["nu"])
    KI, KII = S.sif(gv["Dn"], 0.0, gv["a"], Ey, gv["nu"])
    assert abs(KI / gv["KI"] - 1) < gv["rel_tol"] and KII == 0.0
    KI2, KII2 = S.sif(2 * gv["Dn"], -gv["Dn"], gv["a"], Ey, gv["nu"])   # linear in D
    assert abs(KI2 - 2 * KI) <= 1e-9 * KI and abs(KII2 + KI) <= 1e-9 * KI


def test_gmres_matches_lu(cfg1, cfg2):
    for (g, A), load in ((cfg1, {"p_f": 1e6, "sH": 0.0, "sh": 0.0, "mode": "absolute"}),
                         (cfg2, {"p_f": 10e6, "sH": 30e6, "sh": 25e6, "mode": "absolute"})):
        b = E.farfield_rhs(g, load).reshape(-1)
        x_lu = np.linalg.solve(A, b)
        x, it, rr, ok = gmres(lambda v: A @ v, b, tol=1e-10)
        assert ok and rr <= 1e-10 and 0 < it < 2000
        kappa = np.linalg.cond(A)
        assert np.linalg.norm(x - x_lu) <= 10 * 1e-10 * kappa * np.linalg.norm(x_lu)
        assert np.linalg.norm(b - A @ x) <= 1.0001e-10 * np.linalg.norm(b)


def test_gmres_special_cases():
    x, it, rr, ok = gmres(lambda v: v, np.zeros(5))
    assert it == 0 and ok and not x.any()
    b = np.arange(1.0, 6.0)
    x, it, rr, ok = gmres(lambda v: v, b)
    assert it == 1 and np.allclose(x, b, rtol=1e-15)
    M = np.array([[4.0, 1.0, 0.0], [1.0, 3.0, 1.0], [0.0, 1.0, 2.0]])
    inv = np.array([[5.0, -2.0, 1.0], [-2.0, 8.0, -4.0], [1.0, -4.0, 11.0]]) / 18.0  # closed form
    b = np.array([1.0, -2.0, 0.5])
    x, it, rr, ok = gmres(lambda v: M @ v, b, tol=1e-14)
    assert ok and np.allclose(x, inv @ b, rtol=0, atol=1e-13)
    # restarted GMRES converges to the same answer
    x2, it2, rr2, ok2 = gmres(lambda v: M @ v, b, tol=1e-14, restart=1, max_iter=500)
    assert ok2 and np.allclose(x2, inv @ b, atol=1e-12)
