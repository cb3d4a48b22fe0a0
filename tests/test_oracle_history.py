"""Pins of the time-marching oracle (oracle/history.py: `march`, `history_sum`,
`poro_rhs`) against closed forms and hand-unrolled recurrences, not against
itself.  CPU only.

The step-h system (Eq.(final_sigs)-(final_pp); reading
R10): A^(0) D^h = b - sum_{m=1}^{h} A^(m) D^(h-m).
"""
import numpy as np
import pytest

from oracle import elastic as E
from oracle import history as H
from oracle import poro as P
from synth import CONFIGS
from synth.geometry import Geometry

MAT = dict(CONFIGS[3]["material"])


def _one_element():
    return Geometry(np.array([0.0]), np.array([0.0]), np.array([0.05]), np.array([0.3]),
                    np.zeros(1, int), np.zeros((1, 2), int))


def _tiny(n=3):
    return Geometry(np.array([0.0, 0.3, -0.2])[:n], np.array([0.0, 0.1, 0.25])[:n],
                    np.array([0.05, 0.04, 0.06])[:n], np.array([0.1, 0.9, 2.0])[:n],
                    np.zeros(n, int), np.zeros((1, 2), int))


@pytest.mark.parametrize("kind", ["one_lag", "all_lags"])
def test_march_closed_form_recurrences(kind):
    # synthetic lags with closed-form solutions: an off-by-one in the history
    # slice (D[:h]), in the lag index (h - m) or in the sign of the subtraction
    # changes these sequences
    g = _tiny(2)
    n3 = 3 * g.n
    steps = 7
    Id = np.eye(n3)
    b = np.random.default_rng(3).normal(size=(g.n, 3))
    if kind == "one_lag":
        # A0 = I, A1 = -I, A_m>1 = 0:  D^h = b + D^(h-1)  =>  D^h = (h + 1) b
        lags = [Id, -Id] + [0 * Id] * (steps - 1)
        expect = [(h + 1) * b for h in range(steps)]
    else:
        # A0 = I, A_m = -I:  D^h = b + sum_{eta<h} D^eta  =>  D^h = 2^h b
        lags = [Id] + [-Id] * steps
        expect = [2.0 ** h * b for h in range(steps)]
    D = H.march(g, None, 1.0, b, steps, lags=lags)
    for h in range(steps):
        assert np.allclose(D[h], expect[h], rtol=1e-14, atol=0)
    # distinct lags: A0 = I, A_m = -m I gives D^h = b + sum_m m D^(h-m); first
    # terms b, 2b, 5b, 13b, 34b (every other Fibonacci number)
    lags = [Id] + [-m * Id for m in range(1, steps + 1)]
    D = H.march(g, None, 1.0, b, 5, lags=lags)
    for h, f in enumerate((1, 2, 5, 13, 34)):
        assert np.allclose(D[h], f * b, rtol=1e-14, atol=0)


def test_march_single_element_hand_unrolled():
    # N = 1 poroelastic (S:442 scalar blocks): three steps unrolled by hand
    # from explicitly assembled 3x3 continuous-source kernels K(tau)
    g = _one_element()
    dt = 60.0
    K = [P.assemble_dense(g, MAT, j * dt) for j in (1, 2, 3, 4)]
    A0, A1, A2 = K[0], K[1] - K[0], K[2] - K[1]
    b = np.array([1e6, 5e6, 1e7])
    D0 = np.linalg.solve(A0, b)
    D1 = np.linalg.solve(A0, b - A1 @ D0)
    D2 = np.linalg.solve(A0, b - A1 @ D1 - A2 @ D0)
    D = H.march(g, dict(MAT, kind=1), dt, b.reshape(1, 3), 3)
    for h, ref in enumerate((D0, D1, D2)):
        assert np.abs(D[h, 0] - ref).max() <= 1e-12 * np.abs(ref).max()
    # the march satisfies the step equations it defines: sum over the whole
    # history with the continuous-source kernels (telescoped form
    # sum_j K(j dt) (D^(h+1-j) - D^(h-j))) equals b at every step
    for h in range(3):
        tot = np.zeros(3)
        for j in range(1, h + 2):
            prev = D[h - j, 0] if h - j >= 0 else np.zeros(3)
            tot += K[j - 1] @ (D[h + 1 - j, 0] - prev)
        assert np.abs(tot - b).max() <= 1e-9 * np.abs(b).max()


def test_history_sum_tiny_hand_unrolled():
    # N = 3, h = 4 term by term (SURVEY §8c.7 pin), lags from K(tau) directly
    g = _tiny(3)
    dt = 100.0
    mat = dict(MAT, kind=1)
    K = [P.assemble_dense(g, MAT, j * dt) for j in range(1, 6)]
    Dh = np.random.default_rng(7).normal(size=(4, g.n, 3))
    r = np.zeros(3 * g.n)
    r += (K[1] - K[0]) @ Dh[3].reshape(-1)     # m = 1, D^(h-1)
    r += (K[2] - K[1]) @ Dh[2].reshape(-1)     # m = 2
    r += (K[3] - K[2]) @ Dh[1].reshape(-1)     # m = 3
    r += (K[4] - K[3]) @ Dh[0].reshape(-1)     # m = 4, D^0
    got = H.history_sum(g, mat, dt, Dh)
    assert np.abs(got.reshape(-1) - r).max() <= 1e-12 * np.abs(r).max()


def test_poro_rhs_readings():
    # P15 (config 3, 'net'): horizontal fractures (beta = 0, face normal = y =
    # Shmin direction) see b_s = 0, b_n = 5 MPa, b_p = (sh + 5) - p0 = 10 MPa
    g = Geometry(np.array([0.0, 1.0]), np.array([0.0, 20.0]), np.full(2, 0.025), np.zeros(2),
                 np.arange(2), np.zeros((2, 2), int))
    b = H.poro_rhs(g, CONFIGS[3]["load"])
    assert np.allclose(b, [[0.0, 5e6, 1e7]] * 2, rtol=0, atol=1e-9)
    # P14 (config 4, 'absolute', p_f - p0 = 10 MPa): b_p = 10 MPa on every
    # element; b_n = p_f - sigma_n^ff(beta) = 30 - 25 MPa at beta = 0 and
    # 30 - 30 MPa at beta = pi/2; an isotropic far field has no shear load
    g4 = Geometry(np.zeros(2), np.zeros(2), np.full(2, 0.1), np.array([0.0, np.pi / 2]),
                  np.arange(2), np.zeros((2, 2), int))
    b4 = H.poro_rhs(g4, CONFIGS[4]["load"])
    assert np.allclose(b4[:, 2], 1e7, rtol=0, atol=1e-9)
    assert np.allclose(b4[:, 1], [5e6, 0.0], rtol=0, atol=1e-6)
    assert np.allclose(b4[:, 0], 0.0, atol=1e-6)
    iso = dict(CONFIGS[4]["load"], sH=25e6)
    g45 = Geometry(np.zeros(1), np.zeros(1), np.full(1, 0.1), np.array([0.7]), np.arange(1),
                   np.zeros((1, 2), int))
    assert abs(H.poro_rhs(g45, iso)[0, 0]) <= 1e-6
