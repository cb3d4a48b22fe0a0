"""Pins of the Chebyshev bbFMM oracle (oracle/bbfmm.py).

- S_n against the Lagrange basis on the roots of T_n written as a
  product (an independent formula): cardinality, partition of unity,
  exactness on polynomials of degree < n.
- The Gauss-Legendre rule used along the elements integrates degree 2n-1
  exactly.
- The whole far field converges geometrically in n to the exact dense matvec
  (oracle.elastic, closed-form element integrals): a dropped term, a wrong
  re-centring or a transposed interpolation matrix stalls the error at O(1)
  relative to the far-field share instead.
- The paper's own accuracy statement (NCheb3's error a few
  times NCheb6's) holds as an ordering."""
import numpy as np
import pytest

from oracle import bbfmm as BB
from oracle import elastic as OE
from synth import CONFIGS, make_config, random_dd

G0, NU0 = 8e9, 0.25


def _lagrange(n, x):
    xb = BB.cheb_nodes(n)
    out = np.ones((n, x.size))
    for l in range(n):
        for j in range(n):
            if j != l:
                out[l] *= (x - xb[j]) / (xb[l] - xb[j])
    return out


@pytest.mark.parametrize("n", [2, 3, 6, 8])
def test_cardinal_is_lagrange_basis(n):
    x = np.random.default_rng(n).uniform(-1.3, 1.3, 50)
    S = BB.cardinal(n, BB.cheb_nodes(n), x)
    assert np.allclose(S, _lagrange(n, x), rtol=0, atol=1e-12)
    # cardinality and partition of unity
    assert np.allclose(BB.cardinal(n, BB.cheb_nodes(n), BB.cheb_nodes(n)), np.eye(n), atol=1e-13)
    assert np.allclose(S.sum(axis=0), 1.0, atol=1e-13)
    # exact on x^k, k < n
    xb = BB.cheb_nodes(n)
    for k in range(n):
        assert np.allclose(S.T @ xb ** k, x ** k, atol=1e-11)


def test_nodes_are_roots_of_Tn():
    for n in range(1, 9):
        xb = BB.cheb_nodes(n)
        assert np.allclose(np.polynomial.chebyshev.chebval(xb, [0] * n + [1]), 0, atol=1e-13)
        assert len(set(np.round(xb, 12))) == n


@pytest.mark.parametrize("n", [2, 3, 6, 8])
def test_gauss_legendre_degree(n):
    x, w = np.polynomial.legendre.leggauss(n)
    for k in range(2 * n):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.sum(w * x ** k) - exact) < 1e-13


@pytest.fixture(scope="module")
def cfg2_dense():
    g = make_config(2)
    A = OE.assemble_dense(g, G0, NU0)
    D = random_dd(g.n, 2, 102)
    return g, D, OE.matvec_dense(A, D)


def test_bbfmm_converges_to_dense(cfg2_dense):
    g, D, y = cfg2_dense
    errs = {}
    for n in (2, 3, 4, 6, 8):
        yb = BB.bbfmm_matvec(g, G0, NU0, D, CONFIGS[2]["leaf"], n)
        errs[n] = np.linalg.norm(yb - y) / np.linalg.norm(y)
    # geometric convergence: every step down, and the measured rates of the
    # 2D Chebyshev interpolation on well-separated cells (factor >= 3 per node)
    ns = sorted(errs)
    for a, b in zip(ns, ns[1:]):
        assert errs[b] < errs[a] / 2.5, errs
    assert errs[3] < 1e-3 and errs[6] < 1e-5 and errs[8] < 1e-6, errs
    # NCheb3's error a few times NCheb6's (at least 4x)
    assert errs[3] > 4 * errs[6]


def test_bbfmm_single_source_column(cfg2_dense):
    """One source element: the result is one dense column (near targets exact,
    far targets the interpolated field) within the n = 8 accuracy."""
    g, D, y = cfg2_dense
    Ds = np.zeros_like(D)
    Ds[17] = (1e-3, 2e-3)
    A = OE.assemble_dense(g, G0, NU0)
    ref = OE.matvec_dense(A, Ds)
    yb = BB.bbfmm_matvec(g, G0, NU0, Ds, CONFIGS[2]["leaf"], 8)
    assert np.linalg.norm(yb - ref) / np.linalg.norm(ref) < 1e-5
