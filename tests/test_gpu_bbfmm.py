"""GPU Chebyshev (bbFMM) far field vs the bbFMM oracle.

The GPU path and oracle/bbfmm.py compute the same approximation (same tree,
lists, nodes and quadrature), so they agree to rounding: bar 1e-10 relative
L2.  Against the exact dense matvec the bar is the interpolation accuracy the
oracle pins show (n = 3: 1e-3, n = 6: 1e-5)."""
import numpy as np
import pytest

from oracle import bbfmm as BB
from oracle import elastic as OE
from synth import CONFIGS, make_config, random_dd
from synth.geometry import Geometry

pytestmark = pytest.mark.gpu

G0, NU0 = 8e9, 0.25


@pytest.fixture(scope="module")
def ddm():
    import torch
    import paper_1812_05087_b200 as D
    return D, D.Context(0), torch


def _tree(D, ctx, torch, g, leaf):
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    return D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=leaf, order_p=20)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n", [2, 3, 6, 8])
def test_bbfmm_parity_cfg2(ddm, n):
    D, ctx, torch = ddm
    g = make_config(2)
    leaf = CONFIGS[2]["leaf"]
    t = _tree(D, ctx, torch, g, leaf)
    Dv = random_dd(g.n, 2, 102 + n)
    y = D.matvec(ctx, t, D.material(0, G0, NU0), torch.tensor(Dv, device="cuda"),
                 mode=f"bbfmm{n}").cpu().numpy()
    ref = BB.bbfmm_matvec(g, G0, NU0, Dv, leaf, n)
    assert _rel(y, ref) <= 1e-10
    exact = OE.matvec_dense(OE.assemble_dense(g, G0, NU0), Dv)
    assert _rel(y, exact) <= {2: 2e-3, 3: 1e-3, 6: 1e-5, 8: 1e-6}[n]


def test_bbfmm_parity_small_leaves(ddm):
    """Deeper tree (leaf 8): more M2M/L2L levels, W lists, ragged leaves."""
    D, ctx, torch = ddm
    g = make_config(2)
    t = _tree(D, ctx, torch, g, 8)
    Dv = random_dd(g.n, 2, 5)
    y = D.matvec(ctx, t, D.material(0, G0, NU0), torch.tensor(Dv, device="cuda"),
                 mode="bbfmm5").cpu().numpy()
    assert _rel(y, BB.bbfmm_matvec(g, G0, NU0, Dv, 8, 5)) <= 1e-10


def test_bbfmm_tiny_and_single_level(ddm):
    """Fewer elements than one leaf: no far field at all, result = direct."""
    D, ctx, torch = ddm
    g = make_config(2)
    keep = np.arange(20)
    gs = Geometry(g.xc[keep], g.yc[keep], g.half_len[keep], g.beta[keep], g.frac_id[keep], g.tips[:1])
    t = _tree(D, ctx, torch, gs, 32)
    Dv = random_dd(gs.n, 2, 1)
    mat = D.material(0, G0, NU0)
    Dt = torch.tensor(Dv, device="cuda")
    y = D.matvec(ctx, t, mat, Dt, mode="bbfmm3").cpu().numpy()
    yd = D.matvec(ctx, t, mat, Dt, mode="direct").cpu().numpy()
    assert _rel(y, yd) <= 1e-12


def test_bbfmm_gmres(ddm):
    """GMRES with the bbFMM operator: solution within the operator's accuracy
    of the dense LU solution."""
    D, ctx, torch = ddm
    g = make_config(2)
    c = CONFIGS[2]
    t = _tree(D, ctx, torch, g, c["leaf"])
    m = c["material"]
    load = c["load"]
    b = D.farfield_rhs(ctx, torch.tensor(g.beta, device="cuda"), 2, load["p_f"], load["sH"],
                       load["sh"])
    x, it, rr = D.gmres_solve(ctx, t, D.material_from_dict(m), b, tol=1e-10, mode="bbfmm6")
    A = OE.assemble_dense(g, m["G"], m["nu"])
    x_lu = np.linalg.solve(A, OE.farfield_rhs(g, load).reshape(-1)).reshape(-1, 2)
    assert rr <= 1e-10
    assert _rel(x.cpu().numpy(), x_lu) <= 1e-4


def test_bbfmm_errors(ddm):
    D, ctx, torch = ddm
    g = make_config(2)
    t = _tree(D, ctx, torch, g, 32)
    Dt = torch.zeros((g.n, 2), dtype=torch.float64, device="cuda")
    for bad in ("bbfmm1", "bbfmm9"):
        with pytest.raises(RuntimeError):
            D.matvec(ctx, t, D.material(0, G0, NU0), Dt, mode=bad)
    with pytest.raises(RuntimeError):
        D.matvec(ctx, t, D.material(1, 8e9, 0.2, nu_u=0.3, alpha=0.7, kappa=1e-15),
                 torch.zeros((g.n, 3), dtype=torch.float64, device="cuda"), mode="bbfmm3",
                 elapsed=10.0)
