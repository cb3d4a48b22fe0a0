"""GMRES preconditioners against the oracle's dense matrix.

Leaf-block Jacobi: the blocks are the exact dense sub-matrices of chunks of
<= 32 consecutive (Morton-sorted) elements of one leaf, so M^-1 x must solve
those sub-systems of the oracle's dense influence matrix (bar 1e-9 relative:
the blocks are inverted in fp64 with partial pivoting).  Point-block Jacobi:
the element self blocks.  GMRES with either reaches the LU solution; the leaf
blocks take fewer iterations."""
import numpy as np
import pytest

from oracle import elastic as OE
from oracle import poro as OP
from synth import CONFIGS, make_config, random_dd

pytestmark = pytest.mark.gpu

KCHUNK = 32


@pytest.fixture(scope="module")
def ddm():
    import torch
    import paper_1812_05087_b200 as D
    return D, D.Context(0), torch


def _tree(D, torch, ctx, g, leaf, min_side=0.0):
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    return D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=leaf, order_p=20,
                  min_leaf_side=min_side)


def _chunks(tree):
    """The documented chunking: each leaf's sorted range split into
    ceil(count / 32) near-equal consecutive parts; returns lists of user ids."""
    perm = tree.export("PERM")
    start, count = tree.export("START"), tree.export("COUNT")
    out = []
    for c in sorted(tree.export("LEAVES"), key=lambda c: start[c]):
        s0, n0 = int(start[c]), int(count[c])
        nc = -(-n0 // KCHUNK)
        for q in range(nc):
            a, b = s0 + n0 * q // nc, s0 + n0 * (q + 1) // nc
            out.append(perm[a:b])
    return out


def _check_leaf(A, chunks, x, y, ncomp, tol):
    n_checked = 0
    for ids in chunks:
        rows = (ids[:, None] * ncomp + np.arange(ncomp)[None, :]).reshape(-1)
        Ab = A[np.ix_(rows, rows)]
        xb = x.reshape(-1)[rows]
        yb = y.reshape(-1)[rows]
        ref = np.linalg.solve(Ab, xb)
        # compare each component group on its own scale (poroelastic rows mix units)
        for c in range(ncomp):
            sl = slice(c, None, ncomp)
            assert np.linalg.norm(yb[sl] - ref[sl]) <= tol * np.linalg.norm(ref[sl]) + 1e-300
        n_checked += 1
    return n_checked


def test_leaf_blocks_elastic_cfg2(ddm):
    D, ctx, torch = ddm
    g = make_config(2)
    c = CONFIGS[2]
    m = c["material"]
    tree = _tree(D, torch, ctx, g, 64)      # leaves of up to 64 -> split into 2 chunks
    A = OE.assemble_dense(g, m["G"], m["nu"])
    x = random_dd(g.n, 2, 3)
    y = D.precond_apply(ctx, tree, D.material_from_dict(m), torch.tensor(x, device="cuda"),
                        kind="leaf").cpu().numpy()
    ch = _chunks(tree)
    assert max(len(i) for i in ch) <= KCHUNK and sum(len(i) for i in ch) == g.n
    assert any(len(i) < KCHUNK for i in ch)   # ragged chunks present
    assert _check_leaf(A, ch, x, y, 2, 1e-9) == len(ch)
    # point blocks: the 2x2 self blocks
    yp = D.precond_apply(ctx, tree, D.material_from_dict(m), torch.tensor(x, device="cuda"),
                         kind="point").cpu().numpy()
    for i in range(0, g.n, 97):
        Ab = A[2 * i:2 * i + 2, 2 * i:2 * i + 2]
        assert np.allclose(yp[i], np.linalg.solve(Ab, x[i]), rtol=1e-11, atol=0)


def test_leaf_blocks_poro_cfg4(ddm):
    D, ctx, torch = ddm
    g = make_config(4)
    c = CONFIGS[4]
    m = c["material"]
    dt = c["dt"]
    tree = _tree(D, torch, ctx, g, 32)
    A = OP.assemble_dense(g, m, dt)
    x = random_dd(g.n, 3, 4)
    x[:, 2] *= 1e-9
    y = D.precond_apply(ctx, tree, D.material_from_dict(m), torch.tensor(x, device="cuda"),
                        dt=dt, kind="leaf").cpu().numpy()
    ch = _chunks(tree)
    assert _check_leaf(A, ch, x, y, 3, 1e-8) == len(ch)


def test_gmres_leaf_vs_point_elastic(ddm):
    D, ctx, torch = ddm
    g = make_config(2)
    c = CONFIGS[2]
    m = c["material"]
    tree = _tree(D, torch, ctx, g, c["leaf"])
    load = c["load"]
    b = D.farfield_rhs(ctx, torch.tensor(g.beta, device="cuda"), 2, load["p_f"], load["sH"],
                       load["sh"])
    mat = D.material_from_dict(m)
    A = OE.assemble_dense(g, m["G"], m["nu"])
    x_lu = np.linalg.solve(A, OE.farfield_rhs(g, load).reshape(-1)).reshape(-1, 2)
    res = {}
    for pc in ("leaf", "point", False):
        x, it, rr = D.gmres_solve(ctx, tree, mat, b, tol=1e-10, precond=pc)
        assert rr <= 1e-10
        assert np.linalg.norm(x.cpu().numpy() - x_lu) / np.linalg.norm(x_lu) <= 1e-6
        res[pc] = it
    assert res["leaf"] < res["point"] < res[False], res


def test_gmres_leaf_poro_cfg4(ddm):
    D, ctx, torch = ddm
    g = make_config(4)
    c = CONFIGS[4]
    m = c["material"]
    dt = c["dt"]
    k = OP.constants(m["G"], m["nu"], m["nu_u"], m["alpha"], m["kappa"])
    rc = (160 * k["c"] * dt) ** 0.5 + 2 * g.half_len.max()
    tree = _tree(D, torch, ctx, g, 32, rc)
    mat = D.material_from_dict(m)
    bp = np.random.default_rng(9).uniform(-1, 1, (g.n, 3)) * np.array([1e6, 1e6, 1e-3])
    b = torch.tensor(bp, device="cuda")
    A = OP.assemble_dense(g, m, dt)
    x_lu = np.linalg.solve(A, bp.reshape(-1)).reshape(-1, 3)
    its = {}
    for pc in ("leaf", "point"):
        x, it, rr = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=1e-10, precond=pc, restart=3000,
                                  max_iter=6000)
        assert rr <= 1e-10
        xs = x.cpu().numpy()
        for comp in range(3):
            e = np.linalg.norm(xs[:, comp] - x_lu[:, comp]) / np.linalg.norm(x_lu[:, comp])
            assert e <= 1e-6, (pc, comp, e)
        its[pc] = it
    assert its["leaf"] < its["point"], its
