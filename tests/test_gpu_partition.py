"""Multi-rank compute partition on one GPU: with the tree
partitioned for rank r of W (ddm_tree_partition), a single-process matvec
writes exactly rank r's owned rows, and they are bitwise equal to the
unpartitioned result -- the per-target summation order depends only on the
tree.  This runs every kernel of the multi-rank path except the NCCL exchange
(which needs W GPUs) and checks that the owned ranges tile the rows; it also
checks that caches and graphs built before a re-partition are not reused."""
import numpy as np
import pytest

from synth import CONFIGS, make_config, random_dd
from synth.geometry import Geometry

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ddm():
    import torch
    import paper_1812_05087_b200 as D
    ctx = D.Context(0)
    return D, ctx, torch


def _rows_by_rank(D, ctx, torch, tree, run, worlds=(2, 3, 5)):
    """run() -> device result [n, c]; compares each rank's owned rows with the
    unpartitioned run, bitwise."""
    full = run().cpu().numpy()
    perm = tree.export("PERM")
    for world in worlds:
        covered = np.zeros(tree.n, bool)
        for rank in range(world):
            tree.partition(rank, world)
            lo, hi = tree.counts["OWNED_LO"], tree.counts["OWNED_HI"]
            y = run().cpu().numpy()
            rows = perm[lo:hi]
            assert np.array_equal(y[rows], full[rows]), (world, rank)
            assert not covered[rows].any()
            covered[rows] = True
        assert covered.all(), world
    tree.partition(0, 1)
    assert np.array_equal(run().cpu().numpy(), full)


def test_partition_elastic_fmm(ddm):
    D, ctx, torch = ddm
    g = make_config(2)
    c = CONFIGS[2]
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=20)
    mat = D.material_from_dict(c["material"])
    x = f(random_dd(g.n, 2, 9))

    def run():
        y = torch.full_like(x, float("nan"))
        for _ in range(2):   # the second call replays a captured graph
            D.matvec(ctx, tree, mat, x, y)
        return y

    _rows_by_rank(D, ctx, torch, tree, run)
    tree.free()


def test_partition_poro_cached_and_history(ddm):
    D, ctx, torch = ddm
    g4 = make_config(4)
    keep = g4.frac_id < 10
    g = Geometry(g4.xc[keep], g4.yc[keep], g4.half_len[keep], g4.beta[keep], g4.frac_id[keep],
                 g4.tips[:10])
    c = CONFIGS[4]
    m = c["material"]
    dt = c["dt"]
    M = 2 * m["G"] * (m["nu_u"] - m["nu"]) / (m["alpha"] ** 2 * (1 - 2 * m["nu_u"]) * (1 - 2 * m["nu"]))
    S = m["alpha"] ** 2 * (1 - 2 * m["nu"]) / (2 * m["G"] * (1 - m["nu"])) + 1 / M
    rc = (160 * m["kappa"] / S * 5 * dt) ** 0.5 + 2 * float(g.half_len.max())
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=16, order_p=28,
                  min_leaf_side=rc)
    mat = D.material_from_dict(m)
    x = f(random_dd(g.n, 3, 10))
    Dh = torch.stack([f(random_dd(g.n, 3, 20 + k)) for k in range(4)])

    def run_mv():
        y = torch.full_like(x, float("nan"))
        for _ in range(3):   # on the fly, build the near cache, cached
            D.matvec(ctx, tree, mat, x, y, elapsed=dt)
        return y

    def run_hist():
        r = None
        for h in (2, 3, 4):   # on the fly, build lags, cached
            r = D.history_apply(ctx, tree, mat, dt, Dh[:h].contiguous())
        return r

    _rows_by_rank(D, ctx, torch, tree, run_mv, worlds=(2, 3))
    _rows_by_rank(D, ctx, torch, tree, run_hist, worlds=(2, 3))
    tree.free()


def _sim_case(D, ctx, torch, g, leaf, p, worlds, seed):
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    args = (f(g.xc), f(g.yc), f(g.half_len), f(g.beta))
    mat = D.material(0, 8e9, 0.25)
    x = f(random_dd(g.n, 2, seed))
    ref_tree = D.Tree(ctx, *args, leaf_size=leaf, order_p=p)
    ref = D.matvec(ctx, ref_tree, mat, x).cpu().numpy()
    ref_tree.free()
    for world in worlds:
        trees = [D.Tree(ctx, *args, leaf_size=leaf, order_p=p) for _ in range(world)]
        for r, t in enumerate(trees):
            t.partition(r, world)
        y = D.matvec_sim(ctx, trees, mat, x).cpu().numpy()
        assert np.array_equal(y, ref), world
        for t in trees:
            t.free()


@pytest.mark.parametrize("cfg", [2, 4])
def test_sharded_upward_pass_emulated(ddm, cfg):
    """The sharded multi-rank matvec (P2M of each rank's leaves,
    M2M of its complete cells, multipole all-gather -- played here by device
    copies between the ranks' trees --, M2M of the straddling cells, downward
    pass and assembly of the owned rows) equals the unpartitioned matvec
    bitwise for W = 1, 2, 3, 5, 8."""
    D, ctx, torch = ddm
    g = make_config(cfg)
    _sim_case(D, ctx, torch, g, CONFIGS[cfg]["leaf"], 20, (1, 2, 3, 5, 8), 30 + cfg)


def test_sharded_upward_pass_emulated_cfg5_cut(ddm):
    # a 100 000-element cut of config 5 (leaf 64, p 20: the headline tree's
    # shape, deep enough for straddling cells at many levels), W = 2 and 8
    D, ctx, torch = ddm
    g5 = make_config(5)
    keep = g5.frac_id < 1000
    g = Geometry(g5.xc[keep], g5.yc[keep], g5.half_len[keep], g5.beta[keep], g5.frac_id[keep],
                 g5.tips[:1000])
    _sim_case(D, ctx, torch, g, 64, 20, (2, 8), 55)


def test_sharded_emulated_with_x_lists(ddm, monkeypatch):
    """The same bitwise equality with X lists on (DDM_X_MIN = 8, SURVEY §8f
    f3): each rank runs the P2L of its own leaves, its M2L adds the series of
    the leaves in its cell list, and its near field reads U minus X."""
    D, ctx, torch = ddm
    monkeypatch.setenv("DDM_X_MIN", "8")
    g = make_config(2)
    _sim_case(D, ctx, torch, g, 16, 20, (1, 2, 5), 77)
