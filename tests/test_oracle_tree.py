"""Pins of the quad-tree / list oracle.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import tree as T
from synth import make_config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_morton_bit_interleave():
    assert T.morton_key(1, 0) == 1 and T.morton_key(0, 1) == 2 and T.morton_key(3, 3) == 15
    assert T.morton_key(2 ** 29, 0) == 2 ** 58 and T.morton_key(0, 2 ** 29) == 2 ** 59
    a = np.array([5, 1023, 2 ** 30 - 1])
    b = np.array([9, 0, 2 ** 30 - 1])
    k = T.morton_key(a, b)
    assert [int(v) for v in k] == [T.morton_key(int(x), int(y)) for x, y in zip(a, b)]
    assert int(k[2]) == 2 ** 60 - 1


def test_single_point_is_single_leaf():
    t = T.build_tree(np.array([3.0]), np.array([-1.0]), leaf=1)
    assert t.n_cells == 1 and t.is_leaf[0] and t.count[0] == 1


def test_four_quadrants_depth_one_and_child_order():
    # points listed top-right first; the paper numbers children left->right,
    # bottom->top (child 1 = bottom-left, child 4 = top-right)
    xs = np.array([0.9, 0.1, 0.9, 0.1])
    ys = np.array([0.9, 0.1, 0.1, 0.9])
    t = T.build_tree(xs, ys, leaf=1)
    assert t.n_cells == 5 and t.level.max() == 1 and t.is_leaf[1:].all()
    order = [int(t.perm[t.start[c]]) for c in range(1, 5)]
    gold = GOLD["child_index_convention"]
    assert order[gold["bottom_left"] - 1] == 1      # (0.1, 0.1)
    assert order[gold["top_right"] - 1] == 0        # (0.9, 0.9)
    assert order == [1, 2, 3, 0]                    # BL, BR, TL, TR


def _uniform(level):
    m = 2 ** level
    g = (np.arange(m) + 0.5) / m
    X, Y = np.meshgrid(g, g)
    return T.build_tree(X.ravel(), Y.ravel(), leaf=1)


def test_uniform_grid_list_counts():
    gold = GOLD["uniform_grid_counts"]
    t = _uniform(3)
    assert (t.level == 3).sum() == 64 and t.is_leaf[t.level == 3].all()
    V = T.v_lists(t)

    def cell(lev, i, j):
        return next(c for c in t.cells if c.level == lev and c.ix == i and c.iy == j)

    assert len(V[cell(2, 1, 1).index]) == gold["level2_interior_V"]
    assert len(V[cell(2, 0, 0).index]) == gold["level2_corner_V"]
    assert len(V[cell(3, 3, 3).index]) == gold["level3_interior_V"]
    assert len(V[cell(3, 0, 0).index]) == gold["level3_corner_V"]
    lvl2 = [c for c in t.cells if c.level == 2]
    nb = lambda c: sum(T.adjacent_or_equal(c, o) for o in lvl2) - 1
    assert nb(cell(2, 1, 1)) == gold["level2_interior_neighbours"]
    assert nb(cell(2, 0, 0)) == gold["level2_corner_neighbours"]
    offs = set()
    for b, lst in V.items():
        for a in lst:
            offs.add((t.ix[a] - t.ix[b], t.iy[a] - t.iy[b]))
    assert len(offs) == gold["n_offsets"]
    assert all(max(abs(dx), abs(dy)) in (2, 3) for dx, dy in offs)


def _random_points(rng, n):
    kind = rng.integers(3)
    if kind == 0:
        return rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    if kind == 1:                                  # clustered
        c = rng.uniform(0, 1, (4, 2))
        k = rng.integers(4, size=n)
        return c[k, 0] + 0.02 * rng.normal(size=n), c[k, 1] + 0.02 * rng.normal(size=n)
    t = rng.uniform(0, 1, n)                       # points on lines (fracture-like)
    return t, 0.3 * t + 0.001 * rng.integers(3, size=n)


def test_pair_coverage_on_random_trees():
    rng = np.random.default_rng(11)
    for trial in range(50):
        n = int(rng.integers(1, 160))
        x, y = _random_points(rng, n)
        leaf = int(rng.integers(1, 9))
        t = T.build_tree(x, y, leaf)
        U, V = T.u_lists(t), T.v_lists(t)
        cov = T.pair_coverage(t, U, V)
        assert (cov == 1).all(), trial
        # the W split (M2P cells) keeps the partition property
        wm = int(rng.integers(1, 4))
        Uw, Ww = T.u_lists(t, w_min=wm), T.w_lists(t, wm)
        assert (T.pair_coverage(t, Uw, V, Ww) == 1).all(), (trial, wm)
        for b, lst in Ww.items():   # W cells never touch their target leaf
            for d in lst:
                assert not T.touching(t.cells[d], t.cells[b])
        # the X split (P2L leaves) with it: still every pair exactly once; X
        # leaves are coarser than, and do not touch, their target leaf, which
        # holds >= x_min elements; X(B) is exactly the coarser non-touching
        # part of the unsplit U(B)
        xm = int(rng.integers(1, 4))
        Ux, Xx = T.u_lists(t, w_min=wm, x_min=xm), T.x_lists(t, xm)
        assert (T.pair_coverage(t, Ux, V, Ww, Xx) == 1).all(), (trial, wm, xm)
        for b, lst in Xx.items():
            B = t.cells[b]
            assert not lst or t.count[b] >= xm
            expect = [a for a in Uw[b] if t.cells[a].level < B.level
                      and not T.touching(t.cells[a], B)] if t.count[b] >= xm else []
            assert lst == expect, (trial, b)
            assert sorted(Ux[b] + lst) == Uw[b]
        # every element sits in exactly one leaf; leaves hold <= leaf points
        assert t.count[t.is_leaf].sum() == n
        assert (t.count[t.is_leaf] <= leaf).all()
        # U is symmetric
        for b, lst in U.items():
            for a in lst:
                assert b in U[a]


def test_depth_cap_and_coincident_points():
    x = np.array([0.5, 0.5, 0.5, 0.0, 1.0])
    y = np.array([0.5, 0.5, 0.5, 0.0, 1.0])
    with pytest.raises(T.GeometryError):
        T.build_tree(x, y, leaf=2)
    t = T.build_tree(x, y, leaf=2, min_leaf_side=0.3)   # cap: side >= 0.3 -> L_max = 1
    assert t.level.max() == 1
    with pytest.raises(T.GeometryError):
        T.build_tree(np.array([np.nan]), np.array([0.0]), leaf=1)


def test_config2_sizes():
    g = make_config(2)
    t = T.build_tree(g.xc, g.yc, 32)
    U, V = T.u_lists(t), T.v_lists(t)
    near = sum(int(t.count[b]) * sum(int(t.count[a]) for a in U[b]) for b in U)
    assert (t.n_cells, int(t.is_leaf.sum())) == (195, 140)
    assert sum(len(v) for v in V.values()) == 2124 and near == 327618
    assert (T.pair_coverage(t, U, V) == 1).all()
