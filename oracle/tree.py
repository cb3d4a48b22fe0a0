"""ORACLE (test infrastructure only) — quad-tree and interaction lists.

Plain pointer quad-tree built by recursive insertion, with lists found by
brute-force classification of cell pairs.  Follows PAPER.md §3.1:

* root "square that covers the entire domain"; "any square that
  has more points than a prescribed number is recursively divided into 4
  child squares"; empty children are zero cells and are not
  created;
* child indexing "increases from left to right and from bottom to top"
  (P:593-597): slot = 1 + xbit + 2*ybit, i.e. Morton order with x in bit 0;
* neighbours share at least one vertex; the interaction list
  holds cells "not neighbors at the same level, but their parents are
  neighbors".

Exact readings (R5/R8):
  quantisation  x_min, y_min = min centre; W = max extent (1 if 0);
                s = 2^L / W (one IEEE division), L = 30;
                ix = floor((x - x_min) * s) (one subtract, one multiply,
                never fused), clamped to [0, 2^L - 1]; iy likewise.
  key           bit-interleave of (ix, iy), x in bit 0 (bit loop here).
  order         stable sort by key: equal keys keep input order.
  cells         root exists; a level-l cell exists iff non-empty and its
                parent holds more than `leaf` elements; leaf = cell with
                <= leaf elements or at the depth cap L_max.
  V(b)          existing same-level a with parent(a) adjacent-or-equal to
                parent(b) and a not adjacent-or-equal to b (levels >= 2).
  U(B), leaf B  leaves A whose ancestors at level min(lev A, lev B) are
                adjacent-or-equal (includes B), minus the leaves below a W(B)
                cell and (x_min > 0) the leaves of X(B).
  W(B), leaf B  (w_min > 0) cells D deeper than B whose
                ancestor at B's level is adjacent-or-equal to B, with D not
                touching B (closed boxes disjoint), every ancestor of D below
                B's level touching B, and count(D) >= w_min: D's multipole is
                evaluated at B's targets (M2P).  A non-touching D with fewer
                than w_min elements stays in U (P2P is cheaper).
  X(B), leaf B  (x_min > 0, the dual of W) leaves A coarser
                than B and adjacent-or-equal to B's ancestor at A's level
                (so (A, B) is a U pair), with A not
                touching B, when count(B) >= x_min: A's elements are expanded
                into B's local series (P2L) instead of evaluated at each of
                B's targets.
Cell numbering is canonical: level-major, Morton prefix order within a level.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

L_BITS = 30


class GeometryError(ValueError):
    pass


def quantise(xc: np.ndarray, yc: np.ndarray, L: int = L_BITS):
    """Integer coordinates ix, iy and root parameters (x_min, y_min, W)."""
    if not (np.all(np.isfinite(xc)) and np.all(np.isfinite(yc))):
        raise GeometryError("non-finite coordinates")
    x_min = float(np.min(xc))
    y_min = float(np.min(yc))
    W = max(float(np.max(xc)) - x_min, float(np.max(yc)) - y_min)
    if W == 0.0:
        W = 1.0
    s = float(2 ** L) / W
    top = 2 ** L - 1
    # numpy evaluates these as separate IEEE subtract and multiply (no fusion)
    fx = np.subtract(xc.astype(np.float64), x_min)
    fx = np.multiply(fx, s)
    fy = np.subtract(yc.astype(np.float64), y_min)
    fy = np.multiply(fy, s)
    ix = np.clip(np.floor(fx), 0, top).astype(np.int64)
    iy = np.clip(np.floor(fy), 0, top).astype(np.int64)
    return ix, iy, x_min, y_min, W


def morton_key(ix, iy, L: int = L_BITS):
    """Interleave by an explicit bit loop: bit b of ix -> bit 2b, of iy -> 2b+1.
    Works on Python ints and on numpy integer arrays."""
    if isinstance(ix, np.ndarray):
        ix = ix.astype(np.uint64)
        iy = iy.astype(np.uint64)
        k = np.zeros(ix.shape, dtype=np.uint64)
        one = np.uint64(1)
        for b in range(L):
            k |= ((ix >> np.uint64(b)) & one) << np.uint64(2 * b)
            k |= ((iy >> np.uint64(b)) & one) << np.uint64(2 * b + 1)
        return k
    k = 0
    for b in range(L):
        k |= ((ix >> b) & 1) << (2 * b)
        k |= ((iy >> b) & 1) << (2 * b + 1)
    return k


@dataclass
class Cell:
    level: int
    ix: int                   # level-l integer coordinates
    iy: int
    points: np.ndarray        # input indices of the points in the cell
    parent: "Cell | None"
    children: list
    leaf: bool = False
    index: int = -1


@dataclass
class OracleTree:
    keys: np.ndarray          # [N] u64 Morton keys, input order
    perm: np.ndarray          # [N] sorted position -> input index
    x_min: float
    y_min: float
    W: float
    level: np.ndarray         # per cell (canonical numbering)
    ix: np.ndarray
    iy: np.ndarray
    start: np.ndarray         # first sorted position
    count: np.ndarray
    parent: np.ndarray        # -1 for the root
    first_child: np.ndarray   # -1 if none
    n_child: np.ndarray
    is_leaf: np.ndarray
    cells: list               # Cell objects, canonical order

    @property
    def n_cells(self):
        return len(self.cells)

    def leaves(self) -> np.ndarray:
        return np.nonzero(self.is_leaf)[0]


def build_tree(xc, yc, leaf: int, min_leaf_side: float = 0.0, L: int = L_BITS) -> OracleTree:
    if xc.size < 1 or leaf < 1:
        raise ValueError("need n >= 1 and leaf >= 1")
    ix, iy, x_min, y_min, W = quantise(xc, yc, L)
    keys = morton_key(ix, iy, L)
    perm = np.argsort(keys, kind="stable")
    L_max = L
    if min_leaf_side > 0.0:
        L_max = min(L, int(np.floor(np.log2(W / min_leaf_side))))
        L_max = max(L_max, 0)

    root = Cell(0, 0, 0, np.arange(xc.size), None, [])

    def split(c: Cell):
        if len(c.points) <= leaf or c.level >= L_max:
            if len(c.points) > leaf and c.level >= L:
                raise GeometryError("more than `leaf` coincident points at the depth cap")
            c.leaf = True
            return
        sh = L - c.level - 1
        pts = c.points                           # insertion by the next bit
        slot = ((ix[pts] >> sh) & 1) + 2 * ((iy[pts] >> sh) & 1)
        for q in range(4):                       # slot order = paper's 1..4 order
            sub = pts[slot == q]
            if sub.size:
                ch = Cell(c.level + 1, 2 * c.ix + (q & 1), 2 * c.iy + (q >> 1), sub, c, [])
                c.children.append(ch)
        for ch in c.children:
            split(ch)

    split(root)

    # canonical numbering: level-major, Morton prefix within a level
    levels = {}
    stack = [root]
    while stack:
        c = stack.pop()
        levels.setdefault(c.level, []).append(c)
        stack.extend(c.children)
    cells = []
    for lev in sorted(levels):
        cells.extend(sorted(levels[lev], key=lambda c: morton_key(c.ix, c.iy, L)))
    for i, c in enumerate(cells):
        c.index = i
    rank = np.empty(xc.size, dtype=np.int64)
    rank[perm] = np.arange(xc.size)
    nc = len(cells)
    t = OracleTree(keys, perm, x_min, y_min, W,
                   np.array([c.level for c in cells]), np.array([c.ix for c in cells]),
                   np.array([c.iy for c in cells]),
                   np.array([int(rank[c.points].min()) for c in cells]),
                   np.array([len(c.points) for c in cells]),
                   np.array([c.parent.index if c.parent else -1 for c in cells]),
                   np.array([c.children[0].index if c.children else -1 for c in cells]),
                   np.array([len(c.children) for c in cells]),
                   np.array([c.leaf for c in cells]), cells)
    assert t.count.sum() >= xc.size and nc >= 1
    return t


def adjacent_or_equal(a: Cell, b: Cell) -> bool:
    """Same level; share at least one vertex or are the same cell."""
    assert a.level == b.level
    return abs(a.ix - b.ix) <= 1 and abs(a.iy - b.iy) <= 1


def ancestor(c: Cell, level: int) -> Cell:
    while c.level > level:
        c = c.parent
    return c


def v_lists(t: OracleTree, targets=None) -> dict:
    """Brute force V(b) for each target cell b (all cells by default):
    sorted list of canonical source-cell indices."""
    by_level = {}
    for c in t.cells:
        by_level.setdefault(c.level, []).append(c)
    out = {}
    tg = t.cells if targets is None else [t.cells[i] for i in targets]
    for b in tg:
        lst = []
        if b.level >= 2:
            for a in by_level[b.level]:
                if adjacent_or_equal(a.parent, b.parent) and not adjacent_or_equal(a, b):
                    lst.append(a.index)
        out[b.index] = sorted(lst)
    return out


def touching(a: Cell, b: Cell) -> bool:
    """Closed boxes of cells at any levels intersect (share a point)."""
    if a.level > b.level:
        a, b = b, a
    sh = b.level - a.level                 # b is the finer cell
    lo_x, hi_x = a.ix << sh, (a.ix + 1) << sh
    lo_y, hi_y = a.iy << sh, (a.iy + 1) << sh
    return (lo_x <= b.ix + 1 and b.ix <= hi_x) and (lo_y <= b.iy + 1 and b.iy <= hi_y)


def w_lists(t: OracleTree, w_min: int, targets=None) -> dict:
    """Brute force W(B) for each target leaf B: sorted canonical cell indices
    (definition in the module docstring; empty when w_min <= 0)."""
    leaves = [c for c in t.cells if c.leaf]
    tg = leaves if targets is None else [t.cells[i] for i in targets]
    by_level = {}
    for c in t.cells:
        by_level.setdefault(c.level, []).append(c)
    out = {}
    for B in tg:
        lst = []
        if w_min > 0:
            # candidates: the cells whose ancestor at B's level is adjacent-or-equal
            # to B, i.e. the proper descendants of those cells; test each one
            for Q in by_level[B.level]:
                if not adjacent_or_equal(Q, B):
                    continue
                stack = list(Q.children)
                while stack:
                    D = stack.pop()
                    stack.extend(D.children)
                    if len(D.points) < w_min or touching(D, B):
                        continue
                    E, ok = D.parent, True
                    while E.level > B.level:
                        ok = ok and touching(E, B)
                        E = E.parent
                    if ok:
                        lst.append(D.index)
        out[B.index] = sorted(lst)
    return out


def x_lists(t: OracleTree, x_min: int, targets=None) -> dict:
    """Brute force X(B) for each target leaf B: sorted canonical indices of
    the coarser, non-touching U-pair leaves (definition in the module
    docstring; empty when x_min <= 0 or count(B) < x_min)."""
    leaves = [c for c in t.cells if c.leaf]
    tg = leaves if targets is None else [t.cells[i] for i in targets]
    out = {}
    for B in tg:
        lst = []
        if x_min > 0 and len(B.points) >= x_min:
            for A in leaves:
                if (A.level < B.level and adjacent_or_equal(A, ancestor(B, A.level))
                        and not touching(A, B)):
                    lst.append(A.index)
        out[B.index] = sorted(lst)
    return out


def u_lists(t: OracleTree, targets=None, w_min: int = 0, x_min: int = 0) -> dict:
    """Brute force U(B) for each target leaf B: sorted canonical leaf indices
    (w_min > 0: without the leaves below a W(B) cell; x_min > 0: without the
    leaves of X(B))."""
    leaves = [c for c in t.cells if c.leaf]
    tg = leaves if targets is None else [t.cells[i] for i in targets]
    W = w_lists(t, w_min, [B.index for B in tg]) if w_min > 0 else {}
    X = x_lists(t, x_min, [B.index for B in tg]) if x_min > 0 else {}
    out = {}
    for B in tg:
        wset = set(W.get(B.index, []))
        xset = set(X.get(B.index, []))
        lst = []
        for A in leaves:
            m = min(A.level, B.level)
            if adjacent_or_equal(ancestor(A, m), ancestor(B, m)):
                c, under_w = A, False
                while c is not None and c.level > B.level:
                    under_w = under_w or c.index in wset
                    c = c.parent
                if not under_w and A.index not in xset:
                    lst.append(A.index)
        out[B.index] = sorted(lst)
    return out


def pair_coverage(t: OracleTree, U: dict, V: dict, W: dict | None = None,
                  X: dict | None = None) -> np.ndarray:
    """For every ordered pair of leaves (B target, A source) count how many
    times it is handled: once by U(B), once by X(B), once per W(B) cell
    above-or-at A, or once per level l where anc_l(A) in V(anc_l(B)).  The
    partition property requires all ones."""
    leaves = [c for c in t.cells if c.leaf]
    Vs = {k: set(v) for k, v in V.items()}
    cnt = np.zeros((len(leaves), len(leaves)), dtype=np.int64)
    for i, B in enumerate(leaves):
        uset = set(U[B.index])
        wset = set(W[B.index]) if W is not None else set()
        for j, A in enumerate(leaves):
            n = 1 if A.index in uset else 0
            n += 1 if X is not None and A.index in X[B.index] else 0
            c = A
            while c is not None:
                n += 1 if c.index in wset else 0
                c = c.parent
            for lev in range(2, min(A.level, B.level) + 1):
                if ancestor(A, lev).index in Vs[ancestor(B, lev).index]:
                    n += 1
            cnt[i, j] = n
    return cnt
