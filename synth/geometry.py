"""Fracture-network geometry generators (no method arithmetic).

Elements are constant displacement-discontinuity segments (PAPER.md P:389-391,
"constant spatial ... elements", each FMM point is an element
centre).  Every generator returns a `Geometry` in *user order*: fracture-major,
element k of a fracture running from its first endpoint p1 to its second p2.

Recipe: per random candidate draw, in this order,
centre x ~ U[0, L), centre y ~ U[0, L), half-length h ~ U[h_lo, h_hi),
angle theta ~ U[0, pi) (measured from x = SHmax); endpoints c -/+ h(cos, sin).
A candidate that intersects (touching and collinear overlap included) any
accepted fracture is rejected and redrawn.  numpy Generator(PCG64(seed)).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Geometry:
    xc: np.ndarray          # [N] element centre x (m)
    yc: np.ndarray          # [N] element centre y (m)
    half_len: np.ndarray    # [N] element half-length a (m)
    beta: np.ndarray        # [N] element direction angle (rad), in [0, pi)
    frac_id: np.ndarray     # [N] fracture index of each element
    tips: np.ndarray        # [n_frac, 2] element ids of the two tips of each fracture
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.xc.shape[0])


def _discretise(p1: np.ndarray, p2: np.ndarray, theta: np.ndarray, n_el: int) -> Geometry:
    """Split each fracture p1->p2 into n_el equal elements, numbered fracture-major."""
    nf = p1.shape[0]
    k = (np.arange(n_el, dtype=np.float64) + 0.5) / n_el            # [n_el]
    xc = p1[:, None, 0] + k[None, :] * (p2[:, None, 0] - p1[:, None, 0])
    yc = p1[:, None, 1] + k[None, :] * (p2[:, None, 1] - p1[:, None, 1])
    hl = 0.5 * np.hypot(p2[:, 0] - p1[:, 0], p2[:, 1] - p1[:, 1]) / n_el
    half_len = np.repeat(hl, n_el)
    beta = np.repeat(theta, n_el)
    frac_id = np.repeat(np.arange(nf), n_el)
    tips = np.stack([np.arange(nf) * n_el, np.arange(nf) * n_el + n_el - 1], axis=1)
    return Geometry(xc.reshape(-1).copy(), yc.reshape(-1).copy(), half_len, beta,
                    frac_id, tips)


def straight_crack(a: float = 1.0, n_el: int = 200) -> Geometry:
    """Config 1: one crack on [-a, a] along x (BASELINE.json configs[0])."""
    p1 = np.array([[-a, 0.0]])
    p2 = np.array([[a, 0.0]])
    g = _discretise(p1, p2, np.array([0.0]), n_el)
    g.meta = {"kind": "straight", "a": a, "n_el": n_el}
    return g


def parallel_fractures(n_frac: int = 5, half_length: float = 100.0, spacing: float = 20.0,
                       n_el: int = 4000) -> Geometry:
    """Config 3 layout: fractures along x on [-h, h],
    at y = 0, spacing, 2*spacing, ..."""
    ys = spacing * np.arange(n_frac, dtype=np.float64)
    p1 = np.stack([np.full(n_frac, -half_length), ys], axis=1)
    p2 = np.stack([np.full(n_frac, half_length), ys], axis=1)
    g = _discretise(p1, p2, np.zeros(n_frac), n_el)
    g.meta = {"kind": "parallel", "n_frac": n_frac, "half_length": half_length,
              "spacing": spacing, "n_el": n_el}
    return g


def _orient(ax, ay, bx, by, cx, cy):
    return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)


def segments_intersect(p1, p2, q1x, q1y, q2x, q2y) -> np.ndarray:
    """Vectorised closed-segment intersection test of one segment p1p2 against
    arrays of segments q1q2.  Touching and collinear overlap count as
    intersecting."""
    o1 = np.sign(_orient(p1[0], p1[1], p2[0], p2[1], q1x, q1y))
    o2 = np.sign(_orient(p1[0], p1[1], p2[0], p2[1], q2x, q2y))
    o3 = np.sign(_orient(q1x, q1y, q2x, q2y, p1[0], p1[1]))
    o4 = np.sign(_orient(q1x, q1y, q2x, q2y, p2[0], p2[1]))
    general = (o1 * o2 <= 0) & (o3 * o4 <= 0)
    collinear = (o1 == 0) & (o2 == 0)
    # collinear: intersect iff bounding boxes overlap
    bx = (np.minimum(q1x, q2x) <= max(p1[0], p2[0])) & (np.maximum(q1x, q2x) >= min(p1[0], p2[0]))
    by = (np.minimum(q1y, q2y) <= max(p1[1], p2[1])) & (np.maximum(q1y, q2y) >= min(p1[1], p2[1]))
    return np.where(collinear, bx & by, general)


def random_fractures(n_frac: int, n_el: int, box: float, h_lo: float, h_hi: float,
                     seed: int, max_draws: int = 10_000_000) -> Geometry:
    """Random non-intersecting straight fractures (configs 2, 4, 5)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    P1 = np.empty((n_frac, 2))
    P2 = np.empty((n_frac, 2))
    TH = np.empty(n_frac)
    # axis-aligned bounding boxes of accepted fractures for a cheap prefilter
    lo = np.empty((n_frac, 2))
    hi = np.empty((n_frac, 2))
    na = 0
    draws = 0
    while na < n_frac:
        draws += 1
        if draws > max_draws:
            raise RuntimeError("random_fractures: too many rejections")
        cx = rng.uniform(0.0, box)
        cy = rng.uniform(0.0, box)
        h = rng.uniform(h_lo, h_hi)
        th = rng.uniform(0.0, np.pi)
        c, s = np.cos(th), np.sin(th)
        p1 = np.array([cx - h * c, cy - h * s])
        p2 = np.array([cx + h * c, cy + h * s])
        if na:
            blo = np.minimum(p1, p2)
            bhi = np.maximum(p1, p2)
            cand = np.nonzero((lo[:na, 0] <= bhi[0]) & (hi[:na, 0] >= blo[0]) &
                              (lo[:na, 1] <= bhi[1]) & (hi[:na, 1] >= blo[1]))[0]
            if cand.size and segments_intersect(p1, p2, P1[cand, 0], P1[cand, 1],
                                                P2[cand, 0], P2[cand, 1]).any():
                continue
        P1[na], P2[na], TH[na] = p1, p2, th
        lo[na] = np.minimum(p1, p2)
        hi[na] = np.maximum(p1, p2)
        na += 1
    g = _discretise(P1, P2, TH, n_el)
    g.meta = {"kind": "random", "n_frac": n_frac, "n_el": n_el, "box": box,
              "h_lo": h_lo, "h_hi": h_hi, "seed": seed, "draws": draws}
    g.meta["p1"] = P1
    g.meta["p2"] = P2
    return g
