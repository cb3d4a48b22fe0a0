"""ORACLE (test infrastructure only) — time marching with the direct history sum.

Eq.(final_sigs)-(final_pp): at step h the current-step system is
solved after subtracting the influence of all previous steps' solutions,
    A^(0) D^h = b_h - sum_{eta=0}^{h-1} A^{h-eta} D^eta .
Reading R10: constant temporal elements, each D^eta held over
its step; kernels depend only on the lag, with the continuous-source kernel
K(tau) of oracle/poro.py:
    A^(0) = K(dt),   A^(m) = K((m+1) dt) - K(m dt)   (m >= 1).
For an elastic material K is independent of tau and every A^(m>=1) vanishes.
"""
from __future__ import annotations

import numpy as np

from . import elastic as E
from . import poro as P


def lag_matrix(geom, mat, dt, m):
    """A^(m) as a dense 3N x 3N matrix (ABI convention)."""
    if mat["kind"] == 0:
        if m == 0:
            A2 = E.assemble_dense(geom, mat["G"], mat["nu"])
            A = np.zeros((3 * geom.n, 3 * geom.n))
            for r in (0, 1):
                for c in (0, 1):
                    A[r::3, c::3] = A2[r::2, c::2]
            return A
        return np.zeros((3 * geom.n, 3 * geom.n))
    if m == 0:
        return P.assemble_dense(geom, mat, dt)
    return P.assemble_dense(geom, mat, (m + 1) * dt) - P.assemble_dense(geom, mat, m * dt)


def history_sum(geom, mat, dt, D_hist, lags=None):
    """r_h = sum_{m=1}^{h} A^(m) D^(h-m); D_hist [h, N, 3] (D^0 .. D^(h-1)).
    `lags` may pass precomputed A^(m) (list indexed by m)."""
    h = D_hist.shape[0]
    r = np.zeros(3 * geom.n)
    for m in range(1, h + 1):
        A = lags[m] if lags is not None else lag_matrix(geom, mat, dt, m)
        r += A @ D_hist[h - m].reshape(-1)
    return r.reshape(geom.n, 3)


def march(geom, mat, dt, b, steps, solve=np.linalg.solve, lags=None):
    """Direct time marching with a constant right-hand side b [N, 3]:
    returns D [steps, N, 3].  Step h solves A^(0) D^h = b - r_h.
    `lags` may pass the lag matrices A^(0..steps) (tests drive the recurrence
    with synthetic lags whose solution has a closed form)."""
    if lags is None:
        lags = [lag_matrix(geom, mat, dt, m) for m in range(steps + 1)]
    D = np.zeros((steps, geom.n, 3))
    for h in range(steps):
        rhs = b.reshape(-1) - history_sum(geom, mat, dt, D[:h], lags).reshape(-1)
        D[h] = solve(lags[0], rhs).reshape(geom.n, 3)
    return D


def poro_rhs(geom, load):
    """Right-hand side with the pore-pressure row (readings P14/P15):
    b = (b_s, b_n, b_p) with b_s, b_n from oracle.elastic.farfield_rhs and
    b_p = p_f - p0 ('absolute' mode) or (sh + p_f) - p0 ('net' mode)."""
    b2 = E.farfield_rhs(geom, load)
    out = np.zeros((geom.n, 3))
    out[:, :2] = b2
    if load["mode"] == "net":
        out[:, 2] = load["sh"] + load["p_f"] - load["p0"]
    else:
        out[:, 2] = load["p_f"] - load["p0"]
    return out
