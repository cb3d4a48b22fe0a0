"""ORACLE (test infrastructure only) — fracture propagation loop.

PAPER.md Fig. 8 branch: "After obtaining the solutions, one may
calculate the SIFs mode-I and II using Equation (SIF).  Then, a fracture
propagation criterion may be used to check to see whether the propagation
criterion is satisfied.  Consequently, an element will be added to the model
if propagation happens, and in that case the quad-tree needs to be
constructed again."  The paper names no criterion; reading R23:
the maximum tangential stress criterion (Erdogan & Sih 1963) in the tip's
outward frame (x along the crack, pointing out of it):
  d sigma_thetatheta / d theta = 0:  K_I sin(theta) + K_II (3 cos(theta) - 1) = 0
  theta_c = 2 atan( (K_I - sqrt(K_I^2 + 8 K_II^2)) / (4 K_II) ),  0 if K_II = 0
  K_eq    = cos(theta_c/2) [ K_I cos^2(theta_c/2) - (3/2) K_II sin(theta_c) ]
A tip grows when K_I > 0 and K_eq >= K_IC, by one element of the tip
element's length along (outward angle + theta_c).  Elastic, one temporal
element per step; each step is a dense direct solve (oracle.elastic), so the
loop has no tree: "rebuilding the quad-tree" changes nothing here.
Pins (tests/test_oracle_propagation.py): pure mode I (theta = 0, K_eq =
K_I); pure mode II (theta = -arccos(1/3) = -70.53 deg, K_eq = 2 K_II / sqrt 3);
theta_c is the stationary maximum of the Williams hoop stress on a fine grid
and K_eq = sqrt(2 pi r) sigma_thetatheta(theta_c); K_II -> -K_II mirrors
theta_c; a mode-I tip grows an element on the crack line.
"""
from __future__ import annotations

import numpy as np

from synth.geometry import Geometry

from . import elastic as OE
from . import sif as OS


def mts(KI: float, KII: float):
    """(theta_c, K_eq) of the maximum tangential stress criterion."""
    if KII == 0.0:
        th = 0.0
    else:
        th = 2.0 * np.arctan((KI - np.sqrt(KI * KI + 8.0 * KII * KII)) / (4.0 * KII))
    c = np.cos(0.5 * th)
    return th, c * (KI * c * c - 1.5 * KII * np.sin(th))


def sigma_thetatheta(KI: float, KII: float, th: float, r: float = 1.0) -> float:
    """Near-tip hoop stress (Williams leading term), for the pins."""
    c = np.cos(0.5 * th)
    return (c / np.sqrt(2 * np.pi * r)) * (KI * c * c - 1.5 * KII * np.sin(th))


def grow_tip(x, y, a, beta, end, th):
    """New element at a tip: the tip point is the element's end
    (end 1: + a e^{i beta}), direction = outward angle + theta."""
    sg = 1.0 if end else -1.0
    ex, ey = x + sg * a * np.cos(beta), y + sg * a * np.sin(beta)
    phi = (beta if end else beta + np.pi) + th
    phi = np.mod(phi, 2 * np.pi)
    nx, ny = ex + a * np.cos(phi), ey + a * np.sin(phi)
    if phi < np.pi:
        return nx, ny, a, phi, 1
    return nx, ny, a, phi - np.pi, 0


def propagate(xc, yc, a, beta, tips, G, nu, load, K_IC, steps):
    """The Fig. 8 propagation loop, dense.  tips: list of (element, end).
    Returns (xc, yc, a, beta, tips, history) like the GPU driver."""
    xc, yc, a, beta = (np.array(v, dtype=np.float64) for v in (xc, yc, a, beta))
    tips = [tuple(t) for t in tips]
    E = 2.0 * G * (1.0 + nu)
    hist = []
    for _ in range(steps):
        n = xc.size
        g = Geometry(xc, yc, a, beta, np.zeros(n, int), np.zeros((1, 2), int))
        A = OE.assemble_dense(g, G, nu)
        b = OE.farfield_rhs(g, dict(load, mode="absolute"))
        D = np.linalg.solve(A, b.reshape(-1)).reshape(n, 2)
        ti = np.array([t[0] for t in tips])
        KI, KII = OS.sif(D[ti, 1], D[ti, 0], a[ti], E, nu)
        grow, new = [], []
        for k, (e, end) in enumerate(tips):
            th, keq = mts(KI[k], KII[k])
            gr = bool(KI[k] > 0.0 and keq >= K_IC)
            grow.append(int(gr))
            if gr:
                new.append((k, grow_tip(xc[e], yc[e], a[e], beta[e], end, th)))
        hist.append({"n": n, "KI": KI.tolist(), "KII": KII.tolist(), "grow": grow})
        if not new:
            break
        for k, (nx, ny, na, nb, ne) in new:
            xc = np.append(xc, nx)
            yc = np.append(yc, ny)
            a = np.append(a, na)
            beta = np.append(beta, nb)
            tips[k] = (xc.size - 1, ne)
    return xc, yc, a, beta, tips, hist
