"""ORACLE (test infrastructure only) — the paper's black-box FMM (bbFMM) for the
elastic DDM matvec, step by step (§3.2).

The paper approximates the kernel by Chebyshev interpolation in both arguments
(Eq.(low_rank), S_n of P:738-749) and evaluates the far field in the
stages of Eq.(fmm_2d)/(fastsum_cheb):
  P2M ("P2L", Eq.(p2l))  W_m^I   = sum_j b(y_j) S_n(ybar_m^I, y_j)
  M2M (Eq.(m2m))          W_m^I   = sum_{children J} sum_m' W_m'^J S_n(ybar_m^I, ybar_m'^J)
  M2L (Eq.(m2l))          g_l^I   = sum_{J in V(I)} sum_m K(xbar_l^I, ybar_m^J) W_m^J
  L2L (Eq.(l2l))          f_l^I   = g_l^I + sum_l' f_l'^parent S_n(xbar_l'^parent, xbar_l^I)
  L2P + P2P              f(x)    = sum_l f_l^leaf S_n(xbar_l, x) + exact near field
with S_n(xbar, x) = 1/n + (2/n) sum_{k=1}^{n-1} T_k(xbar) T_k(x) on [-1, 1],
Chebyshev nodes xbar_l = cos((2l - 1) pi / (2n)), and 2D cardinal functions as
products of the 1D ones in cell-normalised coordinates.

Kernel (reading R21): the constant-DD element in
Kolosov–Muskhelishvili form (as the GPU P2P) written as line
integrals of analytic point kernels k2 = (z - zeta)^-2, k3 = (z - zeta)^-3:
  Phi(z)   = sum_j int rho1_j k2 ds,      rho1 = i G C B e,   B = (D_s + i D_n) e
  Phi'(z)  = -2 sum_j int rho1_j k3 ds
  Psi(z)   = sum_j int [rho2_j k2 + rho3_j(s) k3] ds,  rho2 = i G C Q e,
             rho3 = 2 i G C B e conj(zeta(s)),  Q = conj(e)^2 B - conj(B)
  traction T = sigma_n + i sigma_s = 2 Re Phi + e^{2 i b_t} (conj(z) Phi' + Psi)
(the identity conj(zc) + r (z - zc) = conj(zeta) + r (z - zeta) on the element
turns the closed-form Psi of App. A.2 into this integral).  The three
densities are the "b(y)" of Eq.(p2l); the segment integral of S_n times a
density is done by n-point Gauss–Legendre along the element (exact: the
integrand is a polynomial of degree <= 2n - 1 in s).  Psi is carried about
each cell's centre c (Psi~ = Psi + conj(c) Phi', the rho3 density taken
relative to conj(c)), so only cell offsets enter the translations.

Tree and lists are oracle/tree.py's (U, V, and W: a W cell's node weights are
evaluated directly at the targets, the node-to-point form of Eq.(m2l)).
"""
from __future__ import annotations

import numpy as np

from . import tree as T


def cheb_nodes(n: int) -> np.ndarray:
    """xbar_l = cos((2l - 1) pi / (2n)), l = 1..n."""
    return np.cos((2.0 * np.arange(1, n + 1) - 1.0) * np.pi / (2.0 * n))


def cardinal(n: int, xbar: np.ndarray, x: np.ndarray) -> np.ndarray:
    """S_n(xbar_l, x) for every node l and point x: [len(xbar), len(x)]."""
    xbar = np.asarray(xbar, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    out = np.full((xbar.size, x.size), 1.0 / n)
    Ta_prev, Ta = np.ones_like(xbar), xbar.copy()
    Tb_prev, Tb = np.ones_like(x), x.copy()
    for k in range(1, n):
        out += (2.0 / n) * np.outer(Ta, Tb)
        Ta_prev, Ta = Ta, 2.0 * xbar * Ta - Ta_prev
        Tb_prev, Tb = Tb, 2.0 * x * Tb - Tb_prev
    return out


def _cell_geom(t: T.OracleTree, c: int):
    s = t.W / 2.0 ** t.level[c]
    cx = t.x_min + (t.ix[c] + 0.5) * s
    cy = t.y_min + (t.iy[c] + 0.5) * s
    return complex(cx, cy), s


def _nodes(t, c, n):
    """2D Chebyshev nodes of cell c, index m = i * n + k (x-node i, y-node k)."""
    cz, s = _cell_geom(t, c)
    xb = cheb_nodes(n)
    X, Y = np.meshgrid(xb, xb, indexing="ij")
    return cz + 0.5 * s * (X.ravel() + 1j * Y.ravel())


def _interp2(t, c, n, pts):
    """2D cardinal functions S(ybar_m^c, p) for the points p: [n*n, len(p)]."""
    cz, s = _cell_geom(t, c)
    xi = (pts.real - cz.real) / (0.5 * s)
    eta = (pts.imag - cz.imag) / (0.5 * s)
    xb = cheb_nodes(n)
    Sx = cardinal(n, xb, xi)
    Sy = cardinal(n, xb, eta)
    return (Sx[:, None, :] * Sy[None, :, :]).reshape(n * n, -1)


def bbfmm_matvec(geom, G: float, nu: float, D: np.ndarray, leaf: int, n: int,
                 w_min: int = 24) -> np.ndarray:
    """y = A D for the elastic DDM, far field by bbFMM with n Chebyshev nodes
    per dimension, near field exact (U lists), W cells node-to-point.
    D [N, 2] (s, n), returns [N, 2] (sigma_s, sigma_n) in user order."""
    C = 1.0 / (4.0 * np.pi * (1.0 - nu))
    gc = G * C
    t = T.build_tree(geom.xc, geom.yc, leaf)
    ncell = t.n_cells
    zc = geom.xc + 1j * geom.yc
    e = np.exp(1j * geom.beta)
    a = geom.half_len
    B = (D[:, 0] + 1j * D[:, 1]) * e
    Q = np.conj(e) ** 2 * B - np.conj(B)
    rho1 = 1j * gc * B * e
    rho2 = 1j * gc * Q * e
    gl_x, gl_w = np.polynomial.legendre.leggauss(n)
    perm = t.perm                         # sorted position -> user index
    nn = n * n
    # ---- P2M (Eq.(p2l)): node weights w1, w2, w3 (w3 relative to the cell centre)
    W = np.zeros((ncell, 3, nn), dtype=complex)
    for c in np.nonzero(t.is_leaf)[0]:
        cz, s = _cell_geom(t, c)
        for pos in range(t.start[c], t.start[c] + t.count[c]):
            j = perm[pos]
            zeta = zc[j] + gl_x * a[j] * e[j]            # GL points along the element
            wts = gl_w * a[j]                            # ds = a dt
            S = _interp2(t, c, n, zeta)                  # [nn, n]
            W[c, 0] += S @ (wts * rho1[j])
            W[c, 1] += S @ (wts * rho2[j])
            W[c, 2] += S @ (wts * 2j * gc * B[j] * e[j] * np.conj(zeta - cz))
    # ---- M2M (Eq.(m2m)): deepest level first; w3 re-centred on the parent
    for lev in range(int(t.level.max()) - 1, -1, -1):
        for c in np.nonzero((t.level == lev) & ~t.is_leaf)[0]:
            cz, _ = _cell_geom(t, c)
            for q in range(t.first_child[c], t.first_child[c] + t.n_child[c]):
                qz, _ = _cell_geom(t, q)
                S = _interp2(t, c, n, _nodes(t, q, n))   # [nn parent, nn child]
                W[c, 0] += S @ W[q, 0]
                W[c, 1] += S @ W[q, 1]
                W[c, 2] += S @ (W[q, 2] + 2.0 * np.conj(qz - cz) * W[q, 0])
    # ---- M2L (Eq.(m2l)) at the target nodes: Phi, Phi', Psi~ (about the target centre)
    V = T.v_lists(t)
    F = np.zeros((ncell, 3, nn), dtype=complex)
    for c in range(ncell):
        if not V[c]:
            continue
        cz, _ = _cell_geom(t, c)
        xn = _nodes(t, c, n)
        for b in V[c]:
            bz, _ = _cell_geom(t, b)
            d = xn[:, None] - _nodes(t, b, n)[None, :]
            k2 = 1.0 / d ** 2
            k3 = 1.0 / d ** 3
            F[c, 0] += k2 @ W[b, 0]
            F[c, 1] += -2.0 * (k3 @ W[b, 0])
            F[c, 2] += k2 @ W[b, 1] + k3 @ (W[b, 2] + 2.0 * np.conj(bz - cz) * W[b, 0])
    # ---- L2L (Eq.(l2l)): parent node values interpolated at the child nodes
    for lev in range(3, int(t.level.max()) + 1):
        for c in np.nonzero(t.level == lev)[0]:
            P = t.parent[c]
            cz, _ = _cell_geom(t, c)
            pz, _ = _cell_geom(t, P)
            S = _interp2(t, P, n, _nodes(t, c, n))       # [nn parent, nn child]
            F[c, 0] += S.T @ F[P, 0]
            F[c, 1] += S.T @ F[P, 1]
            F[c, 2] += S.T @ (F[P, 2] + np.conj(cz - pz) * F[P, 1])
    # ---- L2P + W (node-to-point) + exact near field, per target
    U = T.u_lists(t, w_min=w_min)
    Wl = T.w_lists(t, w_min)
    out = np.zeros((geom.n, 2))
    for B_ in np.nonzero(t.is_leaf)[0]:
        cz, _ = _cell_geom(t, B_)
        tg = perm[t.start[B_]:t.start[B_] + t.count[B_]]
        zt = zc[tg]
        phi = np.zeros(tg.size, dtype=complex)
        dphi = np.zeros_like(phi)
        psit = np.zeros_like(phi)          # Psi~ about the target's own cell centre
        if t.level[B_] >= 2:
            S = _interp2(t, B_, n, zt)     # [nn, ntg]
            phi += S.T @ F[B_, 0]
            dphi += S.T @ F[B_, 1]
            psit += S.T @ F[B_, 2]
        for Dc in Wl[B_]:
            dz, _ = _cell_geom(t, Dc)
            d = zt[:, None] - _nodes(t, Dc, n)[None, :]
            k2, k3 = 1.0 / d ** 2, 1.0 / d ** 3
            phi += k2 @ W[Dc, 0]
            dphi += -2.0 * (k3 @ W[Dc, 0])
            psit += k2 @ W[Dc, 1] + k3 @ (W[Dc, 2] + 2.0 * np.conj(dz - cz) * W[Dc, 0])
        Tf = 2.0 * phi.real + np.exp(2j * geom.beta[tg]) * (np.conj(zt - cz) * dphi + psit)
        # exact near field over U(B): closed-form element integrals (App. A.2)
        src = np.concatenate([perm[t.start[A]:t.start[A] + t.count[A]] for A in U[B_]])
        z1, z2 = zc[src] - a[src] * e[src], zc[src] + a[src] * e[src]
        r = np.conj(e[src]) ** 2
        for ii, i in enumerate(tg):
            z = zc[i]
            I2 = 1 / (z - z2) - 1 / (z - z1)
            I3 = 0.5 * (1 / (z - z2) ** 2 - 1 / (z - z1) ** 2)
            I3b = (np.conj(zc[src]) + r * (z - zc[src])) * I3 - r * I2
            Phi = 1j * gc * np.sum(B[src] * I2)
            dPhi = -2j * gc * np.sum(B[src] * I3)
            Psi = 1j * gc * np.sum(Q[src] * I2 + 2 * B[src] * I3b)
            Tn = 2 * Phi.real + np.exp(2j * geom.beta[i]) * (np.conj(z) * dPhi + Psi)
            Tt = Tf[ii] + Tn
            out[i] = (Tt.imag, Tt.real)
    return out
