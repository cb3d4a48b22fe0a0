"""ORACLE (test infrastructure only) — elastic constant-DD influence matrix.

What it computes (the plain definition, no FMM): the dense 2N x 2N matrix A of
Eq.(final_sigs) with only the current-step, elastic blocks A_xx, A_xy, A_yx,
A_yy ("A_xx is the shear stress that is induced on the observation
point from a unit shear displacement discontinuity at the influencing point",
P:447-449), and y = A D.

The paper does not print A_ij (it cites Carvalho 1991 / Crouch 1976,
P:442-449).  This file restates the classical Crouch–Starfield constant
displacement-discontinuity element, real-variable form,
in the element frame, then rotates:

  element on y = 0, -a <= x <= a;  C = 1/(4 pi (1 - nu))
  R1 = (x-a)^2 + y^2, R2 = (x+a)^2 + y^2
  f_xy  = C (y/R1 - y/R2)
  f_xx  = -f_yy = C ((x-a)/R1 - (x+a)/R2)
  f_xyy = C (((x-a)^2 - y^2)/R1^2 - ((x+a)^2 - y^2)/R2^2)
  f_yyy = 2 C y ((x-a)/R1^2 - (x+a)/R2^2)
  s_xx = 2G Dx (2 f_xy + y f_xyy) + 2G Dy (f_yy + y f_yyy)
  s_yy = -2G Dx y f_xyy          + 2G Dy (f_yy - y f_yyy)
  s_xy = 2G Dx (f_yy + y f_yyy)  - 2G Dy y f_xyy
  (tension positive, D = u(y=0-) - u(y=0+))

Conventions (DESIGN.md §2 readings R2/R3): stresses and
pressure compression-positive, DDs opening-positive (D_n = -D_y^CS,
D_s = -D_x^CS).  Both signs flip, so A_ABI = A_CS numerically and the system
reads A D = b.  DOF layout element-major interleaved: row/col 2i+0 = shear
(s), 2i+1 = normal (n).  Collocation at element centres (reading R3).

Pins (tests/test_oracle_elastic.py): Sneddon opening (config 1), self term
G/(pi(1-nu)a), displacement jump = D, Hooke + equilibrium by finite
differences of the displacement field, additivity of split elements, r^-2
decay, rotation invariance, symmetric Toeplitz straight crack, and an
independent complex-variable (Kolosov–Muskhelishvili) formula family.
"""
from __future__ import annotations

import numpy as np


def cs_local_stress(x, y, a, Dx, Dy, G, nu):
    """Stress (s_xx, s_yy, s_xy), tension positive, at (x, y) in the element frame
    of a constant DD element of half-length a carrying (Dx, Dy).  Vectorised."""
    C = 1.0 / (4.0 * np.pi * (1.0 - nu))
    xm = x - a
    xp = x + a
    R1 = xm * xm + y * y
    R2 = xp * xp + y * y
    f_xy = C * (y / R1 - y / R2)
    f_xx = C * (xm / R1 - xp / R2)
    f_yy = -f_xx
    f_xyy = C * ((xm * xm - y * y) / (R1 * R1) - (xp * xp - y * y) / (R2 * R2))
    f_yyy = 2.0 * C * y * (xm / (R1 * R1) - xp / (R2 * R2))
    sxx = 2.0 * G * Dx * (2.0 * f_xy + y * f_xyy) + 2.0 * G * Dy * (f_yy + y * f_yyy)
    syy = -2.0 * G * Dx * y * f_xyy + 2.0 * G * Dy * (f_yy - y * f_yyy)
    sxy = 2.0 * G * Dx * (f_yy + y * f_yyy) - 2.0 * G * Dy * y * f_xyy
    return sxx, syy, sxy


def cs_local_disp(x, y, a, Dx, Dy, nu):
    """Displacements (u_x, u_y) of the same element (used only by the pins:
    jump = D and Hooke/equilibrium).  f_x, f_y carry the log / atan terms."""
    C = 1.0 / (4.0 * np.pi * (1.0 - nu))
    xm = x - a
    xp = x + a
    R1 = xm * xm + y * y
    R2 = xp * xp + y * y
    th1 = np.arctan2(y, xm)
    th2 = np.arctan2(y, xp)
    f_x = 0.5 * C * (np.log(R1) - np.log(R2))
    f_y = -C * (th1 - th2)
    f_xy = C * (y / R1 - y / R2)
    f_xx = C * (xm / R1 - xp / R2)
    f_yy = -f_xx
    ux = Dx * (2.0 * (1.0 - nu) * f_y - y * f_xx) + Dy * (-(1.0 - 2.0 * nu) * f_x - y * f_xy)
    uy = Dx * ((1.0 - 2.0 * nu) * f_x - y * f_xy) + Dy * (2.0 * (1.0 - nu) * f_y - y * f_yy)
    return ux, uy


def global_stress(xt, yt, xs, ys, a, bs, Ds, Dn, G, nu):
    """Global-frame stress at (xt, yt) from source element (xs, ys, a, bs) with
    element-local DDs (Ds along the element, Dn normal).  Vectorised."""
    c, s = np.cos(bs), np.sin(bs)
    dx = xt - xs
    dy = yt - ys
    xl = dx * c + dy * s
    yl = -dx * s + dy * c
    lxx, lyy, lxy = cs_local_stress(xl, yl, a, Ds, Dn, G, nu)
    sxx = c * c * lxx - 2.0 * c * s * lxy + s * s * lyy
    syy = s * s * lxx + 2.0 * c * s * lxy + c * c * lyy
    sxy = c * s * lxx + (c * c - s * s) * lxy - c * s * lyy
    return sxx, syy, sxy


def project_traction(sxx, syy, sxy, bt):
    """(sigma_s, sigma_n) on a face with direction angle bt: s = e^{i bt},
    n = i e^{i bt}."""
    c, s = np.cos(bt), np.sin(bt)
    sn = sxx * s * s + syy * c * c - 2.0 * sxy * s * c
    ss = (syy - sxx) * s * c + sxy * (c * c - s * s)
    return ss, sn


def influence_blocks(xt, yt, bt, xs, ys, a, bs, G, nu):
    """2x2 influence blocks for target/source pairs (broadcast arrays).
    Returns (A_ss, A_sn, A_ns, A_nn): rows (sigma_s, sigma_n) at the target
    centre, columns (D_s, D_n) of the source."""
    one = np.ones_like(np.broadcast_to(xs, np.broadcast(xt, xs).shape), dtype=np.float64)
    zero = np.zeros_like(one)
    s_xx, s_yy, s_xy = global_stress(xt, yt, xs, ys, a, bs, one, zero, G, nu)
    A_ss, A_ns = project_traction(s_xx, s_yy, s_xy, bt)
    n_xx, n_yy, n_xy = global_stress(xt, yt, xs, ys, a, bs, zero, one, G, nu)
    A_sn, A_nn = project_traction(n_xx, n_yy, n_xy, bt)
    return A_ss, A_sn, A_ns, A_nn


def assemble_dense(geom, G, nu, row_block: int = 256) -> np.ndarray:
    """Dense 2N x 2N matrix, DOF 2i+c (c = 0 shear, 1 normal)."""
    n = geom.n
    A = np.empty((2 * n, 2 * n))
    for r0 in range(0, n, row_block):
        r1 = min(n, r0 + row_block)
        sl = slice(r0, r1)
        blk = influence_blocks(geom.xc[sl, None], geom.yc[sl, None], geom.beta[sl, None],
                               geom.xc[None, :], geom.yc[None, :], geom.half_len[None, :],
                               geom.beta[None, :], G, nu)
        A[2 * r0:2 * r1:2, 0::2] = blk[0]
        A[2 * r0:2 * r1:2, 1::2] = blk[1]
        A[2 * r0 + 1:2 * r1:2, 0::2] = blk[2]
        A[2 * r0 + 1:2 * r1:2, 1::2] = blk[3]
    return A


def matvec_rows(geom, G, nu, D: np.ndarray, rows: np.ndarray, chunk: int = 8) -> np.ndarray:
    """Matrix-free y[rows] = (A D)[rows] for a subset of target elements,
    summing sources j in ascending order per row (config-5 sampled parity).
    D is [N, 2]; returns [len(rows), 2]."""
    rows = np.asarray(rows)
    out = np.empty((rows.size, 2))
    Ds = D[:, 0]
    Dn = D[:, 1]
    for k0 in range(0, rows.size, chunk):
        idx = rows[k0:k0 + chunk]
        sxx, syy, sxy = global_stress(geom.xc[idx, None], geom.yc[idx, None], geom.xc[None, :],
                                      geom.yc[None, :], geom.half_len[None, :],
                                      geom.beta[None, :], Ds[None, :], Dn[None, :], G, nu)
        ss, sn = project_traction(sxx, syy, sxy, geom.beta[idx, None])
        out[k0:k0 + chunk, 0] = ss.sum(axis=1)
        out[k0:k0 + chunk, 1] = sn.sum(axis=1)
    return out


def matvec_dense(A: np.ndarray, D: np.ndarray) -> np.ndarray:
    """y = A D with D [N, ncomp] element-major; returns [N, ncomp]."""
    return (A @ D.reshape(-1)).reshape(D.shape)


def farfield_rhs(geom, load) -> np.ndarray:
    """Right-hand side of the first step ("transforming the far-field
    stresses to the face of each element and by adding their effect to the
    hydraulic load").  Compression-positive; SHmax along x, Shmin along y.
    The face must carry total normal traction p_f and zero shear:
      sigma_n^ff = sH sin^2 b + sh cos^2 b             (ABI, compression +)
      sigma_s^ff = (sh - sH) sin b cos b  (= project_traction of diag(sH, sh))
      b_s = -sigma_s^ff = (sH - sh) sin b cos b
      b_n = p_f - sigma_n^ff                            (mode 'absolute')
      b_n = p_f (uniform net pressure)                  (mode 'net')
    (reading R14: the sign of b_s follows from the same projection
    as the operator rows; pinned by the inclined-crack sliding test.)
    Returns [N, 2] (s, n)."""
    b = geom.beta
    s, c = np.sin(b), np.cos(b)
    sn_ff = load["sH"] * s * s + load["sh"] * c * c
    ss_ff = (load["sh"] - load["sH"]) * s * c
    out = np.empty((geom.n, 2))
    out[:, 0] = -ss_ff
    if load["mode"] == "net":
        out[:, 1] = load["p_f"]
    else:
        out[:, 1] = load["p_f"] - sn_ff
    return out


def sneddon_opening(x, a, p, E, nu):
    """Sneddon's closed-form opening of a pressurised Griffith crack, plane
    strain: w(x) = 4 (1 - nu^2) p / E * sqrt(a^2 - x^2) (BASELINE configs[0])."""
    return 4.0 * (1.0 - nu * nu) * p / E * np.sqrt(a * a - x * x)
