"""Test-only reference quadrature: double-exponential (tanh-sinh) rule, a
family independent of the graded Gauss-Legendre rule the oracle and the GPU
path share, used to pin that rule to the exact element
integrals of the poroelastic point kernel (oracle/poro.py point_kernel)."""
import numpy as np

from oracle import poro as P


def tanh_sinh(lo, hi, h, tmax=4.0):
    """Nodes and weights on [lo, hi] with step h; nodes are placed by their
    distance from the nearer endpoint (no rounding onto the endpoint)."""
    t = np.arange(-tmax, tmax + h / 2, h)
    u = 0.5 * np.pi * np.sinh(t)
    w = h * 0.5 * np.pi * np.cosh(t) / np.cosh(u) ** 2
    d = 1.0 / (np.exp(np.abs(u)) * np.cosh(u))   # 1 - |x| for x = tanh(u)
    r = 0.5 * (hi - lo)
    s = np.where(u >= 0, hi - r * d, lo + r * d)
    keep = (r * d > 0) & (s > lo) & (s < hi)
    return s[keep], r * w[keep]


def breakpoints(rel, a):
    """The element [-a, a] split at the foot of the perpendicular from the
    target (element-frame offset rel) and at 1 and 4 distances from it."""
    foot = min(max(rel.real, -a), a)
    dp = max(abs(rel.imag), 1e-3 * a)
    return sorted({x for x in (-a, a, foot, foot - dp, foot + dp, foot - 4 * dp, foot + 4 * dp)
                   if -a <= x <= a})


def element_integral_ts(zt, zc, e, a, tau, k, Ds, Dn, q, h=1 / 32):
    """(p, d2Phi) of the element (zc, e, a) at zt by tanh-sinh, plus the
    integral of |p| + |d2Phi| (the scale of the rounding); offsets formed as
    (rel - s) e so nodes next to the target keep their relative accuracy."""
    rel = (zt - zc) * np.conj(e)
    pts = breakpoints(rel, a)
    tp, td, mag = 0.0, 0.0 + 0.0j, 0.0
    for lo, hi in zip(pts[:-1], pts[1:]):
        s, w = tanh_sinh(lo, hi, h)
        off = (rel - s) * e
        m = np.abs(off) > 1e-140          # r^2 would underflow
        pp, dd = P.point_kernel(off[m], tau, k, e, Ds, Dn, q)
        tp += np.sum(w[m] * pp.real)
        td += np.sum(w[m] * dd)
        mag += np.sum(w[m] * (np.abs(pp.real) + np.abs(dd)))
    return tp, td, mag
