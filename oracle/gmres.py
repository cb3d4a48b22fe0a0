"""ORACLE (test infrastructure only) — dense GMRES.

"a modified version of GMRES with FMM for matrix-vector multiplication is used
to iteratively solve for the problem unknowns".  The paper does
not specify the modification (reading R11): this is textbook restarted GMRES
(Saad & Schultz) with

* Arnoldi orthogonalisation by classical Gram-Schmidt applied twice (CGS2),
* Givens rotations on the Hessenberg matrix,
* stop when the recurrence residual |g_{k+1}| <= tol * ||b||, then one
  explicit true residual ||b - A x|| / ||b|| at exit (reading R12),
* restart m, unpreconditioned (the paper mentions no preconditioner).

`apply` is any callable v -> A v (the oracle passes its dense matrix).
Pins: LU solve (numpy.linalg.solve), b = 0, identity, 3x3 closed-form inverse.
"""
from __future__ import annotations

import numpy as np


def gmres(apply, b: np.ndarray, x0: np.ndarray | None = None, tol: float = 1e-10,
          restart: int = 2000, max_iter: int = 10000):
    """Returns (x, iters, rel_resid, converged)."""
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    n = b.size
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64).reshape(-1)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n), 0, 0.0, True
    iters = 0
    m = max(1, min(restart, max_iter, n))
    while True:
        r = b - apply(x)
        beta = np.linalg.norm(r)
        if beta <= tol * bnorm or iters >= max_iter:
            return x, iters, beta / bnorm, beta <= tol * bnorm
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k_done = 0
        for k in range(m):
            w = apply(V[k])
            h = np.zeros(k + 1)
            for _ in range(2):                       # CGS2: two classical passes
                c = V[:k + 1] @ w
                w = w - V[:k + 1].T @ c
                h += c
            hn = np.linalg.norm(w)
            H[:k + 1, k] = h
            H[k + 1, k] = hn
            if hn > 0.0:
                V[k + 1] = w / hn
            for i in range(k):                       # apply previous rotations
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = np.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / den
            sn[k] = H[k + 1, k] / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            iters += 1
            k_done = k + 1
            if abs(g[k + 1]) <= tol * bnorm or iters >= max_iter or hn == 0.0:
                break
        y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
        x = x + V[:k_done].T @ y
