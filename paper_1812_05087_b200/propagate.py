"""Fracture propagation loop (Fig. 8 branch; SURVEY §8f
row f4): solve, SIFs at the tips (Eq.(SIF)), propagation criterion, add an
element at every tip that grows, rebuild the quad-tree, repeat.  The host
loop around the C-ABI calls (ddm_build_tree, ddm_gmres_solve, ddm_sif,
ddm_tip_growth); the arithmetic runs in libddm.so, the host only gathers tip
values and appends the new elements.  Elastic, one temporal element per
step (the paper leaves the coupling of propagation and time marching open).
"""
from __future__ import annotations

import torch

from . import api


def propagate(ctx, xc, yc, half_len, beta, tips, mat, load: dict, K_IC: float, steps: int,
              leaf_size: int = 32, order_p: int = 28, tol: float = 1e-10, stream=None):
    """xc, yc, half_len, beta: float64 device tensors (elements); tips: int
    tensor [ntips, 2] of (element index, end) with end 1 = the element's
    + e^{i beta} endpoint; mat: elastic material; load: far-field dict
    (p_f, sH, sh).  Returns (xc, yc, half_len, beta, tips, history) with one
    dict per step (n, iters, rel_resid, KI, KII, grow as host lists)."""
    dev = xc.device
    tips = tips.to(device=dev, dtype=torch.int64)
    E = 2.0 * mat.G * (1.0 + mat.nu)
    history = []
    for _ in range(steps):
        tree = api.Tree(ctx, xc, yc, half_len, beta, leaf_size=leaf_size, order_p=order_p,
                        stream=stream)
        b = api.farfield_rhs(ctx, beta, 2, load["p_f"], load["sH"], load["sh"], stream=stream)
        x, it, rr = api.gmres_solve(ctx, tree, mat, b, tol=tol, stream=stream)
        tree.free()
        ti = tips[:, 0]
        KI, KII = api.sif(ctx, x[ti, 1].contiguous(), x[ti, 0].contiguous(),
                          half_len[ti].contiguous(), E, mat.nu, stream=stream)
        end = tips[:, 1].to(torch.int32).contiguous()
        grow, nx, ny, na, nb, ne = api.tip_growth(
            ctx, KI, KII, xc[ti].contiguous(), yc[ti].contiguous(), half_len[ti].contiguous(),
            beta[ti].contiguous(), end, K_IC, stream=stream)
        g = grow.to(torch.bool)
        history.append({"n": int(xc.numel()), "iters": it, "rel_resid": rr,
                        "KI": KI.tolist(), "KII": KII.tolist(), "grow": grow.tolist()})
        if not bool(g.any()):
            break
        n0 = xc.numel()
        xc = torch.cat([xc, nx[g]])
        yc = torch.cat([yc, ny[g]])
        half_len = torch.cat([half_len, na[g]])
        beta = torch.cat([beta, nb[g]])
        new_idx = n0 + torch.arange(int(g.sum()), device=dev)
        tips = tips.clone()
        tips[g, 0] = new_idx
        tips[g, 1] = ne[g].to(torch.int64)
    return xc, yc, half_len, beta, tips, history
