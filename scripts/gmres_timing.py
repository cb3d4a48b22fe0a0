"""GMRES solve timing on config 3 (poroelastic, full size) and config 2:
solve wall time (device-synchronised), iterations.  python scripts/gmres_timing.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
for cfg in [int(c) for c in os.environ.get("GMRES_CFGS", "2,3").split(",")]:
    c = CONFIGS[cfg]
    g = make_config(cfg)
    mat = D.material_from_dict(c["material"])
    ld = c["load"]
    if cfg == 3:
        m = c["material"]
        M = 2 * m["G"] * (m["nu_u"] - m["nu"]) / (m["alpha"] ** 2 * (1 - 2 * m["nu_u"]) * (1 - 2 * m["nu"]))
        S = m["alpha"] ** 2 * (1 - 2 * m["nu"]) / (2 * m["G"] * (1 - m["nu"])) + 1 / M
        rc = (160 * m["kappa"] / S * c["dt"]) ** 0.5 + 2 * float(g.half_len.max())
        tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                      order_p=c["p_star"], min_leaf_side=rc)
        b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=True,
                           b_p=ld["sh"] + ld["p_f"] - ld["p0"])
        kw = dict(dt=c["dt"], restart=3000, max_iter=6000)
    else:
        tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=20)
        b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
        kw = {}
    D.gmres_solve(ctx, tree, mat, b, tol=1e-10, **kw)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, it, rr = D.gmres_solve(ctx, tree, mat, b, tol=1e-10, **kw)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"cfg{cfg} solve {min(ts):.2f} ms, {it} iters, rel {rr:.2e}", flush=True)
    tree.free()
