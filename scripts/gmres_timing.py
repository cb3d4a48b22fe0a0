"""GMRES timing breakdown (config 3 poroelastic, config 2 elastic): solve time
for a fixed number of iterations vs the matvec time alone.
  python scripts/gmres_timing.py [iters]"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
out = {}
for cfg in (2, 3):
    c = CONFIGS[cfg]
    g = make_config(cfg)
    m = c["material"]
    poro = m["kind"] == 1
    ms = 0.0
    if poro:
        G, nu, nuu, al, kap = m["G"], m["nu"], m["nu_u"], m["alpha"], m["kappa"]
        M = 2 * G * (nuu - nu) / (al * al * (1 - 2 * nuu) * (1 - 2 * nu))
        S = al * al * (1 - 2 * nu) / (2 * G * (1 - nu)) + 1 / M
        ms = math.sqrt(160 * (kap / S) * c["dt"]) + 2 * g.half_len.max()
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                  order_p=c["p"], min_leaf_side=ms)
    mat = D.material_from_dict(m)
    ld = c["load"]
    nc = 3 if poro else 2
    if poro:
        b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=True,
                           b_p=ld["sh"] + ld["p_f"] - ld["p0"])
    else:
        b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
    dt = c.get("dt", 0.0)
    for pc in (True, False):
        t = time.perf_counter()
        x, it2, rr2 = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=c["tol"], restart=3000,
                                    max_iter=6000, raise_noconv=False, precond=pc)
        torch.cuda.synchronize()
        out[f"cfg{cfg}_solve_precond{int(pc)}"] = {"iters": it2, "rel": rr2,
                                                   "ms": (time.perf_counter() - t) * 1e3}
    x, it, rr = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=1e-30, restart=3000, max_iter=iters,
                              raise_noconv=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    x, it, rr = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=1e-30, restart=3000, max_iter=iters,
                              raise_noconv=False)
    torch.cuda.synchronize()
    tg = time.perf_counter() - t
    y = torch.empty_like(b)
    t = time.perf_counter()
    for _ in range(iters):
        D.matvec(ctx, tree, mat, b, y, elapsed=dt)
    torch.cuda.synchronize()
    tm = time.perf_counter() - t
    out[f"cfg{cfg}"] = {"iters": it, "gmres_ms": tg * 1e3, "matvecs_ms": tm * 1e3,
                        "overhead_ms_per_iter": (tg - tm) * 1e3 / it}
print(json.dumps(out))
