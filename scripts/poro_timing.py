"""Poroelastic FMM matvec timing (configs 3 and 4) with the serial per-stage
breakdown.  python scripts/poro_timing.py"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd

ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
res = {}
for cfg in (4, 3):
    c = CONFIGS[cfg]
    g = make_config(cfg)
    m = c["material"]
    G, nu, nuu, al, kap = m["G"], m["nu"], m["nu_u"], m["alpha"], m["kappa"]
    M = 2 * G * (nuu - nu) / (al * al * (1 - 2 * nuu) * (1 - 2 * nu))
    S = al * al * (1 - 2 * nu) / (2 * G * (1 - nu)) + 1 / M
    rcut = math.sqrt(160 * (kap / S) * c["dt"]) + 2 * g.half_len.max()
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                  order_p=c["p"], min_leaf_side=rcut)
    mat = D.material_from_dict(m)
    Dv = random_dd(g.n, 3, 7)
    Dv[:, 2] *= 1e-9
    Dd = f(Dv)
    y = torch.empty_like(Dd)
    for _ in range(2):
        D.matvec(ctx, tree, mat, Dd, y, elapsed=c["dt"])
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        D.matvec(ctx, tree, mat, Dd, y, elapsed=c["dt"])
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 5 * 1e3
    ctx.set_profiling(True, serial=True)
    D.matvec(ctx, tree, mat, Dd, y, elapsed=c["dt"])
    torch.cuda.synchronize()
    st = ctx.stage_times()
    ctx.set_profiling(False)
    res[f"cfg{cfg}"] = {"matvec_ms": ms, "stages_serial_ms": st, "tree": tree.counts}
print(json.dumps(res, indent=1))
