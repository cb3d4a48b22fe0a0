"""Where GMRES time goes on config 3 (poroelastic): matvec time with graph
replay vs with a new operand pointer each call (the GMRES pattern), and the
solve time for growing iteration counts (orthogonalisation cost ~ k).
  python scripts/gmres_cost.py"""
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

ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
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
              order_p=c.get("p_star", c["p"]), min_leaf_side=ms)
mat = D.material_from_dict(m)
ld = c["load"]
if poro:
    b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=True,
                       b_p=ld["sh"] + ld["p_f"] - ld["p0"])
else:
    b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
dt = c.get("dt", 0.0)
out = {"n": g.n}
y = torch.empty_like(b)
bufs = [b.clone() for _ in range(20)]


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for k in range(reps):
        fn(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


out["matvec_graph_ms"] = ev_time(lambda k=0: D.matvec(ctx, tree, mat, b, y, elapsed=dt), 20)
out["matvec_newptr_ms"] = ev_time(lambda k=0: D.matvec(ctx, tree, mat, bufs[k % 20], y, elapsed=dt), 20)


def solve_sync(k=0):
    D.matvec(ctx, tree, mat, bufs[k % 20], y, elapsed=dt)
    torch.cuda.synchronize()


out["matvec_newptr_sync_ms"] = ev_time(solve_sync, 20)
for it in (100,):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, k, rr = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=1e-30, restart=3000, max_iter=it,
                             raise_noconv=False)
    torch.cuda.synchronize()
    out[f"gmres_{it}_ms"] = (time.perf_counter() - t0) * 1e3
for rs, mi, tol in ():
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, k, rr = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=tol, restart=rs, max_iter=mi,
                             raise_noconv=False)
    torch.cuda.synchronize()
    out[f"gmres_rs{rs}_mi{mi}_tol{tol}"] = {"iters": k, "rel": rr, "ms": (time.perf_counter() - t0) * 1e3}
for pc in ("leaf", "point", False):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, k, rr = D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=c["tol"], restart=3000,
                             max_iter=6000, raise_noconv=False, precond=pc)
    torch.cuda.synchronize()
    out[f"solve_precond_{pc}"] = {"iters": k, "rel": rr, "ms": (time.perf_counter() - t0) * 1e3}
print(json.dumps(out, indent=1))
