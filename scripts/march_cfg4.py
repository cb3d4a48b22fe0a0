"""Config 4 time marching on the GPU: per-step GMRES iterations and times, fast
vs per-lag history at the last step.  python scripts/march_cfg4.py [steps]"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from oracle.history import poro_rhs   # RHS values only (same formula as ddm_farfield_rhs)
from synth import CONFIGS, make_config

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = CONFIGS[4]
g = make_config(4)
m = c["material"]
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
G, nu, nuu, al, kap = m["G"], m["nu"], m["nu_u"], m["alpha"], m["kappa"]
M = 2 * G * (nuu - nu) / (al * al * (1 - 2 * nuu) * (1 - 2 * nu))
S = al * al * (1 - 2 * nu) / (2 * G * (1 - nu)) + 1 / M
cc = kap / S
rc = math.sqrt(160 * cc * (steps + 1) * c["dt"]) + 2 * g.half_len.max()
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"],
              min_leaf_side=rc)
mat = D.material_from_dict(m)
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False,
                   b_p=ld["p_f"] - ld["p0"])
t0 = time.perf_counter()
Dh, stats = D.march(ctx, tree, mat, c["dt"], b, steps, tol=c["tol"])
torch.cuda.synchronize()
wall = time.perf_counter() - t0
out = {"steps": steps, "wall_s": wall, "tree": tree.counts,
       "iters": [s["iters"] for s in stats],
       "gmres_s": sum(s["gmres_s"] for s in stats), "history_s": sum(s["history_s"] for s in stats)}
h = steps - 1
for mode in ("fmm", "perlag"):
    D.history_apply(ctx, tree, mat, c["dt"], Dh[:h], mode=mode)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        D.history_apply(ctx, tree, mat, c["dt"], Dh[:h], mode=mode)
    torch.cuda.synchronize()
    out[f"history_{mode}_h{h}_ms"] = (time.perf_counter() - t) / 3 * 1e3
print(json.dumps(out))
