"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck, one tool per run): configs 1 and 2 through every elastic path
(FMM, direct, bbFMM, GMRES, the emulated 3-rank sharded matvec) and 4 of
config 4's fractures through the poroelastic matvec (on the fly and cached),
fast history and GMRES.  python scripts/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd
from synth.geometry import Geometry

ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
for cfg in (1, 2):
    c = CONFIGS[cfg]
    g = make_config(cfg)
    mat = D.material_from_dict(c["material"])
    args = (f(g.xc), f(g.yc), f(g.half_len), f(g.beta))
    tree = D.Tree(ctx, *args, leaf_size=c["leaf"], order_p=20)
    x = f(random_dd(g.n, 2, cfg))
    y = torch.empty_like(x)
    for mode in ("fmm", "fmm", "fmm", "direct", "bbfmm3"):
        D.matvec(ctx, tree, mat, x, y, mode=mode)
    ld = c["load"]
    b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
    D.gmres_solve(ctx, tree, mat, b, tol=1e-10)
    trees = [D.Tree(ctx, *args, leaf_size=c["leaf"], order_p=20) for _ in range(3)]
    for r, t in enumerate(trees):
        t.partition(r, 3)
    D.matvec_sim(ctx, trees, mat, x)
    for t in trees:
        t.free()
    tree.free()
g4 = make_config(4)
keep = g4.frac_id < 4
g = Geometry(g4.xc[keep], g4.yc[keep], g4.half_len[keep], g4.beta[keep], g4.frac_id[keep], g4.tips[:4])
c = CONFIGS[4]
m = c["material"]
dt = c["dt"]
M = 2 * m["G"] * (m["nu_u"] - m["nu"]) / (m["alpha"] ** 2 * (1 - 2 * m["nu_u"]) * (1 - 2 * m["nu"]))
S = m["alpha"] ** 2 * (1 - 2 * m["nu"]) / (2 * m["G"] * (1 - m["nu"])) + 1 / M
rc = (160 * m["kappa"] / S * 5 * dt) ** 0.5 + 2 * float(g.half_len.max())
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=16, order_p=20,
              min_leaf_side=rc)
mat = D.material_from_dict(m)
x = f(random_dd(g.n, 3, 5))
for _ in range(3):
    D.matvec(ctx, tree, mat, x, elapsed=dt)
Dh = torch.stack([f(random_dd(g.n, 3, 6 + k)) for k in range(3)])
for h in (1, 2, 3):
    D.history_apply(ctx, tree, mat, dt, Dh[:h].contiguous())
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False, b_p=ld["p_f"] - ld["p0"])
D.gmres_solve(ctx, tree, mat, b, dt=dt, tol=1e-10)
torch.cuda.synchronize()
print("sanitize case done")
