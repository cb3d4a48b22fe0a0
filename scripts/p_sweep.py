"""Diagnostic: FMM matvec error vs expansion order p (solution and random vectors)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from oracle import elastic as OE
from synth import CONFIGS, make_config, random_dd
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
for cfg in [int(c) for c in (sys.argv[1:] or ["1", "2"])]:
    g = make_config(cfg); c = CONFIGS[cfg]
    A = OE.assemble_dense(g, 8e9, 0.25)
    b = OE.farfield_rhs(g, c["load"]); x = np.linalg.solve(A, b.reshape(-1)).reshape(-1, 2)
    Dv = random_dd(g.n, 2, 100 + cfg); yr = OE.matvec_dense(A, Dv)
    mat = D.material(0, 8e9, 0.25)
    for p in (6, 10, 14, 18, 20, 22, 26, 30, 34, 40):
        t = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=p)
        e1 = np.linalg.norm(D.matvec(ctx, t, mat, f(x)).cpu().numpy() - b) / np.linalg.norm(b)
        e2 = np.linalg.norm(D.matvec(ctx, t, mat, f(Dv)).cpu().numpy() - yr) / np.linalg.norm(yr)
        print(f"cfg{cfg} p={p:2d} sol={e1:.3e} rand={e2:.3e}", flush=True)
