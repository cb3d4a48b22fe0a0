"""One warm config-3 GMRES solve (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
import bench
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
g = make_config(3); c = CONFIGS[3]
mat = D.material_from_dict(c["material"]); tau = c["dt"]
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p_star"],
              min_leaf_side=bench._poro_rc(c, g, tau))
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=True, b_p=ld["sh"] + ld["p_f"] - ld["p0"])
x, it, rr = D.gmres_solve(ctx, tree, mat, b, dt=tau, tol=c["tol"], restart=3000, max_iter=6000)
torch.cuda.synchronize()
x, it, rr = D.gmres_solve(ctx, tree, mat, b, dt=tau, tol=1e-3, restart=3000, max_iter=6000)
torch.cuda.synchronize()
print("iters", it)
