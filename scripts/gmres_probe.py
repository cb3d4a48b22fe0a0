"""Config-3 GMRES with the trace on: true-residual checks and timing."""
import os, sys, time
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
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, it, rr = D.gmres_solve(ctx, tree, mat, b, dt=tau, tol=c["tol"], restart=3000, max_iter=6000)
    torch.cuda.synchronize(); print("solve", k, it, rr, round((time.perf_counter() - t0) * 1e3, 2), "ms", flush=True)
y = torch.empty_like(b)
for _ in range(3): D.matvec(ctx, tree, mat, b, y, elapsed=tau)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): D.matvec(ctx, tree, mat, b, y, elapsed=tau)
e1.record(); torch.cuda.synchronize(); print("matvec", e0.elapsed_time(e1) / 50, "ms")
yy = torch.empty_like(b)
e0.record()
for _ in range(50): D.precond_apply(ctx, tree, mat, b, yy, dt=tau)
e1.record(); torch.cuda.synchronize(); print("precond_apply (user order, incl. gathers)", e0.elapsed_time(e1) / 50, "ms")
