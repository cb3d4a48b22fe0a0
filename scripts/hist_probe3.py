"""Config-4 march with per-stage events around each history call: find slow steps."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from paper_1812_05087_b200 import api
from synth import CONFIGS, make_config
import bench
c = CONFIGS[4]; g = make_config(4)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
mat = D.material_from_dict(c["material"]); dt = c["dt"]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"],
              min_leaf_side=bench._poro_rc(c, g, (c["steps"] + 1) * dt))
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False, b_p=ld["p_f"] - ld["p0"])
n = tree.n
Dm = torch.zeros((steps, n, 3), dtype=torch.float64, device="cuda")
rhs = torch.empty_like(b)
for h in range(steps):
    ctx.set_profiling(True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.history_rhs(ctx, tree, mat, dt, Dm[:h], b, rhs)
    e1.record()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st = {k: round(v, 2) for k, v in ctx.stage_times().items() if v > 0}
    ctx.set_profiling(False)
    wall = (t1 - t0) * 1e3
    if wall > 15 or h % 40 == 0:
        print(h, "wall", round(wall, 1), "ev", round(e0.elapsed_time(e1), 1), st, flush=True)
    if h > 0:
        Dm[h].copy_(Dm[h - 1])
    api.gmres_solve(ctx, tree, mat, rhs, x=Dm[h], dt=dt, tol=c["tol"])
    torch.cuda.synchronize()
