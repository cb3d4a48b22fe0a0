"""Config-4 march: per-step history / GMRES wall times (ms) and lag-build cost."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
import bench
c = CONFIGS[4]; g = make_config(4)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
mat = D.material_from_dict(c["material"]); dt = c["dt"]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"],
              min_leaf_side=bench._poro_rc(c, g, (c["steps"] + 1) * dt))
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False, b_p=ld["p_f"] - ld["p0"])
Dh, st = D.march(ctx, tree, mat, dt, b, steps, tol=c["tol"])
hs = [s["history_s"] * 1e3 for s in st]
print("history ms every 10th:", [round(x, 1) for x in hs[::10]], "max", round(max(hs), 1), "sum", round(sum(hs), 1))
# lag build cost alone: fresh tree, history twice at h = steps-1 (second call builds all lags)
tree2 = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"],
               min_leaf_side=bench._poro_rc(c, g, (c["steps"] + 1) * dt))
h = steps - 1
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    D.history_apply(ctx, tree2, mat, dt, Dh[:h])
    torch.cuda.synchronize(); print("call", k, "h", h, round((time.perf_counter() - t0) * 1e3, 1), "ms")
