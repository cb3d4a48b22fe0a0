"""Wall time of the first poroelastic matvecs on fresh trees (allocation + stream build + on-the-fly near field)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
import bench
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
g = make_config(3); c = CONFIGS[3]; mat = D.material_from_dict(c["material"]); tau = c["dt"]
for rep in range(3):
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p_star"],
                  min_leaf_side=bench._poro_rc(c, g, tau))
    b = f(np.random.default_rng(1).uniform(-1e-3, 1e-3, (g.n, 3)))
    y = torch.empty_like(b)
    ts = []
    for k in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        D.matvec(ctx, tree, mat, b, y, elapsed=tau)
        torch.cuda.synchronize(); ts.append(round((time.perf_counter() - t0) * 1e3, 2))
    print("tree", rep, "matvec ms", ts, flush=True)
    tree.free()
