"""Config-4 poroelastic march (200 steps) as bench.py runs it: wall time and
the per-step GMRES / history split.  python scripts/march_probe.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ws = sys.argv[2] if len(sys.argv) > 2 else "extrap3"
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
g = make_config(4)
c = CONFIGS[4]
mat = D.material_from_dict(c["material"])
dt = c["dt"]
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
              order_p=c["p_star"], min_leaf_side=bench._poro_rc(c, g, (c["steps"] + 1) * dt))
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False,
                   b_p=ld["p_f"] - ld["p0"])
D.march(ctx, tree, mat, dt, b, 4, tol=c["tol"])   # warm: graphs, caches
torch.cuda.synchronize()
t0 = time.perf_counter()
Dh, st = D.march(ctx, tree, mat, dt, b, steps, tol=c["tol"], warm_start=ws)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
_, st = D.march(ctx, tree, mat, dt, b, steps, tol=c["tol"], timing=True, warm_start=ws)
its = sum(s["iters"] for s in st)
print(f"march {steps} steps ({ws}): wall {wall:.3f} s, gmres {sum(s['gmres_s'] for s in st):.3f} s "
      f"({its} iterations), history {sum(s['history_s'] for s in st):.3f} s", flush=True)
