"""Config-4 poroelastic matvec (cached near field, graph replay) for launch
lists: python scripts/cfg4_matvec.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = CONFIGS[4]
g = make_config(4)
m = c["material"]
dt = c["dt"]
M = 2 * m["G"] * (m["nu_u"] - m["nu"]) / (m["alpha"] ** 2 * (1 - 2 * m["nu_u"]) * (1 - 2 * m["nu"]))
S = m["alpha"] ** 2 * (1 - 2 * m["nu"]) / (2 * m["G"] * (1 - m["nu"])) + 1 / M
rc = (160 * m["kappa"] / S * (c["steps"] + 1) * dt) ** 0.5 + 2 * float(g.half_len.max())
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
              order_p=c["p_star"], min_leaf_side=rc)
mat = D.material_from_dict(m)
x = f(random_dd(g.n, 3, 4))
y = torch.empty_like(x)
for _ in range(reps):
    D.matvec(ctx, tree, mat, x, y, elapsed=dt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    D.matvec(ctx, tree, mat, x, y, elapsed=dt)
e1.record()
torch.cuda.synchronize()
print("cfg4 matvec ms", e0.elapsed_time(e1) / 100, tree.counts)
