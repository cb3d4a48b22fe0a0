"""Profiling driver: config-5 tree + a few FMM matvecs (for ncu launch lists /
--set full captures).  python scripts/profile_matvec.py [reps] [p] [cfg] [mode]
(mode: "fmm" default, "bbfmm3", "bbfmm6", "direct")"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfgn = int(sys.argv[3]) if len(sys.argv) > 3 else 5
mode = sys.argv[4] if len(sys.argv) > 4 else "fmm"
c = CONFIGS[cfgn]
p = int(sys.argv[2]) if len(sys.argv) > 2 else c["p"]
ctx = D.Context(0)
g = make_config(cfgn)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=p)
mat = D.material_from_dict(c["material"])
Dv = f(random_dd(g.n, 2, c.get("d_seed", 55)))
y = torch.empty_like(Dv)
for _ in range(reps):
    D.matvec(ctx, tree, mat, Dv, y, mode=mode)
torch.cuda.synchronize()
print("ok", tree.counts)
