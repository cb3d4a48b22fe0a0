"""Tree build timing (ddm_tree_build_times) for a config, built three times in
one process (the first build includes one-time module loading), plus the
first and second FMM matvec on the last tree.  python scripts/tree_timing.py [cfg]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = CONFIGS[cfg]
g = make_config(cfg)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
xc, yc, hl, be = f(g.xc), f(g.yc), f(g.half_len), f(g.beta)
mat = D.material_from_dict(c["material"])
out = []
for r in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = D.Tree(ctx, xc, yc, hl, be, leaf_size=c["leaf"], order_p=c["p"])
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    bt = tree.build_times()
    Dv = f(random_dd(g.n, 2, 1))
    mv = []
    for _ in range(2):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        D.matvec(ctx, tree, mat, Dv)
        torch.cuda.synchronize()
        mv.append((time.perf_counter() - t1) * 1e3)
    out.append({"build": bt, "wall_ms": wall, "matvec_first_ms": mv[0], "matvec_second_ms": mv[1]})
    tree.free()
print(json.dumps(out, indent=1))
