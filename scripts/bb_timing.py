"""bbFMM (Chebyshev far field, f2) vs the complex-variable FMM on config 5:
matvec time (CUDA events, graph replay), serial per-stage times, and the
relative error of each far field against p = 28 series (~1e-13).
  python scripts/bb_timing.py [n ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd

ns = [int(a) for a in sys.argv[1:]] or [3, 6]
ctx = D.Context(0)
c = CONFIGS[5]
g = make_config(5)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
mat = D.material(0, 8e9, 0.25)
Dv = f(random_dd(g.n, 2, c["d_seed"]))
ref_tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=28)
ref = D.matvec(ctx, ref_tree, mat, Dv).clone()
del ref_tree
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"])
out = {}
y = torch.empty_like(Dv)
for mode in ["fmm"] + [f"bbfmm{n}" for n in ns]:
    for _ in range(3):
        D.matvec(ctx, tree, mat, Dv, y, mode=mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        D.matvec(ctx, tree, mat, Dv, y, mode=mode)
    e1.record()
    torch.cuda.synchronize()
    err = (torch.linalg.norm(y - ref) / torch.linalg.norm(ref)).item()
    ctx.set_profiling(True, serial=True)
    D.matvec(ctx, tree, mat, Dv, y, mode=mode)
    torch.cuda.synchronize()
    st = ctx.stage_times()
    ctx.set_profiling(False)
    out[mode] = {"ms": e0.elapsed_time(e1) / reps, "rel_err_vs_p28": err,
                 "serial_stage_ms": {k: round(v, 4) for k, v in st.items() if v > 0}}
print(json.dumps(out, indent=1))
