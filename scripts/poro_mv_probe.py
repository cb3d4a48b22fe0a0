"""Steady-state poroelastic matvec time (graph replay, cached near field) and
per-stage serial times for configs 3 and 4."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
import bench
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
for cfg in (4, 3):
    c = CONFIGS[cfg]; g = make_config(cfg)
    mat = D.material_from_dict(c["material"]); dt = c["dt"]
    p = c["p"] if cfg == 4 else c["p_star"]
    tau_rc = (c["steps"] + 1) * dt if cfg == 4 else dt
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=p,
                  min_leaf_side=bench._poro_rc(c, g, tau_rc))
    x = f(np.random.default_rng(1).uniform(-1e-3, 1e-3, (g.n, 3)))
    y = torch.empty_like(x)
    for _ in range(5):
        D.matvec(ctx, tree, mat, x, y, elapsed=dt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        D.matvec(ctx, tree, mat, x, y, elapsed=dt)
    e1.record(); torch.cuda.synchronize()
    mv = e0.elapsed_time(e1) / 50
    ctx.set_profiling(True, serial=True)
    acc = {}
    for _ in range(5):
        D.matvec(ctx, tree, mat, x, y, elapsed=dt); torch.cuda.synchronize()
        for k, v in ctx.stage_times().items(): acc[k] = acc.get(k, 0) + v / 5
    ctx.set_profiling(False)
    print(cfg, "matvec_ms", round(mv, 4), "levels", tree.counts["LEVELS"], "cells", tree.counts["CELLS"],
          {k: round(v, 4) for k, v in acc.items() if v > 0})
