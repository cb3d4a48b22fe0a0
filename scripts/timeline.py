"""Concurrent-schedule timeline of one config-5 matvec: each stage's END (ms)
relative to the start of prep (DDM_STAGE_ENDS=1), averaged over 8 matvecs,
plus the un-instrumented step time.  python scripts/timeline.py [cfg]"""
import os
import sys

os.environ["DDM_STAGE_ENDS"] = "1"
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
mat = D.material_from_dict(c["material"])
if c["material"]["kind"] == 1:
    import bench
    tau = c["dt"]
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                  order_p=c["p_star"], min_leaf_side=bench._poro_rc(c, g, tau))
    Dv = f(random_dd(g.n, 3, 55))
    kw = dict(elapsed=tau)
else:
    tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                  order_p=c.get("p", 20))
    Dv = f(random_dd(g.n, 2, 55))
    kw = {}
y = torch.empty_like(Dv)
mv = lambda: D.matvec(ctx, tree, mat, Dv, y, **kw)
for _ in range(3):
    mv()
torch.cuda.synchronize()
if os.environ.get("TIMELINE_PROFILE"):   # one graph-replayed matvec for an ncu launch list
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    mv()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
ctx.set_profiling(True)
acc = {}
for _ in range(8):
    mv()
    torch.cuda.synchronize()
    for k, v in ctx.stage_times().items():
        acc[k] = acc.get(k, 0) + v / 8
ctx.set_profiling(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mv()
e1.record()
torch.cuda.synchronize()
print("stage ends (ms after prep start):",
      ", ".join(f"{k} {v:.3f}" for k, v in sorted(acc.items(), key=lambda kv: kv[1]) if v > 0))
print(f"step (graph, no instrumentation) {e0.elapsed_time(e1) / 20:.3f} ms")
