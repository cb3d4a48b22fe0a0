"""Projected per-rank matvec time of the sharded multi-rank path on ONE GPU
(DESIGN.md §6): the config-5 tree partitioned as rank r of W, the matvec run
with DDM_SHARD_NOEXCHANGE=1 (a rank's own work: halo prep, near field of its
leaves, P2M/M2M of its complete cells, straddling M2M, downward pass, L2P and
assembly of its rows -- without the NCCL all-gathers, whose cost is not
measurable on one GPU; results are NOT valid in this mode).  Reports the max
over ranks per W.   DDM_SHARD_NOEXCHANGE=1 python scripts/rank_timing.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd

assert os.environ.get("DDM_SHARD_NOEXCHANGE") == "1", "timing-only mode"
cfg = 5
c = CONFIGS[cfg]
g = make_config(cfg)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"])
mat = D.material_from_dict(c["material"])
x = f(random_dd(g.n, 2, 55))
y = torch.empty_like(x)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
out = {}
for world in (1, 2, 4, 8):
    per = []
    for rank in range(world):
        tree.partition(rank, world)
        for _ in range(3):
            D.matvec(ctx, tree, mat, x, y)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            D.matvec(ctx, tree, mat, x, y)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        per.append(float(np.median(ts)))
    out[world] = {"max_rank_ms": max(per), "per_rank_ms": per}
    print(world, out[world], flush=True)
base = out[1]["max_rank_ms"]
print("RESULT " + json.dumps({"ms": {w: v["max_rank_ms"] for w, v in out.items()},
                              "speedup": {w: base / v["max_rank_ms"] for w, v in out.items()}}))

# serial per-stage breakdown of the slowest rank at W = 8
world = 8
worst = int(np.argmax(out[8]["per_rank_ms"]))
tree.partition(worst, world)
ctx.set_profiling(True, serial=True)
acc = {}
for _ in range(5):
    flush.zero_()
    D.matvec(ctx, tree, mat, x, y)
    torch.cuda.synchronize()
    for k, v in ctx.stage_times().items():
        acc[k] = acc.get(k, 0.0) + v / 5
ctx.set_profiling(False)
print("STAGES_W8 " + json.dumps(acc))
