"""History-sum cost vs the number of previous steps h on config 4 (fast form):
CUDA events around ddm_history_apply with seeded random D history."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
import bench
c = CONFIGS[4]; g = make_config(4)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
mat = D.material_from_dict(c["material"]); dt = c["dt"]
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"],
              min_leaf_side=bench._poro_rc(c, g, (c["steps"] + 1) * dt))
rng = np.random.default_rng(3)
H = int(sys.argv[1]) if len(sys.argv) > 1 else 199
Dh = f(rng.uniform(-1e-3, 1e-3, (H, g.n, 3)) * np.array([1, 1, 1e-9]))
out = {}
for h in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "10", "50", "100", "199"])]:
    D.history_apply(ctx, tree, mat, dt, Dh[:h])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        D.history_apply(ctx, tree, mat, dt, Dh[:h])
    e1.record(); torch.cuda.synchronize()
    out[h] = round(e0.elapsed_time(e1) / 3, 3)
print(json.dumps(out))
