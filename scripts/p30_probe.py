import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
import bench
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
c = CONFIGS[2]; g = make_config(2)
mat = D.material_from_dict(c["material"])
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=30)
x = f(np.random.default_rng(1).uniform(-1e-3, 1e-3, (g.n, 2)))
y = torch.empty_like(x)
D.matvec(ctx, tree, mat, x, y)
torch.cuda.synchronize()
print("elastic ok")
