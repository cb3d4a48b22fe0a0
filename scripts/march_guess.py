"""Config-4 200-step march: total GMRES iterations and time for each initial guess."""
import os, sys, time, json
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
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False, b_p=ld["p_f"] - ld["p0"])
ref = None
for ws in ("prev", "extrap2", "extrap3"):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    Dh, st = D.march(ctx, tree, mat, dt, b, 200, tol=c["tol"], warm_start=ws)
    torch.cuda.synchronize(); w = time.perf_counter() - t0
    its = [s["iters"] for s in st]
    if ref is None: ref = Dh.clone()
    diff = (torch.linalg.norm(Dh - ref) / torch.linalg.norm(ref)).item()
    print(ws, "iters", sum(its), "gmres_s", round(sum(s["gmres_s"] for s in st), 3), "wall", round(w, 3),
          "max_rr", max(s["rel_resid"] for s in st), "rel diff vs first run", diff, flush=True)
