import sys, os, time, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
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
Dh, st = D.march(ctx, tree, mat, dt, b, 10, tol=c["tol"])
print(json.dumps([round(s["history_s"] * 1e3, 2) for s in st]), json.dumps([round(s["gmres_s"] * 1e3, 2) for s in st]))
# repeated history applications at h = 9: wall clock vs CUDA events
rhs = torch.empty_like(b)
walls, evs = [], []
for _ in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    D.history_rhs(ctx, tree, mat, dt, Dh[:9], b, rhs)
    e1.record()
    torch.cuda.synchronize()
    walls.append(round((time.perf_counter() - t0) * 1e3, 2))
    evs.append(round(e0.elapsed_time(e1), 2))
print("wall", walls)
print("events", evs)
# per-stage events of repeated history applications (profiling mode, concurrent)
ctx.set_profiling(True)
for _ in range(12):
    D.history_rhs(ctx, tree, mat, dt, Dh[:9], b, rhs)
    torch.cuda.synchronize()
    print({k: round(v, 2) for k, v in ctx.stage_times().items() if v > 0})
ctx.set_profiling(False)
