import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1812_05087_b200 as D
from oracle import poro as OP
from synth import CONFIGS, make_config, random_dd
from synth.geometry import Geometry
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
g4 = make_config(4); keep = g4.frac_id < 8
gs = Geometry(g4.xc[keep], g4.yc[keep], g4.half_len[keep], g4.beta[keep], g4.frac_id[keep], g4.tips[:8])
c4 = CONFIGS[4]; pm = c4["material"]; dt = c4["dt"]
Mp = 2 * pm["G"] * (pm["nu_u"] - pm["nu"]) / (pm["alpha"] ** 2 * (1 - 2 * pm["nu_u"]) * (1 - 2 * pm["nu"]))
Sp = pm["alpha"] ** 2 * (1 - 2 * pm["nu"]) / (2 * pm["G"] * (1 - pm["nu"])) + 1 / Mp
rc = (160 * pm["kappa"] / Sp * 5 * dt) ** 0.5 + 2 * float(gs.half_len.max())
tp = D.Tree(ctx, f(gs.xc), f(gs.yc), f(gs.half_len), f(gs.beta), leaf_size=16, order_p=28, min_leaf_side=rc)
matp = D.material_from_dict(pm)
Dp = random_dd(gs.n, 3, 7); Dp[:, 2] *= 1e-9
ref = (OP.assemble_dense(gs, pm, dt) @ Dp.reshape(-1)).reshape(-1, 3)
for mode in ("direct", "fmm", "fmm", "fmm"):
    y = D.matvec(ctx, tp, matp, f(Dp), elapsed=dt, mode=mode).cpu().numpy()
    print(mode, [float(np.linalg.norm(y[:, k] - ref[:, k]) / np.linalg.norm(ref[:, k])) for k in range(3)], float(np.abs(y).max()))
