"""The environment knobs select alternative code paths once per process
(static reads); each combination runs in a subprocess and must give the same
answers as the default path: GMRES (config 2) against LU, the poroelastic
matvec and history sum (8 fractures of config 4) against the dense oracle."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np, torch
import paper_1812_05087_b200 as D
from oracle import elastic as OE, history as OH, poro as OP
from synth import CONFIGS, make_config, random_dd
from synth.geometry import Geometry
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
out = {}
g = make_config(2); c = CONFIGS[2]; m = c["material"]
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=28)
mat = D.material_from_dict(m)
ld = c["load"]
b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
x, it, rr = D.gmres_solve(ctx, tree, mat, b, tol=1e-10)
A = OE.assemble_dense(g, m["G"], m["nu"])
xl = np.linalg.solve(A, OE.farfield_rhs(g, ld).reshape(-1)).reshape(-1, 2)
out["gmres"] = float(np.linalg.norm(x.cpu().numpy() - xl) / np.linalg.norm(xl))
g4 = make_config(4); keep = g4.frac_id < 8
gs = Geometry(g4.xc[keep], g4.yc[keep], g4.half_len[keep], g4.beta[keep], g4.frac_id[keep], g4.tips[:8])
c4 = CONFIGS[4]; pm = c4["material"]; dt = c4["dt"]
Mp = 2 * pm["G"] * (pm["nu_u"] - pm["nu"]) / (pm["alpha"] ** 2 * (1 - 2 * pm["nu_u"]) * (1 - 2 * pm["nu"]))
Sp = pm["alpha"] ** 2 * (1 - 2 * pm["nu"]) / (2 * pm["G"] * (1 - pm["nu"])) + 1 / Mp
rc = (160 * pm["kappa"] / Sp * 5 * dt) ** 0.5 + 2 * float(gs.half_len.max())
tp = D.Tree(ctx, f(gs.xc), f(gs.yc), f(gs.half_len), f(gs.beta), leaf_size=16, order_p=28, min_leaf_side=rc)
matp = D.material_from_dict(pm)
Dp = random_dd(gs.n, 3, 7); Dp[:, 2] *= 1e-9
K = [None] + [OP.assemble_dense(gs, pm, j * dt) for j in range(1, 5)]
ref = (K[1] @ Dp.reshape(-1)).reshape(-1, 3)
errs = []
for _ in range(3):
    y = D.matvec(ctx, tp, matp, f(Dp), elapsed=dt).cpu().numpy()
    errs.append(max(float(np.linalg.norm(y[:, k] - ref[:, k]) / np.linalg.norm(ref[:, k])) for k in range(3)))
out["poro_matvec"] = max(errs)
Dh = np.stack([random_dd(gs.n, 3, 8 + k) for k in range(3)]); Dh[:, :, 2] *= 1e-9
lags = [None] + [K[j + 1] - K[j] for j in range(1, 4)]
herr = []
for h in (1, 2, 3):
    r = D.history_apply(ctx, tp, matp, dt, f(Dh[:h])).cpu().numpy()
    rh = OH.history_sum(gs, dict(pm, kind=1), dt, Dh[:h], lags)
    herr.append(max(float(np.linalg.norm(r[:, k] - rh[:, k]) / np.linalg.norm(rh[:, k])) for k in range(3)))
out["history"] = max(herr)
print("RESULT " + json.dumps(out))
""" % ROOT


@pytest.mark.parametrize("env", [
    {},
    {"DDM_GMRES_SYNC": "1"},
    {"DDM_GMRES_FUSE_PC": "0"},
    {"DDM_NEAR_CACHE": "0", "DDM_HIST_CACHE": "0"},
    {"DDM_PDL": "0", "DDM_SUBTREE": "0", "DDM_EARLY_FAR": "0"},
    {"DDM_NO_GRAPH": "1", "DDM_SERIAL": "1"},
    {"DDM_PDL": "1", "DDM_SUBTREE": "1", "DDM_GMRES_BATCH": "3"},
    # the multi-rank exchange path (NCCL all-gather of the owned rows, NCCL
    # all-reduce of the GMRES dots) on a one-rank communicator
    {"DDM_FORCE_NCCL": "1"},
    {"DDM_FORCE_NCCL": "1", "DDM_GMRES_SYNC": "1"},
    # every library allocation poisoned with NaN / -1 (uninitialised reads
    # surface in the checked results; compute-sanitizer is closed on the pool)
    {"DDM_POISON": "1"},
    {"DDM_GMRES_DGKS": "1"},
    {"DDM_POISON": "1", "DDM_GMRES_GRAPH": "0", "DDM_P2P_LEAF": "0", "DDM_L2P_BLOCK": "0"},
    # vector-parallel CGS kernels instead of the row-blocked ones
    {"DDM_GMRES_ROWS": "0", "DDM_P2P_ORDER": "0", "DDM_L2P_ORDER": "0"},
    # round 2 (late): CGS row blocks of 512 / 256 rows, GMRES step without PDL,
    # M2L with one warp per cell; X lists on (§4.13)
    {"DDM_GMRES_ROWT": "512", "DDM_GMRES_PDL": "0", "DDM_M2L_SPLIT": "1"},
    {"DDM_GMRES_ROWT": "256", "DDM_M2L_SPLIT": "2", "DDM_X_MIN": "1", "DDM_POISON": "1"},
])
def test_knob_paths_agree_with_oracle(env):
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=dict(os.environ, **env),
                       capture_output=True, text=True, timeout=600)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
    assert line, r.stderr[-3000:]
    res = json.loads(line[0][7:])
    assert res["gmres"] <= 1e-6, (env, res)
    assert res["poro_matvec"] <= 1e-8, (env, res)
    assert res["history"] <= 1e-8, (env, res)
