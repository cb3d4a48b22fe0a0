"""Tuning harness: build variants of libddm.so with compile-time knobs and
time the matvec stages on config 5 (serial mode, per-stage CUDA events).

  python scripts/tune.py "DDM_P2P_MINB=1" "DDM_P2P_MINB=10" ...
Each argument is a comma-separated list of defines for one variant
("base" = no defines).  Prints one line per variant."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MEASURE = r"""
import os, sys, json
sys.path.insert(0, %r)
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd
cfg = int(os.environ.get("TUNE_CFG", "5"))
c = CONFIGS[cfg]; g = make_config(cfg)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
              order_p=int(os.environ.get("TUNE_P", c["p"])))
mat = D.material_from_dict(c["material"])
Dv = f(random_dd(g.n, 2, 55)); y = torch.empty_like(Dv)
for _ in range(3): D.matvec(ctx, tree, mat, Dv, y)
torch.cuda.synchronize()
ctx.set_profiling(True)
acc = {}
for _ in range(8):
    D.matvec(ctx, tree, mat, Dv, y); torch.cuda.synchronize()
    for k, v in ctx.stage_times().items(): acc[k] = acc.get(k, 0) + v / 8
ctx.set_profiling(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): D.matvec(ctx, tree, mat, Dv, y)
e1.record(); torch.cuda.synchronize()
acc["total"] = e0.elapsed_time(e1) / 10
print("RESULT " + json.dumps(acc))
""" % ROOT


def main():
    from paper_1812_05087_b200 import build as B
    variants = sys.argv[1:] or ["base"]
    for v in variants:
        defs = [] if v == "base" else v.split(",")
        out = f"/tmp/ddm_var_{abs(hash(v))}.so"
        B.build(defines=defs, out=out, force=True)
        # TUNE_SERIAL=1 (serial stages), 0 (concurrent schedule) or "both"
        mode = os.environ.get("TUNE_SERIAL", "1")
        for serial in (["1", "0"] if mode == "both" else [mode]):
            env = dict(os.environ, DDM_LIB=out, DDM_SERIAL=serial)
            r = subprocess.run([sys.executable, "-c", MEASURE], env=env, capture_output=True, text=True)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
            if not line:
                print(v, "FAILED", r.stderr[-2000:])
                continue
            d = json.loads(line[0][7:])
            tag = f"{v} [{'serial' if serial == '1' else 'concurrent'}]"
            print(f"{tag:52s} " + " ".join(f"{k}={d[k]:.3f}" for k in
                                          ("total", "prep", "p2p", "p2l", "p2m", "m2m", "m2l", "l2l", "l2p", "final")),
                  flush=True)


if __name__ == "__main__":
    main()
