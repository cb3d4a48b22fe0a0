"""A/B check of a compile-time variant: build libddm.so with the given
defines (as scripts/tune.py does) and compare its FMM matvec with the default
build's on configs 2 and 5 (bitwise, and the largest relative difference).

  python scripts/ab_compare.py DDM_M2L_PIPE=1[,OTHER=...]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
RUN = r"""
import sys; sys.path.insert(0, %r)
import numpy as np, torch
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config, random_dd
cfg = int(sys.argv[1]); c = CONFIGS[cfg]; g = make_config(cfg)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"])
mat = D.material_from_dict(c["material"])
Dv = f(random_dd(g.n, 2, 55))
ys = [D.matvec(ctx, tree, mat, Dv, mode="fmm").cpu().numpy() for _ in range(3)]
np.save(sys.argv[2], ys[-1])
""" % ROOT


def main():
    from paper_1812_05087_b200 import build as B
    defs = sys.argv[1].split(",")
    libs = {"base": B.build(out="/tmp/ddm_ab_base.so", force=True),
            "variant": B.build(defines=defs, out="/tmp/ddm_ab_var.so", force=True)}
    for cfg in (2, 5):
        ys = {}
        for name, lib in libs.items():
            out = f"/tmp/ab_{cfg}_{name}.npy"
            r = subprocess.run([sys.executable, "-c", RUN, str(cfg), out], env=dict(os.environ, DDM_LIB=lib),
                               capture_output=True, text=True)
            if r.returncode:
                print(cfg, name, "FAILED", r.stderr[-2000:])
                break
            ys[name] = np.load(out)
        if len(ys) == 2:
            d = np.abs(ys["variant"] - ys["base"]).max() / np.abs(ys["base"]).max()
            print(f"config {cfg}: bitwise {np.array_equal(ys['variant'], ys['base'])}, max rel diff {d:.3e}",
                  flush=True)


if __name__ == "__main__":
    main()
