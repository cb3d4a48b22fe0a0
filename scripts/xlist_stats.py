"""How much of the near field (P2P pairs) is X-type on config 5: source leaf
A coarser than target leaf B and not touching B (the pairs a P2L list would
take).  python scripts/xlist_stats.py [cfg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c = CONFIGS[cfg]
g = make_config(cfg)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=c["p"])
lev, ix, iy = tree.export("LEVEL"), tree.export("IX"), tree.export("IY")
start, count = tree.export("START"), tree.export("COUNT")
leaves = tree.export("LEAVES")
uoff, ulo, uhi = tree.export("U_OFF"), tree.export("U_LO"), tree.export("U_HI")
n = g.n
el_leaf_cell = np.empty(n, np.int64)
for cc in leaves:
    el_leaf_cell[start[cc]:start[cc] + count[cc]] = cc
tot = 0
xpairs = 0
xb = {}   # X pairs by target-leaf size bucket
coarser_touch = 0
same_or_finer = 0
for k, B in enumerate(leaves):
    nb = count[B]
    for r in range(uoff[k], uoff[k + 1]):
        lo, hi = ulo[r], uhi[r]
        # source leaves within this merged range
        cells = np.unique(el_leaf_cell[lo:hi])
        for A in cells:
            na = count[A]
            tot += na * nb
            if lev[A] < lev[B]:
                d = lev[B] - lev[A]
                # B's ancestor at A's level: touching test in level-lev[B] coordinates
                ax0, ay0 = ix[A] << d, iy[A] << d
                size = 1 << d
                # A covers [ax0, ax0 + size) x [ay0, ay0 + size) at level lev[B]
                gapx = max(ax0 - (ix[B] + 1), ix[B] - (ax0 + size), 0)
                gapy = max(ay0 - (iy[B] + 1), iy[B] - (ay0 + size), 0)
                if gapx > 0 or gapy > 0:
                    xpairs += na * nb
                    bk = min(int(nb) // 16, 4)
                    e = xb.setdefault(bk, [0, 0])
                    e[0] += na * nb          # pairs
                    e[1] += na               # (source element, target leaf) P2L units
                else:
                    coarser_touch += na * nb
            else:
                same_or_finer += na * nb
print(f"near pairs {tot} (tree says {tree.counts['NEAR_PAIRS']}); X-type {xpairs} "
      f"({100.0 * xpairs / tot:.1f} %); coarser touching {coarser_touch} "
      f"({100.0 * coarser_touch / tot:.1f} %); same level or finer source {same_or_finer} "
      f"({100.0 * same_or_finer / tot:.1f} %)")
for bk in sorted(xb):
    pr, un = xb[bk]
    # instruction estimate: P2P 28 per pair vs P2L ~520 per (source element, target leaf)
    print(f"target leaf size {16*bk:3d}-{16*bk+15:3d}: {pr} pairs ({100.0*pr/tot:.1f} % of near), "
          f"{un} P2L units, P2P/P2L instruction ratio {28.0*pr/(520.0*un):.2f}")
