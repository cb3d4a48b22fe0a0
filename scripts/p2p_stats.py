"""Near-field and leaf statistics of a config's tree (design data for the P2P
and P2M mappings): leaf sizes, P2M warp-lane efficiency, U ranges per leaf
and their lengths.  python scripts/p2p_stats.py [cfg]"""
import json
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
leaves = tree.export("LEAVES")
cnt = tree.export("COUNT")[leaves]
uoff, ulo, uhi = tree.export("U_OFF"), tree.export("U_LO"), tree.export("U_HI")
woff = tree.export("W_OFF")
nr = np.diff(uoff)
rl = uhi - ulo
near = np.add.reduceat(rl, uoff[:-1])
out = {
    "leaves": int(leaves.size), "elements": int(cnt.sum()),
    "leaf_count_hist": np.histogram(cnt, bins=[1, 9, 17, 25, 33, 41, 49, 57, 65, 1 << 30])[0].tolist(),
    "p2m_lane_eff_warp_per_leaf": float(cnt.sum() / (32 * np.ceil(cnt / 32)).sum()),
    "ranges_per_leaf_mean": float(nr.mean()), "ranges_per_leaf_max": int(nr.max()),
    "range_len_mean": float(rl.mean()), "range_len_median": float(np.median(rl)),
    "range_len_hist": np.histogram(rl, bins=[1, 5, 9, 17, 33, 65, 129, 257, 1 << 30])[0].tolist(),
    "near_sources_per_leaf_mean": float(near.mean()), "near_sources_per_leaf_max": int(near.max()),
    "near_pairs": int((near * cnt).sum()),
    "w_cells_per_leaf_mean": float(np.diff(woff).mean()),
    "counts": tree.counts,
}
print(json.dumps(out, indent=1))
