import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
c = CONFIGS[5]; g = make_config(5)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
t = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=20)
leaves = t.export("LEAVES"); woff = t.export("W_OFF"); widx = t.export("W_IDX"); cnt = t.export("COUNT")
nB = cnt[leaves]; nW = np.diff(woff)
ev = int((nB * nW).sum()); moved = sum(int(nB[k]) * int(cnt[widx[woff[k]:woff[k+1]]].sum()) for k in range(len(leaves)))
print("W entries", t.counts["W"], "M2P evaluations", ev, "pairs moved", moved, "src per eval", moved / max(ev,1))
print("near pairs", t.counts["NEAR_PAIRS"])
