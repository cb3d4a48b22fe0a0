import sys, numpy as np, torch, collections
sys.path.insert(0, '.')
import paper_1812_05087_b200 as D
from synth import CONFIGS, make_config
c = CONFIGS[5]; g = make_config(5)
ctx = D.Context(0)
f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
t = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"], order_p=20)
leaves = t.export("LEAVES"); off = t.export("U_OFF"); lo = t.export("U_LO"); hi = t.export("U_HI")
lev = t.export("LEVEL"); start = t.export("START"); cnt = t.export("COUNT")
n = g.n
el_leaf = np.empty(n, np.int64)
for k, cl in enumerate(leaves): el_leaf[start[cl]:start[cl]+cnt[cl]] = k
pairs = collections.Counter(); tot = 0
for k, cl in enumerate(leaves):
    nt = cnt[cl]; lb = lev[cl]
    for r in range(off[k], off[k+1]):
        ks = el_leaf[lo[r]:hi[r]]
        # counts per source leaf in the range
        u, m = np.unique(ks, return_counts=True)
        for kk, mm in zip(u, m):
            d = int(lev[leaves[kk]]) - int(lb)
            pairs[d] += int(nt) * int(mm); tot += int(nt) * int(mm)
print("total", tot)
for d in sorted(pairs): print("level(src)-level(tgt) =", d, pairs[d], round(pairs[d]/tot, 4))
print("leaf count hist", np.histogram(cnt[leaves], bins=[1,9,17,33,49,65])[0])
# adjacency of level-mismatched near pairs (boxes touch?)
ix = t.export("IX"); iy = t.export("IY")
def box(cl):
    L = int(lev[cl]); s = 2.0 ** (-L)
    return ix[cl] * s, iy[cl] * s, s
adj = collections.Counter(); nonadj = collections.Counter()
for k, cl in enumerate(leaves):
    nt = int(cnt[cl]); bx, by, bs = box(cl)
    for r in range(off[k], off[k+1]):
        ks = el_leaf[lo[r]:hi[r]]
        u, m = np.unique(ks, return_counts=True)
        for kk, mm in zip(u, m):
            ca = leaves[kk]
            d = int(lev[ca]) - int(lev[cl])
            if d == 0: continue
            ax, ay, as_ = box(ca)
            gapx = max(ax - (bx + bs), bx - (ax + as_), 0.0)
            gapy = max(ay - (by + bs), by - (ay + as_), 0.0)
            (adj if (gapx == 0.0 and gapy == 0.0) else nonadj)[d] += nt * int(mm)
print("mismatched adjacent", sum(adj.values()), "non-adjacent", sum(nonadj.values()))
for d in sorted(set(adj) | set(nonadj)): print(d, adj[d], nonadj[d])
