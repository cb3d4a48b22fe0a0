"""One config-3 (or config-2 / config-4 step) GMRES solve inside a cudaProfilerStart/Stop
range, for an ncu launch list of the solve's kernels:

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/gmres_launches.csv python scripts/gmres_ncu.py 3
  python scripts/gmres_ncu.py --table gpurun_out/gmres_launches.csv
"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        a = agg.setdefault(name.replace("unnamed>::", ""), [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:44s} {n:6d} launches {v / 1e3:10.1f} us  {100 * v / tot:5.1f} %")
    print(f"{'total (serialised)':44s} {sum(n for n, _ in agg.values()):6d} launches {tot / 1e3:10.1f} us")


def main(cfg):
    import numpy as np
    import torch

    import bench
    import paper_1812_05087_b200 as D
    from synth import CONFIGS, make_config

    ctx = D.Context(0)
    f = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")
    c = CONFIGS[cfg]
    g = make_config(cfg)
    mat = D.material_from_dict(c["material"])
    ld = c["load"]
    if cfg == 3:
        tau = c["dt"]
        tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                      order_p=c["p_star"], min_leaf_side=bench._poro_rc(c, g, tau))
        b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=True,
                           b_p=ld["sh"] + ld["p_f"] - ld["p0"])
        kw = dict(dt=tau, restart=3000, max_iter=6000)
    elif cfg == 4:   # the first solve of the config-4 march
        dt = c["dt"]
        tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                      order_p=c["p_star"],
                      min_leaf_side=bench._poro_rc(c, g, (c["steps"] + 1) * dt))
        b = D.farfield_rhs(ctx, f(g.beta), 3, ld["p_f"], ld["sH"], ld["sh"], net=False,
                           b_p=ld["p_f"] - ld["p0"])
        kw = dict(dt=dt, restart=3000, max_iter=6000)
    else:
        tree = D.Tree(ctx, f(g.xc), f(g.yc), f(g.half_len), f(g.beta), leaf_size=c["leaf"],
                      order_p=20)
        b = D.farfield_rhs(ctx, f(g.beta), 2, ld["p_f"], ld["sH"], ld["sh"])
        kw = {}
    for _ in range(2):
        D.gmres_solve(ctx, tree, mat, b, tol=1e-10, **kw)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    x, it, rr = D.gmres_solve(ctx, tree, mat, b, tol=1e-10, **kw)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("iters", it, "rel", rr)


if __name__ == "__main__":
    if sys.argv[1] == "--table":
        table(sys.argv[2])
    else:
        main(int(sys.argv[1]))
