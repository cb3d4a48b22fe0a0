cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for env in "DDM_GMRES_SYNC=0" "DDM_GMRES_SYNC=1" "DDM_GMRES_BATCH=4" "DDM_GMRES_BATCH=16"; do
  env $env python bench.py --steps 10 --no-extras > /dev/null 2>&1
  env $env python - <<'PY'
import sys, os, json
sys.path.insert(0, ".")
import torch, bench
import paper_1812_05087_b200 as D
ctx = D.Context(0)
r = bench.gmres_extra(D, ctx, torch, torch.device("cuda", 0), 200)
print(os.environ.get("DDM_GMRES_SYNC"), os.environ.get("DDM_GMRES_BATCH"), json.dumps({k: {kk: (round(vv, 2) if isinstance(vv, float) else vv) for kk, vv in v.items() if kk in ("solve_ms", "iters", "rel_resid", "gmres_s", "history_s", "wall_s", "max_rel_resid")} for k, v in r.items()}))
PY
done
