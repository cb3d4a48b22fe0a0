#!/bin/bash
# GMRES iterations / time vs the reorthogonalisation threshold (DDM_GMRES_ETA2)
for cfg in 2 3; do for e in 0.5 1e-2 1e-4 0; do
  echo "cfg $cfg eta2 $e: $(DDM_GMRES_ETA2=$e python scripts/gmres_cost.py $cfg 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print({k: d[k] for k in d if k.startswith("solve") or k.startswith("gmres_rs3000_mi6000")})')"
done; done
