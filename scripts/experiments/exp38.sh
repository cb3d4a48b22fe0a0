# M2L pairs per batch (loads in flight vs registers)
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_M2L_BATCH=2 DDM_M2L_BATCH=6 DDM_M2L_BATCH=8 2>&1 | grep total
TUNE_SERIAL=0 python scripts/tune.py base DDM_M2L_BATCH=6 DDM_M2L_BATCH=8 2>&1 | grep total
