cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2M_MINB=3 DDM_M2L_MINB=3 DDM_M2L_MINB=1 2>&1 | grep total
TUNE_SERIAL=0 python scripts/tune.py base DDM_P2M_MINB=3 DDM_M2L_MINB=3 2>&1 | grep total
