cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_L2P_MINB=4 DDM_L2P_MINB=5 DDM_L2P_MINB=6 2>&1 | grep total
