# P2P items per warp (grid shrink)
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2P_IPW=2 DDM_P2P_IPW=4 2>&1 | grep total
TUNE_SERIAL=0 python scripts/tune.py base DDM_P2P_IPW=2 DDM_P2P_IPW=4 2>&1 | grep total
