cd $GRAFT_REPO_ROOT
TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | tail -1
DDM_NO_GRAPH=1 TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | tail -1
