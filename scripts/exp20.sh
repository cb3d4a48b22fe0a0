cd $GRAFT_REPO_ROOT
python scripts/hist_probe.py 2>&1 | tail -3
python scripts/hist_probe.py 2>&1 | tail -3
