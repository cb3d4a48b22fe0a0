cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_poro.py -x -q 2>&1 | tail -3
python scripts/hist_scaling.py 2>&1 | tail -1
python scripts/hist_probe.py 2>&1 | head -1
