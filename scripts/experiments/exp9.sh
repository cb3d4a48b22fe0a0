cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | tail -1
DDM_NO_GRAPH=1 TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | tail -1
python scripts/gmres_timing.py 100 2>&1 | tail -1
DDM_NO_GRAPH=1 python scripts/gmres_timing.py 100 2>&1 | tail -1
