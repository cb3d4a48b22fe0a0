# P2M powers by even/odd chains
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py -x -q 2>&1 | tail -1
TUNE_SERIAL=1 python scripts/tune.py base 2>&1 | grep total
TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total
