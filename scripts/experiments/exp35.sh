# P2P with per-item record-range tables (one int2 per range instead of u_lo/u_hi -> rbeg chains)
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_matvec.py tests/test_gpu_partition.py tests/test_gpu_bbfmm.py -x -q 2>&1 | tail -1
TUNE_SERIAL=1 python scripts/tune.py base 2>&1 | grep total
TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total
