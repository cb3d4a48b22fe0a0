# far chain starts at the fork (P2M reads D through perm) vs after prep
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py tests/test_gpu_partition.py -x -q 2>&1 | tail -1
python scripts/poro_mv_probe.py 2>&1 | cut -c1-40
DDM_EARLY_FAR=0 python scripts/poro_mv_probe.py 2>&1 | cut -c1-40
TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total
DDM_EARLY_FAR=0 TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total
python scripts/gmres_probe.py 2>&1 | grep "solve 2"
DDM_EARLY_FAR=0 python scripts/gmres_probe.py 2>&1 | grep "solve 2"
