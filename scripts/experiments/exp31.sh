# subtree M2M/L2L passes on small trees: parity + timing
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py tests/test_gpu_partition.py -x -q 2>&1 | tail -1
python scripts/poro_mv_probe.py 2>&1 | cut -c1-200
DDM_SUBTREE=0 python scripts/poro_mv_probe.py 2>&1 | cut -c1-200
python scripts/gmres_probe.py 2>&1 | grep "solve 2"
DDM_SUBTREE=0 python scripts/gmres_probe.py 2>&1 | grep "solve 2"
