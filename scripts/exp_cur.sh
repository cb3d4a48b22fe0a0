timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_partition.py tests/test_gpu_poro.py tests/test_gpu_precond.py -x -q 2>&1 | tail -2
for cfg in 3 4; do echo "cfg $cfg"; python scripts/timeline.py $cfg 2>&1 | grep step; DDM_M2L_SPLIT=1 python scripts/timeline.py $cfg 2>&1 | grep step; DDM_M2L_SPLIT=2 python scripts/timeline.py $cfg 2>&1 | grep step; DDM_M2L_SPLIT=4 python scripts/timeline.py $cfg 2>&1 | grep step; done
GMRES_CFGS=2,3 python scripts/gmres_timing.py 3 2>&1 | grep solve
