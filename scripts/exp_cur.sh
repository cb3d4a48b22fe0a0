timeout 1200 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_partition.py tests/test_gpu_poro.py tests/test_gpu_precond.py tests/test_gpu_knobs.py -x -q 2>&1 | tail -2
for cfg in 3 4; do echo "cfg $cfg"; python scripts/timeline.py $cfg 2>&1 | grep step; DDM_TOP_CLUSTER=0 python scripts/timeline.py $cfg 2>&1 | grep step; done
GMRES_CFGS=2,3 python scripts/gmres_timing.py 3 2>&1 | grep solve
GMRES_CFGS=2,3 DDM_TOP_CLUSTER=0 python scripts/gmres_timing.py 3 2>&1 | grep solve
python scripts/march_probe.py 2>&1 | grep march
