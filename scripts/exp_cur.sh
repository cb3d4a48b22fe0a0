timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py tests/test_gpu_precond.py tests/test_gpu_knobs.py -x -q -k "gmres or march or precond or knob" 2>&1 | tail -3
GMRES_CFGS=2,3 DDM_GMRES_TRACE=1 python scripts/gmres_timing.py 3 2>&1 | grep -E "solve|cluster" | sort | uniq -c | head
GMRES_CFGS=2 DDM_GMRES_CLUSTER=0 python scripts/gmres_timing.py 3 2>&1 | grep solve
python scripts/march_probe.py 2>&1 | grep march
DDM_GMRES_CLUSTER=0 python scripts/march_probe.py 2>&1 | grep march
