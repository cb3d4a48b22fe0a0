timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py tests/test_gpu_precond.py -x -q -k "gmres or march or precond" 2>&1 | tail -1
GMRES_CFGS=2,3 python scripts/gmres_timing.py 3 2>&1 | grep solve
GMRES_CFGS=2,3 DDM_GMRES_RPT=1 python scripts/gmres_timing.py 3 2>&1 | grep solve
python scripts/march_probe.py 2>&1 | grep march
DDM_GMRES_RPT=1 python scripts/march_probe.py 2>&1 | grep march
