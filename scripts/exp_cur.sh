timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_poro.py tests/test_gpu_precond.py tests/test_gpu_knobs.py -x -q -k "gmres or march or precond or knob" 2>&1 | tail -2
for rt in 0 512 256 128; do echo "ROWT $rt"; GMRES_CFGS=2 DDM_GMRES_ROWT=$rt DDM_GMRES_TRACE=1 python scripts/gmres_timing.py 3 2>&1 | grep -E "solve|row-blocked" | sort | uniq -c; DDM_GMRES_ROWT=$rt python scripts/march_probe.py 2>&1 | grep march; done
DDM_GMRES_ROWS=0 python scripts/march_probe.py 2>&1 | grep march
