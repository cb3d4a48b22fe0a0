timeout 600 python -m pytest tests/test_gpu_matvec.py -x -q -k march_guess 2>&1 | tail -1
for ws in extrap3 extrap4 extrap5; do python scripts/march_probe.py 200 $ws 2>&1 | grep march; done
