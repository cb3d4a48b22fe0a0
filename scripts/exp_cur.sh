timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_partition.py -x -q -k "x_lists or partition or cfg5 or parity" 2>&1 | tail -3
for xm in 0 20 32; do echo "X_MIN=$xm"; DDM_X_MIN=$xm TUNE_SERIAL=1 python scripts/tune.py base DDM_P2L_MINB=3 2>&1 | grep -v Warn; DDM_X_MIN=$xm TUNE_SERIAL=0 python scripts/tune.py base DDM_P2L_MINB=3 2>&1 | grep -v Warn; done
