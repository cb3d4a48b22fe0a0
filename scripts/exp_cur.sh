timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_partition.py tests/test_gpu_poro.py -x -q -k "parity or partition or sim or history_small or gmres_cfg4" 2>&1 | tail -2
for cfg in 3 4 5; do echo "cfg $cfg"; python scripts/timeline.py $cfg 2>&1 | grep step; done
GMRES_CFGS=2,3 python scripts/gmres_timing.py 3 2>&1 | grep solve
