DDM_M2L_SPLIT=2 python scripts/timeline.py 5 2>&1 | grep step
DDM_M2L_SPLIT=2 DDM_M2L_CAP=2 python scripts/timeline.py 5 2>&1 | grep step
DDM_W_MIN=32 python scripts/timeline.py 5 2>&1 | grep step
DDM_W_MIN=16 python scripts/timeline.py 5 2>&1 | grep step
