for i in 1 2; do python scripts/timeline.py 5 2>&1 | grep step; DDM_M2L_CAP=2 python scripts/timeline.py 5 2>&1 | grep step; done
python scripts/timeline.py 3 2>&1 | grep step
DDM_L2P_CAP=1 python scripts/timeline.py 5 2>&1 | grep step
