cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2P_FLAT DDM_P2P_FLAT,DDM_P2P_MINB=5 DDM_P2P_FLAT,DDM_TPL=3,DDM_P2P_MINB=5 2>&1 | tee gpurun_out/exp7.log
TUNE_SERIAL=0 python scripts/tune.py base DDM_P2P_FLAT 2>&1 | tee -a gpurun_out/exp7.log
