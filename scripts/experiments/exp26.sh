cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2P_UNROLL=1,DDM_P2P_MINB=8 2>&1 | grep total | tee gpurun_out/exp26.log
TUNE_SERIAL=0 python scripts/tune.py base DDM_P2P_UNROLL=1,DDM_P2P_MINB=8 2>&1 | grep total | tee -a gpurun_out/exp26.log
