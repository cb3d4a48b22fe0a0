# stream near field: occupancy / unroll / targets-per-lane variants
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2P_MINB=5 DDM_P2P_MINB=4 DDM_P2P_UNROLL=1 DDM_P2P_UNROLL=1,DDM_P2P_MINB=7 DDM_TPL=1,DDM_P2P_MINB=8 DDM_TPL=4,DDM_P2P_MINB=4 2>&1 | grep total | tee gpurun_out/exp16.log
TUNE_SERIAL=0 python scripts/tune.py base DDM_P2P_MINB=5 DDM_P2P_UNROLL=1 2>&1 | grep total | tee -a gpurun_out/exp16.log
