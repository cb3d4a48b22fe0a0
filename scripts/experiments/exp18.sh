# stream near field: L1 prefetch distance
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2P_PREFETCH=2 DDM_P2P_PREFETCH=4 DDM_P2P_PREFETCH=8 DDM_P2P_PREFETCH=16 2>&1 | grep total | tee gpurun_out/exp18.log
