# P2P source-staging variants: register prefetch (PF) and cp.async smem double buffer (CPA); targets per lane
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_P2P_PF=1,DDM_P2P_MINB=4 DDM_P2P_PF=1,DDM_P2P_MINB=5 DDM_P2P_CPA=1,DDM_CPA_CHUNK=16 DDM_P2P_CPA=1,DDM_TPL=3,DDM_P2P_MINB=5 DDM_TPL=3,DDM_P2P_MINB=5 DDM_TPL=3,DDM_P2P_MINB=4 DDM_TPL=4,DDM_P2P_MINB=4 2>&1 | grep -v "^ \|^Trace\|^  File" | tee gpurun_out/exp12.log
