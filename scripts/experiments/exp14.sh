# near-field block lifetime (sources per item, warps per block) in the concurrent step
cd $GRAFT_REPO_ROOT
export TUNE_SERIAL=0
python scripts/tune.py base DDM_SRC_CHUNK=256 DDM_SRC_CHUNK=128 DDM_P2P_WARPS=2 DDM_P2P_WARPS=8 DDM_P2P_WARPS=2,DDM_SRC_CHUNK=256 base 2>&1 | grep total | tee gpurun_out/exp14.log
TUNE_SERIAL=1 python scripts/tune.py DDM_SRC_CHUNK=256 DDM_P2P_WARPS=2 2>&1 | grep total | tee -a gpurun_out/exp14.log
