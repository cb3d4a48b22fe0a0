cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base DDM_EXP_NO_M2L DDM_EXP_NO_L2L DDM_EXP_NO_M2L,DDM_EXP_NO_L2L 2>&1 | tee gpurun_out/exp2.log
