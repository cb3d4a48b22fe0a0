cd $GRAFT_REPO_ROOT
export TUNE_SERIAL=0
python scripts/tune.py base 2>&1 | tee gpurun_out/exp8.log
DDM_PASS_BLOCKS_PER_SM=2 python scripts/tune.py base 2>&1 | tee -a gpurun_out/exp8.log
DDM_PASS_BLOCKS_PER_SM=0 python scripts/tune.py base 2>&1 | tee -a gpurun_out/exp8.log
DDM_PRIO_SWAP=1 python scripts/tune.py base 2>&1 | tee -a gpurun_out/exp8.log
DDM_PRIO_SWAP=1 DDM_PASS_BLOCKS_PER_SM=0 python scripts/tune.py base 2>&1 | tee -a gpurun_out/exp8.log
