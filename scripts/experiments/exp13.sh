# far-pass grid cap in the concurrent step (DDM_PASS_BLOCKS_PER_SM), repeated
cd $GRAFT_REPO_ROOT
export TUNE_SERIAL=0
for rep in 1 2 3; do for fc in 1 0 2 3 4; do
  echo -n "PASS_BLOCKS_PER_SM=$fc "
  DDM_PASS_BLOCKS_PER_SM=$fc python scripts/tune.py base 2>&1 | tail -1
done; done 2>&1 | tee gpurun_out/exp13.log
