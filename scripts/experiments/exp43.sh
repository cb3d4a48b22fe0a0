# far-pass grid cap re-tuned after the early far chain
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for fc in 1 2 3 0; do
  echo -n "PASS_BLOCKS_PER_SM=$fc "; DDM_PASS_BLOCKS_PER_SM=$fc TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total
done; done
