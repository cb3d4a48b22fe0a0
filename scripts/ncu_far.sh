# ncu --set full of the far-field kernels in serial mode (one matvec)
cd $GRAFT_REPO_ROOT
DDM_SERIAL=1 DDM_PASS_BLOCKS_PER_SM=0 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"${NCU_K:-upward|downward}" -c ${NCU_C:-2} -o gpurun_out/${NCU_O:-far} python scripts/profile_matvec.py 1 > gpurun_out/ncu_far.log 2>&1
tail -2 gpurun_out/ncu_far.log
