set -x
cd $GRAFT_REPO_ROOT
TUNE_SERIAL=1 python scripts/tune.py base > gpurun_out/tune_serial.log 2>&1
TUNE_SERIAL=0 python scripts/tune.py base >> gpurun_out/tune_serial.log 2>&1
DDM_PASS_BLOCKS_PER_SM=0 TUNE_SERIAL=0 python scripts/tune.py base >> gpurun_out/tune_serial.log 2>&1
DDM_PASS_BLOCKS_PER_SM=2 TUNE_SERIAL=0 python scripts/tune.py base >> gpurun_out/tune_serial.log 2>&1
cat gpurun_out/tune_serial.log
DDM_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"upward|downward|finalize|p2p_kernel" -c 4 -o gpurun_out/far_full python scripts/profile_matvec.py 1 > gpurun_out/ncu_far.log 2>&1
tail -3 gpurun_out/ncu_far.log
