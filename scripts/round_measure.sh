# GPU test suite + bench line + launch list + ncu --set full captures of the
# dominant kernels (series FMM: P2P and the far kernels; bbFMM n = 6: M2L)
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
DDM_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"p2p_kernel|p2m_kernel|m2l_kernel|l2p_kernel|prep_stream|finalize" -c 6 -o gpurun_out/full python scripts/profile_matvec.py 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
DDM_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bb_" -c 12 -o gpurun_out/full_bb6 python scripts/profile_matvec.py 1 20 5 bbfmm6 > gpurun_out/ncu_bb.log 2>&1; echo "ncu bb rc=$?"
