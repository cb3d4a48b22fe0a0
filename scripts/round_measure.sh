# bench line + launch list + one ncu --set full capture of the dominant kernel
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
DDM_SERIAL=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"p2p_kernel|p2m_kernel|m2l_kernel|l2p_kernel|prep_sources|finalize" -c 6 -o gpurun_out/full python scripts/profile_matvec.py 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
