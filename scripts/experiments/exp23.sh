cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench_r1b.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r1b.log
