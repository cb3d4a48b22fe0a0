cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench_r1c.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r1c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], json.dumps(d['gmres']))"
