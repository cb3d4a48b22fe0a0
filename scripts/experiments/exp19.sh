# poroelastic near-field cache: parity tests + GMRES timings
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_poro.py tests/test_gpu_precond.py -x -q 2>&1 | tail -3 | tee gpurun_out/exp19.log
python bench.py --steps 20 > gpurun_out/exp19_bench.log 2>&1; tail -1 gpurun_out/exp19_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d['gmres']))" | tee -a gpurun_out/exp19.log
DDM_NEAR_CACHE=0 python bench.py --steps 5 > gpurun_out/exp19_bench0.log 2>&1; tail -1 gpurun_out/exp19_bench0.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nocache', json.dumps(d['gmres']))" | tee -a gpurun_out/exp19.log
