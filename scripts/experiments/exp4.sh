cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -k "matvec or poro_fmm or poro_sampled or history" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
TUNE_SERIAL=1 python scripts/tune.py base DDM_SRC_CHUNK=1000000 DDM_SRC_CHUNK=1024 2>&1 | tee gpurun_out/exp4.log
TUNE_SERIAL=0 python scripts/tune.py base DDM_SRC_CHUNK=1000000 2>&1 | tee -a gpurun_out/exp4.log
