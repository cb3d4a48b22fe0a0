# GPU round trip: parity tests, then serial + concurrent stage timings on config 5
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1
echo "TESTS_EXIT $?" >> gpurun_out/gpu_tests.log
tail -4 gpurun_out/gpu_tests.log
TUNE_SERIAL=1 python scripts/tune.py base > gpurun_out/tune.log 2>&1
TUNE_SERIAL=0 python scripts/tune.py base >> gpurun_out/tune.log 2>&1
cat gpurun_out/tune.log
