# node-sharing source stream for the elastic near field: parity + timing
cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/exp15.log
TUNE_SERIAL=1 python scripts/tune.py base 2>&1 | grep total | tee -a gpurun_out/exp15.log
TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total | tee -a gpurun_out/exp15.log
