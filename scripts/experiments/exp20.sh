cd $GRAFT_REPO_ROOT
python scripts/hist_probe.py 2>&1 | tail -15
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
