cd $GRAFT_REPO_ROOT
for wm in 8 16 24 32 48; do
  echo "w_min=$wm"; DDM_W_MIN=$wm TUNE_SERIAL=1 python scripts/tune.py base 2>&1 | tail -1
  DDM_W_MIN=$wm TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | tail -1
done
