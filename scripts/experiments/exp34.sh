# W-list threshold after the node-sharing near field (P2P 28 instead of 36 fp64 instr / pair)
cd $GRAFT_REPO_ROOT
for wm in 24 32 48 64 0; do
  echo -n "w_min=$wm "; DDM_W_MIN=$wm TUNE_SERIAL=0 python scripts/tune.py base 2>&1 | grep total
  echo -n "w_min=$wm serial "; DDM_W_MIN=$wm TUNE_SERIAL=1 python scripts/tune.py base 2>&1 | grep total
done
