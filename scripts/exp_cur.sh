GMRES_CFGS=2,3 python scripts/gmres_timing.py 3 2>&1 | grep solve
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:"cgs_rows" --launch-skip 300 -c 4 --csv python scripts/gmres_ncu.py 3 2>/dev/null | grep -E "cgs_rows" | cut -d, -f5,13-15
