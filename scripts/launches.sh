# per-kernel durations of one config-5 matvec (ncu launch list, serialised)
cd $GRAFT_REPO_ROOT
DDM_SERIAL=${DDM_SERIAL:-1} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control ${LL_CACHE:-all} --csv \
  --log-file gpurun_out/${LL_O:-launches}.csv python scripts/profile_matvec.py ${LL_REPS:-2} > gpurun_out/ll.log 2>&1
python scripts/launch_table.py gpurun_out/${LL_O:-launches}.csv
