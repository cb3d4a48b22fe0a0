cd $GRAFT_REPO_ROOT
LL_CACHE=none bash scripts/launches.sh
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
recs=[(r[ki].split('(')[0][-25:], r[gi], float(r[vi])) for r in rows[1:]]
last=max(i for i,(k,g,v) in enumerate(recs) if 'prep_sources' in k)
for k,g,v in recs[last:]: print(f"{k:28s} {g:>16s} {v/1e3:8.1f}")
PY
