"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv log:
kernels of the LAST matvec (after the final prep_sources launch)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
recs = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]
last = max(i for i, (k, _) in enumerate(recs) if "prep_sources" in k or "prep_stream" in k or "poro_prep" in k)
end = next((i for i in range(last, len(recs)) if "finalize" in recs[i][0]), len(recs) - 1)
agg = collections.OrderedDict()
for k, v in recs[last:end + 1]:
    name = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    name = name.replace("unnamed>::", "")
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v for _, v in agg.values())
for k, (n, v) in agg.items():
    print(f"{k:40s} {n:4d} launches {v / 1e3:9.1f} us  {100 * v / tot:5.1f} %")
print(f"{'total (serialised)':40s} {sum(n for n, _ in agg.values()):4d} launches {tot / 1e3:9.1f} us")
