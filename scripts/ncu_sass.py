"""Aggregate the SASS source page of one kernel in an ncu report: instructions
executed and stall samples per opcode, and the hottest instructions.
  python scripts/ncu_sass.py REPORT KERNEL_REGEX [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source=sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ix = {k: h.index(k) for k in h}
agg = collections.defaultdict(lambda: [0, 0, 0])
recs = []
for r in rows[1:]:
    if len(r) != len(h) or r[0] == "Address":
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    th = int(r[ix["Thread Instructions Executed"]] or 0)
    a = agg[op.split(".")[0]]
    a[0] += n
    a[1] += s
    a[2] += th
    recs.append((s, n, r[ix["Address"]][-5:], src[:60]))
tot = sum(v[0] for v in agg.values())
print(f"total warp instructions {tot}")
for op, (n, s, th) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:10s} {n:12d} {100.0*n/tot:6.2f}%  stall_samples {s:7d}  lanes/instr {th/max(n,1):5.1f}")
print("--- hottest by stall samples")
for s, n, a, src in sorted(recs, reverse=True)[:top]:
    print(f"{a} {s:6d} {n:10d}  {src}")
