"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total and mean time, share.  Usage: launch_list.py f.csv [--seq]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
seq = []
for r in rows[1:]:
    name = r[ki].replace("<unnamed>::", "").split("(")[0].replace("void ", "").split("<")[0]
    seq.append((int(r[ii]), name, float(r[vi].replace(",", "")) / 1e3))
if "--seq" in sys.argv:
    for i, n, us in seq:
        print(f"{i:5d} {n[:48]:48s} {us:10.1f} us")
agg = defaultdict(lambda: [0, 0.0])
for _, n, us in seq:
    agg[n][0] += 1
    agg[n][1] += us
tot = sum(v[1] for v in agg.values())
for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:48]:48s} n={c:5d} total={us / 1e3:9.3f} ms mean={us / c:9.1f} us share={us / tot:.3f}")
