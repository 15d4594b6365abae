"""Top stall lines of an `ncu --page source --csv` export (SASS view with the
source file:line column when built with -lineinfo).  usage: ncu_source_top2.py src.csv [n]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
# the export holds one block per kernel: a "Kernel Name" row, a header row, then instructions
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1][:100]
        h = rows[i + 1]
        j = i + 2
        body = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            if len(rows[j]) > 5:
                body.append(rows[j])
            j += 1
        si, ns = h.index("Source"), h.index("# Samples")
        tot = sum(int(r[ns] or 0) for r in body)
        print("==", name, "samples", tot)
        stall_cols = [k for k, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        agg = defaultdict(int)
        for r in body:
            for k in stall_cols:
                agg[h[k]] += int(r[k] or 0)
        print("   stalls:", ", ".join(f"{k}={v}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]))
        for r in sorted(body, key=lambda r: -int(r[ns] or 0))[:n]:
            print(f"   {int(r[ns]):7d}  {r[si].strip()[:110]}")
        i = j
    else:
        i += 1
