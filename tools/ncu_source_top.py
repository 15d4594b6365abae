"""Top source lines / stall reasons of an `ncu --page source --csv
--print-source cuda,sass` export.  Usage: python tools/ncu_source_top.py f.csv [N]"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
data, h, cur = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        h = r
        continue
    data.append((cur, r))
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
src = [(f, r) for f, r in data if r[0] != "" and len(r) == len(h)]
tot = sum(num(r[si]) for f, r in src) or 1.0
for f, r in sorted(src, key=lambda x: -num(x[1][si]))[:N]:
    print(f"{num(r[si]) / tot * 100:5.1f}% {f}:{r[0]} ie={r[ie]} {r[1].strip()[:90]}")
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
t = {h[i]: 0.0 for i in cols}
for f, r in src:
    if len(r) != len(h):
        continue
    for i in cols:
        t[h[i]] += num(r[i])
s = sum(t.values()) or 1.0
print({k: round(v / s * 100, 1) for k, v in sorted(t.items(), key=lambda x: -x[1])[:8]})
