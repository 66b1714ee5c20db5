"""Stall-reason totals from an `ncu --page source --csv --print-source sass`
dump, excluding the end-of-kernel parking lines (the top BRA.U + ERRBAR):
python scripts/ncu_stalls.py dump.csv"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
si, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) > ai and r[ai].isdigit()]
park = max(body, key=lambda r: int(r[ai]))
tot = Counter()
for r in body:
    if r is park or "ERRBAR" in r[si]:
        continue
    for c in cols:
        v = r[h.index(c)]
        if v.replace(".", "", 1).isdigit():
            tot[c] += float(v)
s = sum(tot.values()) or 1
for c, v in tot.most_common():
    print(f"{c:22s} {100 * v / s:5.1f}%")
