"""Top SASS lines by warp-stall samples from an `ncu --page source --csv
--print-source sass` dump:  python scripts/ncu_hot.py dump.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ai, si, ci = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) > ci and r[ci].replace(".", "", 1).isdigit()]
tot = sum(float(r[ci]) for r in body) or 1.0
print(f"total samples {tot:.0f}")
idx = {id(r): i for i, r in enumerate(body)}
for r in sorted(body, key=lambda r: -float(r[ci]))[:n]:
    print(f"{100 * float(r[ci]) / tot:5.1f}%  {r[ai]}  {r[si][:90]}")
