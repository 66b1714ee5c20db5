"""Source-line stall hot spots of one kernel launch in an ncu report (run in
the dev container): python scripts/ncu_lines.py REPORT KERNEL_REGEX [skip] [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                      "-k", f"regex:{kre}", "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
print(lines[0][:200])
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
li = h.index("# Source") if "# Source" in h else 0
srci = h.index("Source")
data = []
tot = 0
for r in rows[1:]:
    try:
        v = float(r[si])
    except (ValueError, IndexError):
        continue
    tot += v
    data.append((v, r[li], r[srci].strip()[:110]))
data.sort(key=lambda x: -x[0])
print(f"total samples {tot:.0f}")
for v, ln, src in data[:top]:
    print(f"{100 * v / tot:5.1f}%  {ln:>6}  {src}")
