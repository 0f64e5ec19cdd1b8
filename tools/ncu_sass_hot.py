"""Per-SASS-instruction execution counts and stall samples of one kernel in an
ncu report (needs the report's source page).  Usage:
  python tools/ncu_sass_hot.py REPORT KERNEL_REGEX [top]"""
import csv
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ci = {x: i for i, x in enumerate(h)}
data = rows[1:]
tot = sum(int(r[ci["Instructions Executed"]] or 0) for r in data)
samp = sum(int(r[ci["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total warp-instructions", tot, "stall samples", samp)
ops = Counter()
for r in data:
    op = r[ci["Source"]].split()[0] if r[ci["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ci["Source"]].split()[1]
    ops[op.split(".")[0]] += int(r[ci["Instructions Executed"]] or 0)
print("by opcode:")
for op, c in ops.most_common(25):
    print(f"  {op:10s} {c:12d} {c / tot:6.3f}")
print("hottest stall addresses:")
data.sort(key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))
for r in data[:top]:
    print(f"  {r[ci['Warp Stall Sampling (All Samples)']]:>6s} {r[ci['Instructions Executed']]:>10s}  {r[ci['Source']].strip()[:90]}")
