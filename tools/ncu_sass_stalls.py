"""Stall-reason breakdown of the hottest SASS instructions of one kernel:
  python tools/ncu_sass_stalls.py REPORT KERNEL_REGEX [top]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 10
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kre}", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ci = {x: i for i, x in enumerate(h)}
data = rows[1:]
data.sort(key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: 0.0 for c in cols}
for r in data:
    for c in cols:
        try:
            tot[c] += float(r[ci[c]])
        except ValueError:
            pass
print("kernel totals:", ", ".join(f"{c}={v:g}" for c, v in sorted(tot.items(), key=lambda t: -t[1])[:8]))
for r in data[:top]:
    rs = []
    for c in cols:
        try:
            v = float(r[ci[c]])
        except ValueError:
            continue
        if v > 0:
            rs.append((v, c))
    rs.sort(reverse=True)
    print(f"{r[ci['Address']][-5:]} {r[ci['Warp Stall Sampling (All Samples)']]:>6s} "
          f"{r[ci['Source']].strip()[:60]:60s} " + ", ".join(f"{c[6:]}={v:g}" for v, c in rs[:4]))
