"""Turn the ncu outputs of tools/make_profiles.sh into the committed evidence:
  profiles/<tag>_launches.csv   per-kernel-type summary of one C3 step (launch list)
  profiles/<tag>_full.txt       key --set full metrics of the four kernels (largest tensor)
  profiles/traffic.json         DRAM bytes per launch of each kernel over the step
Usage: python tools/profile_summary.py TAG"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "gpurun_out")
dst = os.path.join(root, "profiles")
os.makedirs(dst, exist_ok=True)

k = ncu_summary.load(os.path.join(src, f"{tag}_launches.csv"))
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for d in k.values():
    a = agg[d["name"].split("<")[0]]
    a[0] += 1
    a[1] += d["gpu__time_duration.sum"]
    a[2] += d.get("dram__bytes_read.sum", 0)
    a[3] += d.get("dram__bytes_write.sum", 0)
T = sum(a[1] for a in agg.values())
buf = io.StringIO()
w = csv.writer(buf)
w.writerow(["kernel", "launches", "total_us", "share_of_step", "avg_us", "dram_read_bytes",
            "dram_write_bytes", "dram_bytes_per_launch", "dram_GBps"])
traffic = {}
for name, (n, t, r, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    w.writerow([name, n, round(t, 1), round(t / T, 4), round(t / n, 2), int(r), int(wr),
                int((r + wr) / n), round((r + wr) / t / 1e3, 1)])
    traffic[name] = {"launches": n, "dram_bytes_per_launch": (r + wr) / n,
                     "share_of_step": t / T, "avg_us": t / n}
open(os.path.join(dst, f"{tag}_launches.csv"), "w").write(
    "# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
    "--clock-control none over one C3 step (tools/make_profiles.sh); serialised and "
    "cold-cache: compare shares, not absolutes\n" + buf.getvalue())
json.dump({"source": f"profiles/{tag}_launches.csv", "kernels": traffic},
          open(os.path.join(dst, "traffic.json"), "w"), indent=1)
rep = os.path.join(src, f"{tag}_full.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_details.py"), rep],
                         capture_output=True, text=True).stdout
    open(os.path.join(dst, f"{tag}_full.txt"), "w").write(
        "# ncu --set full --clock-control none, largest C3 tensor (bn1 input, 256x64x112x112 "
        "fp32), tools/make_profiles.sh\n" + out)
for suffix, what in (("c4_full", "largest C4 tensor (1024x64x112x112 bf16, mixed widths)"),
                     ("adapt_full", "NEXT-3 kernels: K6 grad_sqnorm on the largest C3 (fp32) and "
                                    "C4 (bf16) tensors, K5 stage 2 on 311 layers x 1024 samples")):
    rep = os.path.join(src, f"{tag}_{suffix}.ncu-rep")
    if os.path.exists(rep):
        out = subprocess.run([sys.executable, os.path.join(root, "tools", "ncu_details.py"), rep],
                             capture_output=True, text=True).stdout
        open(os.path.join(dst, f"{tag}_{suffix}.txt"), "w").write(
            f"# ncu --set full --clock-control none, {what}, tools/make_profiles.sh\n" + out)
print(buf.getvalue())
