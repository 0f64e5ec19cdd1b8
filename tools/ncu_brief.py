"""Brief ncu summary of one or more .ncu-rep files: headline metrics, DRAM
bytes, pipe utilisation, top stall reasons, instruction mix per opcode.
  python tools/ncu_brief.py REP [REP ...]"""
import collections
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "L2 Hit Rate"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    print(f"== {rep}")
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = {x: i for i, x in enumerate(rows[0])}
    name = rows[1][h["Kernel Name"]].split("(")[0]
    print("   kernel", name)
    seen = set()
    for r in rows[1:]:
        n = r[h["Metric Name"]]
        if n in WANT and n not in seen:
            seen.add(n)
            print(f"   {n}: {r[h['Metric Value']]} {r[h['Metric Unit']]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hh, units, vals = raw[0], raw[1], raw[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"):
        if k in hh:
            i = hh.index(k)
            print(f"   {k}: {vals[i]} {units[i]}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source",
                                           "sass"]))))
    hi = [i for i, r in enumerate(src) if "Source" in r][0]
    sh = {x: i for i, x in enumerate(src[hi])}
    stall = collections.Counter()
    ops = collections.Counter()
    for r in src[hi + 1:]:
        s = r[sh["Source"]].strip()
        op = (s.split()[1] if s.startswith("@") else (s.split()[0] if s else "")).split(".")[0]
        try:
            ops[op] += int(r[sh["Instructions Executed"]] or 0)
        except ValueError:
            pass
        for c in sh:
            if c.startswith("stall_") and "Not Issued" not in c:
                try:
                    stall[c[6:]] += float(r[sh[c]] or 0)
                except ValueError:
                    pass
    tot = sum(stall.values()) or 1
    print("   stall samples:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in stall.most_common(8)))
    te = sum(ops.values()) or 1
    print("   instruction mix:", ", ".join(f"{k} {100 * v / te:.1f}%" for k, v in ops.most_common(12)))
