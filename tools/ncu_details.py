"""Print the key ncu --set full metrics of every kernel in a report."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.sum",
       "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_fmaheavy.sum",
       "sm__inst_executed_pipe_lsu.sum", "sm__inst_executed_pipe_uniform.sum",
       "sm__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio"]


def run(rep):
    det = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"],
                                         capture_output=True, text=True).stdout.splitlines()))
    h = det[0]
    ci = {x: i for i, x in enumerate(h)}
    cur = None
    for row in det[1:]:
        k = row[ci["ID"]] + " " + row[ci["Kernel Name"]].split("(")[0][-60:]
        if k != cur:
            print("==", k)
            cur = k
        if row[ci["Metric Name"]] in WANT:
            print("   ", row[ci["Metric Name"]], row[ci["Metric Value"]], row[ci["Metric Unit"]])
    raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                         capture_output=True, text=True).stdout.splitlines()))
    h = raw[0]
    for row in raw[2:]:
        print("== raw", row[0], row[4].split("(")[0][-50:])
        for i, x in enumerate(h):
            if x in RAW:
                print("   ", x, row[i])


if __name__ == "__main__":
    run(sys.argv[1])
