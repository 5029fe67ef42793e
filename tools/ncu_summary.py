"""Summarise an ncu report (details page + selected raw metrics) as text."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
keep = ("Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Active Warps per SM", "Eligible Warps Per Scheduler",
        "No Eligible", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Branch Efficiency", "Memory Throughput", "Grid Size", "Block Size",
        "Local Memory Spilling Requests")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keep:
        print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:40s} {d['Metric Unit']:14s} {d['Metric Value']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u, v = rr[0], rr[1], rr[2]
pat = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct")
for a, b, c in zip(h, u, v):
    if a in pat:
        print(f"{'raw':40s} {a:70s} {b:10s} {c}")
stall = []
for a, b, c in zip(h, u, v):
    if a.startswith("smsp__average_warps_issue_stalled_") and a.endswith("_per_issue_active.ratio"):
        try:
            stall.append((float(c), a))
        except ValueError:
            pass
for val, a in sorted(stall, reverse=True)[:10]:
    print(f"{'stall':40s} {a:70s} {val:.3f}")
