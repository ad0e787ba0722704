"""Summarise an ncu report (tools, not product): key details-page metrics, the per-instruction
stall profile from the raw page, and DRAM traffic per launch.
    python tools/ncu_summary.py gpurun_out/<rep>.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
        "Issued Warp Per Scheduler", "No Eligible", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "SM Frequency",
        "Executed Ipc Active", "Block Limit Registers", "Grid Size", "Block Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "sm__cycles_elapsed.avg.per_second", "gpu__time_duration.sum")


def run(args):
    return subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout


for rep in sys.argv[1:]:
    print(f"=== {rep}")
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details"]))))
    h = rows[0]
    si, mi, ui, vi = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    for r in rows[1:]:
        if r[mi] in KEEP:
            print(f"  {r[si][:28]:28s} {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw"]))))
    h, units, vals = raw[0], raw[1], raw[2]
    for k in RAW:
        if k in h:
            i = h.index(k)
            print(f"  raw {k:62s} {vals[i]:>16s} {units[i]}")
    stalls = [(h[i], vals[i]) for i in range(len(h))
              if h[i].startswith("smsp__average_warp_latency_issue_stalled_") or
              (h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("_not_issued"))]
    def f(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    stalls = sorted(stalls, key=lambda kv: -f(kv[1]))[:10]
    for k, v in stalls:
        print(f"  stall {k:70s} {v}")
