"""Key counters of one `ncu --set full` capture (tools, not product):
    python tools/ncu_kernel_summary.py <report.ncu-rep> <queries per launch>
Prints a markdown table: duration, DRAM bytes, FP64 / ALU / issue utilisation, clock, registers,
occupancy, executed SASS per query by opcode, top stall reasons."""
import csv
csv.field_size_limit(1 << 30)
import io
import subprocess
import sys

rep, nq = sys.argv[1], int(sys.argv[2])
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def page(*extra):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", *extra], capture_output=True,
                       text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


raw = page()
h, units, v = raw[0], raw[1], raw[2]
print("| metric | value |\n|---|---|")
for k in KEYS:
    if k in h:
        print(f"| `{k}` | {v[h.index(k)]} {units[h.index(k)]} |")
rd, wr = (float(v[h.index(k)].replace(",", "")) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
mult = {"Gbyte": 1e9, "Mbyte": 1e6, "byte": 1, "Kbyte": 1e3}
ur, uw = units[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_write.sum")]
tot = rd * mult.get(ur, 1) + wr * mult.get(uw, 1)
print(f"\nDRAM traffic per launch: {tot / 1e9:.4f} GB = {tot / nq:.2f} B/query "
      f"(algorithmic 105 B/query = {105 * nq / 1e9:.4f} GB)")
det = page("--print-metric-instances", "details")
op = det[2][det[0].index("sass__inst_executed_per_opcode")]
w = nq / 32
per = [(o.strip(), float(c) / w) for o, c in (it.split(":") for it in op.split("(", 1)[1].rstrip(")").split(";"))]
fp64 = sum(c for o, c in per if o in ("DADD", "DMUL", "DFMA", "DSETP"))
print(f"\nExecuted SASS per query (warp instructions x 32 / queries): total {sum(c for _, c in per):.1f}, "
      f"FP64 pipe (DADD+DMUL+DFMA+DSETP) **{fp64:.1f}**; " + ", ".join(f"{o} {c:.1f}" for o, c in per[:20]))
st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
      and not h[i].endswith("_not_issued")]
st = sorted(st, key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
print("\nTop stall reasons (pc samples): " + ", ".join(f"{k.split('stalled_')[1]} {val}" for k, val in st))
print(f"\nTRAFFIC_BYTES_PER_LAUNCH={tot:.0f}")
