"""Write profiles/<name>.md from a tools/profile_gpu.sh capture (tools, not product), and record
the per-launch DRAM traffic of each captured kernel in profiles/traffic.json for bench.py.
    python tools/profile_summary.py <tag> <name> [--n 16777216 --config 2]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, name = sys.argv[1], sys.argv[2]
n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 1 << 24
cfg = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else 2
OUT = os.path.join(ROOT, "gpurun_out")


def ncu_csv(rep, page, *extra):
    r = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


lines = [f"# ncu summary `{name}` (capture tag `{tag}`)", "",
         "Command: `tools/profile_gpu.sh` under gpurun on one B200 — bench.py (C2, 2^24 queries per "
         "launch), `--clock-control none`.  Launch-list times are cold-cache and serialised: compare "
         "shares, not absolutes.  Full-set metrics are from one `--set full` capture per kernel.", ""]

# launch list
rows = list(csv.reader(open(os.path.join(OUT, f"{tag}_launches.csv"))))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
lines += ["## Launch list (`gpu__time_duration.sum`, bench.py --steps 5 --warmup 3 --e2e-steps 1)", "",
          "| kernel | launches | total µs | mean µs | share |", "|---|---|---|---|---|"]
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    lines.append(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot:.3f} |")
lines.append("")

traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
for mode in ("eft", "naive"):
    rep = os.path.join(OUT, f"{tag}_{mode}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = ncu_csv(rep, "raw")
    hh, units, vals = raw[0], raw[1], raw[2]
    get = lambda k: (vals[hh.index(k)], units[hh.index(k)]) if k in hh else ("-", "")  # noqa: E731
    lines += [f"## `sgi_intersect_tma_kernel` mode={mode} (`--set full`)", "", "| metric | value |", "|---|---|"]
    for k in KEYS:
        v, u = get(k)
        lines.append(f"| `{k}` | {v} {u} |")
    det = ncu_csv(rep, "raw", "--print-metric-instances", "details")
    op = det[2][det[0].index("sass__inst_executed_per_opcode")]
    warps = n / 32
    per = []
    for item in op.split("(", 1)[1].rstrip(")").split(";"):
        o, c = item.split(":")
        per.append((o.strip(), float(c) / warps))
    fp64 = sum(c for o, c in per if o in ("DADD", "DMUL", "DFMA", "DSETP"))
    lines += ["", f"Executed SASS per query (warp instructions / warps): FP64 pipe "
                  f"(DADD+DMUL+DFMA+DSETP) = **{fp64:.1f}**; top opcodes: " +
              ", ".join(f"{o} {c:.1f}" for o, c in per[:12]), ""]
    stalls = [(hh[i], vals[i]) for i in range(len(hh)) if hh[i].startswith("smsp__pcsamp_warps_issue_stalled_")
              and not hh[i].endswith("_not_issued")]
    stalls = sorted(stalls, key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
    lines += ["Top stall reasons (pc sampling): " + ", ".join(
        f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v}" for k, v in stalls), ""]
    rd, wr = float(get("dram__bytes_read.sum")[0]), float(get("dram__bytes_write.sum")[0])
    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}
    total = rd * scale[get("dram__bytes_read.sum")[1]] + wr * scale[get("dram__bytes_write.sum")[1]]
    traffic[f"{mode}:{cfg}:{n}"] = total
    lines.append(f"DRAM traffic per launch: {total/1e9:.3f} GB (algorithmic 105 B x {n} = {105*n/1e9:.3f} GB)")
    lines.append("")

with open(os.path.join(ROOT, "profiles", f"{name}.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
with open(traffic_path, "w") as f:
    json.dump(traffic, f, indent=1)
print("\n".join(lines))
