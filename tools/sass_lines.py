"""Attribute an ncu capture's per-SASS-instruction metrics (warp-stall samples, instructions
executed) to CUDA source lines via nvdisasm's line info (tools, not product).
    python tools/sass_lines.py <report.ncu-rep> <lib.so> <kernel-name substring> [top]
The library must be the build that was profiled (compiled with -lineinfo)."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

csv.field_size_limit(1 << 30)
rep, lib, sub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines = {}
for cub in os.listdir(tmp):
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout
    for block in txt.split("//--------------------- .text.")[1:]:
        name = block.split(" ", 1)[0]
        if sub not in name:
            continue
        cur = ("?", 0)
        for l in block.splitlines():
            m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
            if m:
                lines[int(m.group(1), 16)] = cur
        break
r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                   capture_output=True, text=True)
rows = list(csv.reader(r.stdout.splitlines()))
hi = [i for i, x in enumerate(rows) if "Address" in x and "Source" in x][0]
h = rows[hi]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
samp, inst = collections.Counter(), collections.Counter()
for k, x in enumerate(rows[hi + 1:]):
    key = lines.get(16 * k, ("?", 0))
    samp[key] += int(x[si] or 0)
    inst[key] += int(x[ei] or 0)
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
byfile_s, byfile_i = collections.Counter(), collections.Counter()
for (f, _), v in samp.items():
    byfile_s[f] += v
for (f, _), v in inst.items():
    byfile_i[f] += v
print("by file: " + ", ".join(f"{f} {100 * byfile_s[f] / ts:.1f}% stalls / {100 * byfile_i[f] / ti:.1f}% instr"
                             for f in sorted(byfile_i, key=lambda f: -byfile_i[f])))
print(f"{'file:line':40s} {'stall%':>7s} {'instr%':>7s}")
for key in sorted(set(samp) | set(inst), key=lambda k: -(samp[k] / ts + inst[k] / ti))[:top]:
    print(f"{key[0] + ':' + str(key[1]):40s} {100 * samp[key] / ts:7.2f} {100 * inst[key] / ti:7.2f}")
