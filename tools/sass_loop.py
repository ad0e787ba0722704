"""Opcode histogram of a kernel's hottest loop body in SASS (tools, not product): from the
first instruction matching --start (default: the mbarrier TRYWAIT) to the backward branch that
closes the loop.
    python tools/sass_loop.py <lib.so> <function-substring> [start-regex]
"""
import re
import subprocess
import sys
from collections import Counter

lib, fun = sys.argv[1], sys.argv[2]
start = sys.argv[3] if len(sys.argv) > 3 else "TRYWAIT"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
block = next(b for b in re.split(r"\n\s+Function : ", txt)[1:] if fun in b.split("\n")[0])
ins = re.findall(r"/\*([0-9a-f]{4,5})\*/\s+((?:@!?U?P\w+\s+)?)([A-Z][A-Z0-9_.]*)([^;]*);", block)
i0 = next(i for i, x in enumerate(ins) if re.search(start, x[2] + x[3]))
a0 = int(ins[i0][0], 16)
body = []
for addr, pred, op, args in ins[i0:]:
    body.append(op.split(".")[0])
    if op.startswith("BRA"):
        m = re.search(r"0x([0-9a-f]+)", args)
        if m and int(m.group(1), 16) < a0:
            break
c = Counter(body)
fp64 = sum(c[k] for k in ("DADD", "DMUL", "DFMA", "DSETP"))
print(f"loop body {len(body)} instructions, FP64 {fp64}, other {len(body) - fp64}")
print(" ".join(f"{k}={v}" for k, v in c.most_common()))
