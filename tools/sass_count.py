"""Count SASS instructions per opcode in each kernel's main body (up to its last EXIT; the
slow-path subroutines of __ddiv_rn/__dsqrt_rn follow it).  Tools, not product.
    python tools/sass_count.py paper_2510_09892_b200/libsgi.so
"""
import re
import subprocess
import sys
from collections import Counter

FP64 = ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "DSET")
txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
for block in re.split(r"\n\s+Function : ", txt)[1:]:
    name = block.split("\n")[0].strip()
    ins = re.findall(r"/\*([0-9a-f]{4,5})\*/\s+((?:@!?U?P\w+\s+)?)([A-Z][A-Z0-9_.]*)", block)
    last_exit = max((i for i, (_, _, op) in enumerate(ins) if op == "EXIT"), default=len(ins) - 1)
    body = Counter(op.split(".")[0] for _, _, op in ins[:last_exit + 1])
    fp64 = sum(body[k] for k in FP64)
    short = re.sub(r"_ZN\d+_GLOBAL__N__\w+?\d+(sgi_\w+?)I?L?i?(\d)?E.*", r"\1<\2>", name)
    print(f"{short[:60]:60s} body={sum(body.values()):5d} FP64={fp64:4d} "
          + " ".join(f"{k}={body[k]}" for k in (*FP64, "MUFU", "FSETP", "FSEL", "SEL", "PLOP3", "LOP3", "IMAD", "IADD3", "ISETP", "LDS", "LDG", "STG", "BRA", "CALL") if body[k]))
