"""Executed SASS per query by call site in the query code (tools, not product).
    python tools/sass_callsites.py <report.ncu-rep> <lib.so> <kernel-name substring> <queries> [top]
Joins an ncu capture's per-instruction "Instructions Executed" (source page) with nvdisasm's
inline chains (-gi) and charges each instruction to the innermost frame in sgi_query.cuh (else
sgi_capi.cu / the innermost frame): thread instructions per query, FP64 pipe and total, per
source line and per enclosing function.  The library must be the build that was profiled; the
opcodes are checked instruction by instruction."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

csv.field_size_limit(1 << 30)
FP64 = ("DADD", "DMUL", "DFMA", "DSETP")


def chains(lib, sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   capture_output=True)
    for cub in sorted(os.listdir(tmp)):
        txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)],
                             capture_output=True, text=True).stdout
        for block in txt.split("//--------------------- .text.")[1:]:
            if sub not in block.split(" ", 1)[0]:
                continue
            out, cur, fresh = {}, [], True
            for l in block.splitlines():
                m = re.match(r'\s*//## File "(.*?)", line (\d+)', l)
                if m:
                    if fresh:
                        cur, fresh = [], False
                    cur.append((os.path.basename(m.group(1)), int(m.group(2))))
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?)\s*;", l)
                if m:
                    out[int(m.group(1), 16)] = (list(cur), m.group(2))
                    fresh = True
            return out
    raise SystemExit(f"kernel {sub!r} not found in {lib}")


def functions(path):
    """line -> enclosing function name (the last `name(` definition above the line)."""
    names, cur = {}, "?"
    with open(path) as f:
        for i, l in enumerate(f, 1):
            m = re.match(r"^(?:__device__.*?|\w.*?)\b(\w+)\(", l)
            if m and not l.startswith((" ", "#", "/")) and "__forceinline__" in l or (
                    m and re.match(r"^\S.*\b\w+\(.*\)\s*\{?$", l) and not l.startswith(("//", "#"))):
                cur = m.group(1)
            names[i] = cur
    return names


def main():
    rep, lib, sub, nq = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    ch = chains(lib, sub)
    r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                       capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    hi = [i for i, x in enumerate(rows) if "Address" in x and "Source" in x][0]
    h = rows[hi]
    si, ti = h.index("Source"), h.index("Thread Instructions Executed")
    wi = h.index("Warp Stall Sampling (All Samples)")
    qsrc = os.path.join(os.path.dirname(os.path.abspath(lib)), "csrc", "sgi_query.cuh")
    fn = functions(qsrc) if os.path.exists(qsrc) else {}
    by_line, by_fn = collections.Counter(), collections.Counter()
    fp_line, fp_fn = collections.Counter(), collections.Counter()
    st_line, st_fn = collections.Counter(), collections.Counter()
    mism = 0
    for k, x in enumerate(rows[hi + 1:]):
        if len(x) <= ti:
            continue
        frames, op = ch.get(16 * k, ([], "?"))
        if op.split()[0].lstrip("@!P0123456789T ").split(".")[0] not in x[si]:
            mism += 1
        n = int(x[ti] or 0) / nq
        q = [f for f in frames if f[0] == "sgi_query.cuh"]
        key = q[0] if q else (frames[0] if frames else ("?", 0))
        fkey = fn.get(key[1], "?") if key[0] == "sgi_query.cuh" else key[0]
        isfp = x[si].split()[0].split(".")[0] in FP64 if x[si].split() else False
        by_line[key] += n
        by_fn[fkey] += n
        st_line[key] += int(x[wi] or 0)
        st_fn[fkey] += int(x[wi] or 0)
        if isfp:
            fp_line[key] += n
            fp_fn[fkey] += n
    if mism:
        print(f"WARNING: {mism} opcodes differ between the capture and {lib}")
    print(f"total {sum(by_line.values()):.1f} thread instr/query, FP64 {sum(fp_line.values()):.1f}")
    ts = sum(st_line.values()) or 1
    print(f"{'function':28s} {'instr/q':>8s} {'fp64/q':>8s} {'stall%':>7s}")
    for k, v in by_fn.most_common():
        if v >= 0.05:
            print(f"{k:28s} {v:8.2f} {fp_fn[k]:8.2f} {100 * st_fn[k] / ts:7.2f}")
    print(f"\n{'file:line':28s} {'instr/q':>8s} {'fp64/q':>8s} {'stall%':>7s}")
    keys = sorted(by_line, key=lambda k: -(by_line[k] / max(sum(by_line.values()), 1) + st_line[k] / ts))
    for k in keys[:top]:
        print(f"{k[0] + ':' + str(k[1]):28s} {by_line[k]:8.2f} {fp_line[k]:8.2f} {100 * st_line[k] / ts:7.2f}")


if __name__ == "__main__":
    main()
