"""Attribute an ncu SASS-page CSV (instructions executed, stall samples) to
CUDA source lines using the cubin's line table (dev tool).

    python profiles/sass_lines.py <cubin> <mangled kernel> <ncu_sass.csv> [top]
"""
import csv
import re
import subprocess
import sys
from collections import defaultdict


def line_map(cubin, kernel):
    elf = subprocess.run(["cuobjdump", "-elf", cubin], capture_output=True, text=True).stdout
    idx, in_sym = None, False
    for ln in elf.splitlines():
        in_sym = in_sym or ln.startswith(".section .symtab")
        f = ln.split()
        if in_sym and len(f) == 7 and f[-1] == kernel:
            idx = int(f[0], 16)
            break
    out = subprocess.run(["nvdisasm", "-g", "-fun", str(idx), cubin], capture_output=True,
                         text=True).stdout
    cur, m = None, {}
    for ln in out.splitlines():
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = f"{g.group(1).split('/')[-1]}:{g.group(2)}"
            continue
        a = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if a:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    cubin, kernel, sass = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    m = line_map(cubin, kernel)
    rows = list(csv.reader(open(sass)))
    hdr = rows[1]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
        "Warp Stall Sampling (All Samples)")
    base = None
    inst, stall = defaultdict(float), defaultdict(float)
    tot_i = tot_s = 0.0
    for r in rows[2:]:
        if len(r) <= ie or not r[ia].startswith("0x"):
            continue
        addr = int(r[ia], 16)
        base = addr if base is None else base
        key = m.get(addr - base, "?")
        inst[key] += float(r[ie] or 0)
        stall[key] += float(r[iss] or 0)
        tot_i += float(r[ie] or 0)
        tot_s += float(r[iss] or 0)
    print(f"total inst {tot_i:.0f}, stall samples {tot_s:.0f}")
    for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{k:28s} inst {100 * v / tot_i:5.1f}%  stall {100 * stall[k] / max(tot_s, 1):5.1f}%")


if __name__ == "__main__":
    main()
