"""Summarise an ncu --set full capture of the step kernel (run here, no GPU).

    python profiles/analyze_ncu.py gpurun_out/<tag>_step.ncu-rep [cells]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else 256.0**3


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("--page", "raw")
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
summary = {}
for d in rows[2:3]:
    for w in want:
        if w in hdr:
            summary[w] = d[hdr.index(w)]
            print(f"{w:62s} {d[hdr.index(w)]} {units[hdr.index(w)]}")
    st = [(hdr[i], float(d[i])) for i in range(len(hdr))
          if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled") and d[i].replace(".", "").isdigit()]
    st.sort(key=lambda x: -x[1])
    tot = sum(v for _, v in st) or 1
    print("stalls: " + ", ".join(f"{h.split('stalled_')[1]} {v / tot * 100:.0f}%" for h, v in st[:8]))
rows = page("--page", "source", "--print-source", "sass")
hdr = rows[1]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0].startswith("Kernel"):
        break
    data.append(r)
tot = sum(int(r[i_ex]) for r in data if r[i_ex].isdigit())
print(f"warp-instructions per 32-cell warp-plane: {tot / (cells / 32):.1f}")
c = Counter()
for r in data:
    if r[i_ex].isdigit():
        toks = r[i_src].split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c[op.split(".")[0]] += int(r[i_ex])
print("mix: " + " ".join(f"{op}:{v / tot * 100:.1f}%" for op, v in c.most_common(16)))
