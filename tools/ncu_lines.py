#!/usr/bin/env python3
"""Per-source-line instruction counts, shared wavefronts and bank-conflict
excess from an ncu report captured with -lineinfo and --import-source.
Usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = defaultdict(lambda: [0, 0, 0, ""])
cur_file = ""


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0]:
        continue  # SASS rows repeat their source line's totals
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("L1 Wavefronts Shared")
    wx = hdr.index("L1 Wavefronts Shared Excessive")
    a = agg[(cur_file, int(r[0]))]
    a[0] += num(r[ie])
    a[1] += num(r[ws])
    a[2] += num(r[wx])
    a[3] = r[1].strip()
tot = sum(v[0] for v in agg.values())
print(f"# per-line executed warp instructions of {rep.split('/')[-1]} (total {tot:.3e})")
print(f"{'file:line':24s} {'inst%':>6s} {'shared wf':>10s} {'excess':>10s}  source")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0][:16]+':'+str(k[1]):24s} {100*v[0]/tot:6.2f} {v[1]:10.3e} {v[2]:10.3e}  {v[3][:70]}")
