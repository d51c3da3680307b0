#!/usr/bin/env python3
"""Registers / spills per kernel from nvcc -Xptxas -v output (build/ptxas.log)."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1605_00854_b200/build/ptxas.log").read()
cur = None
rows = []
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:  # the entry's own line and its out-of-line device functions': keep the sum
        cur["spill"] = cur.get("spill", 0) + int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
for r, n in zip(rows, names):
    short = n.split("(")[0].replace("pbn_b200::", "").replace("void ", "")
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', 0):>4} B  {short}")
