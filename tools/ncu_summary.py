#!/usr/bin/env python3
"""Compact text summary of an ncu report (details + key raw metrics + hottest
SASS regions) for profiles/. Usage: ncu_summary.py report.ncu-rep > out.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
hdr = det[0]
print(f"# ncu summary of {rep.split('/')[-1]}")
print(f"kernel: {det[1][hdr.index('Kernel Name')]}")
keep = ("Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "L1/TEX Cache Throughput", "DRAM Throughput",
        "Dynamic Shared Memory Per Block", "Block Size", "Grid Size", "Branch Efficiency")
sec, name, unit, val = (hdr.index(x) for x in ("Section Name", "Metric Name", "Metric Unit",
                                               "Metric Value"))
for r in det[1:]:
    if r[name] in keep:
        print(f"  {r[sec][:28]:28s} {r[name]:40s} {r[val]:>16s} {r[unit]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed"]
print("raw:")
for w in want:
    if w in h:
        print(f"  {w:80s} {v[h.index(w)]}")
for i, n in enumerate(h):
    if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
        try:
            if float(v[i]) > 0.1:
                print(f"  stall {n[34:-23]:30s} {v[i]}")
        except ValueError:
            pass
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
sh, data = sass[1], sass[2:]
ie, src = sh.index("Instructions Executed"), sh.index("Source")
runs, prev, acc, cnt, start = [], None, 0.0, 0, None
for r in data:
    n = float(r[ie] or 0)
    if n < 1e5:
        continue
    key = round(n / 1e5)
    if key != prev:
        if prev is not None:
            runs.append((start, prev * 1e5, cnt, acc))
        prev, start, acc, cnt = key, r[src].strip()[:48], 0.0, 0
    acc += n
    cnt += 1
runs.append((start, prev * 1e5, cnt, acc))
tot = sum(r[3] for r in runs)
print("hottest straight-line SASS runs (executions x instructions):")
for s, n, c, a in sorted(runs, key=lambda x: -x[3])[:12]:
    print(f"  {a / tot * 100:5.1f}%  {n / 1e6:8.2f}M x {c:3d}  first: {s}")
