#!/usr/bin/env python
"""Summarise an ncu report: key SOL metrics, per-opcode instruction mix and
the top stall sites.   python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
want = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "L2 Hit Rate", "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "SM Frequency", "Dynamic Shared Memory Per Block", "Memory Throughput")
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:45s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
vals = rr[2] if len(rr) > 2 else rr[1]
for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed_op_dmma.sum", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "gpu__time_duration.sum"):
    for i, k in enumerate(hh):
        if k == key:
            print(f"{key:60s} {vals[i]} {rr[1][i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot_s = sum(int(r[iW] or 0) for r in data) or 1
tot_e = sum(int(r[iE] or 0) for r in data) or 1
ops, opss = Counter(), Counter()
for r in data:
    t = r[iS].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    ops[op] += int(r[iE] or 0)
    opss[op] += int(r[iW] or 0)
print(f"instructions {tot_e}  stall samples {tot_s}")
for op, c in ops.most_common(18):
    print(f"  {op:10s} {c:12d} {100 * c / tot_e:5.1f}%  stall {100 * opss[op] / tot_s:5.1f}%")
print("top stall sites:")
for r in sorted(data, key=lambda r: -int(r[iW] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {r[0][-5:]} {r[iS][:64]:64s} {r[iW]:>6s} {r[iE]:>10s}")
