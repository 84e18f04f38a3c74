#!/usr/bin/env python
"""Per-source-line warp-stall samples and executed instructions of an ncu
report (--page source --print-source cuda,sass):  python tools/ncu_lines.py rep [n]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
iL, iS, iW, iE = 0, 1, h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall, inst, text = defaultdict(int), defaultdict(int), {}
cur = None
for r in rows[hdr + 1:]:
    if not r:
        continue
    if r[0] and r[0].isdigit():
        cur = int(r[0])
        text[cur] = r[1]
    try:
        stall[cur] += int(r[iW] or 0)
        inst[cur] += int(r[iE] or 0)
    except (ValueError, IndexError):
        pass
tot = sum(stall.values()) or 1
for ln, s in sorted(stall.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{ln:5d} {100 * s / tot:5.1f}% stall {inst[ln]:11d} inst  {text.get(ln, '')[:90]}")
