#!/usr/bin/env python
"""Condense gpurun_out/ab.txt (tools/gpu_ab.sh) into per-config ratios to the default build."""
import collections
import re
import sys

rows = collections.defaultdict(dict)
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.txt"
for line in open(path):
    if line.startswith("parity"):
        print(line.rstrip())
    m = re.match(r"(\w+ m=\d+ n=\d+(?: walls)?) \[([\w.-]+)\]: best ([\d.]+) ms.* ([\d.]+) GDOF/s", line)
    if m:
        rows[m.group(1)].setdefault(m.group(2), []).append((float(m.group(3)), float(m.group(4))))
for k, d in rows.items():
    base = min(t for t, _ in d["default"])
    print(f"{k:26s}", " ".join(f"{v}:{min(t for t, _ in ts) / base:.3f}" for v, ts in d.items()),
          f"| default {base:.4f} ms {max(g for _, g in d['default']):.1f} GDOF/s")
