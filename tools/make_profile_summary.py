#!/usr/bin/env python
"""Condense gpurun_out/ ncu artefacts into the tracked profiles/ summary.

  python tools/make_profile_summary.py <launches.csv> <prof.ncu-rep> <key> [round]

Writes/updates profiles/ncu_summary.json:
  launches[<key>]: the cell-map kernel's full-capture metrics (dram bytes per
                   launch = the bench's roofline "traffic", duration, DMMA pipe
                   utilisation, registers, stall mix)
  launch_list[<key>]: per-kernel totals and shares from the
                   `--metrics gpu__time_duration.sum` launch list (cold-cache,
                   serialised: compare shares, not absolutes)
(copy the launch list and `ncu -i <rep> --page details --csv` to profiles/ beside it,
named per round: tools/gpu_bench.sh is the command that produced them).
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    iK, iV, iM = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in data:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = r[iK].split("(")[0].strip()
        tot[k] += float(r[iV].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values()) or 1.0
    return {k: {"launches": cnt[k], "mean_us": tot[k] / cnt[k] / 1e3, "share": tot[k] / T} for k in tot}


def full_capture(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units, v = rr[0], rr[1], rr[2]
    get = {k: (v[i], units[i]) for i, k in enumerate(h)}

    def num(k):
        val, unit = get.get(k, ("nan", ""))
        x = float(val.replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "Ghz": 1e9, "Mhz": 1e6,
                 "Kbyte/block": 1e3}.get(unit, 1.0)
        return x * scale

    out = {
        "kernel": get.get("Kernel Name", ("?", ""))[0],
        "duration_s": num("gpu__time_duration.sum"),
        "dram_read_bytes": num("dram__bytes_read.sum"),
        "dram_write_bytes": num("dram__bytes_write.sum"),
        "dmma_pipe_pct": num("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "shared_pipe_pct": num("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
        "smem_per_block": num("launch__shared_mem_per_block_dynamic"),
        "sm_mhz": num("smsp__cycles_elapsed.avg.per_second") / 1e6,
    }
    out["dram_bytes"] = out["dram_read_bytes"] + out["dram_write_bytes"]
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(val.replace(",", "") or 0)
              for k, (val, _) in get.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    out["stall_share"] = {k: round(x / tot, 3) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    return out


def main():
    launches_csv, rep, key = sys.argv[1], sys.argv[2], sys.argv[3]
    rnd = sys.argv[4] if len(sys.argv) > 4 else "r02"
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(path)) if os.path.exists(path) else {}
    summ["round"] = rnd
    summ["how"] = ("launch list: ncu --metrics gpu__time_duration.sum --clock-control none -c 400 on "
                   "`python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu --no-c3 --no-c5`; full capture: "
                   "ncu --set full --clock-control none -k regex:cellmap -s 3 -c 1 on the same command "
                   "(tools/gpu_bench.sh).  Cold-cache, serialised: shares, not absolutes.")
    summ.setdefault("launches", {})[key] = full_capture(rep)
    if launches_csv != "-":
        summ.setdefault("launch_list", {})[key] = launch_list(launches_csv)
    with open(path, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ["launches"][key], indent=1))


if __name__ == "__main__":
    main()
