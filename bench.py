#!/usr/bin/env python
"""Benchmark: Hermite DOF-updates/s (FP64), 2D dissipative half step on B200.

Workload (BASELINE.json configs[1], "C2"): 2D periodic dissipative Hermite,
m = 4, 1024 x 1024 nodes, lambda = c dt / h = 0.9, synthetic standing wave
u = sin(2 pi x) sin(2 pi y) cos(2 pi sqrt2 t) from t0 = 0.1.
A step is one half step (dt/2) of the whole grid; a DOF-update is one nodal
coefficient advanced one half step: (m+1)^2 + m^2 = 41 per node.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun, one rank per GPU): weak scaling, each rank owns a
1024 x 1024 slab of a (1024 N) x 1024 periodic grid and exchanges one node
row per half step with its ring neighbour over NCCL.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Hermite DOF-updates/s (FP64) 2D m=4..8 at 1/2/4/8 B200; % of FP64/HBM roofline"
UNIT = "GDOF-updates/s"


def f_alg_diss(m: int) -> int:
    """Canonical symmetric-split live flop count per target cell."""
    def I(mux, muy, rx, ry):
        return 2 * (muy + 1) * (2 * (mux + 1) + rx * 2 * (mux + 1)) + rx * (2 * (muy + 1) + ry * 2 * (muy + 1))

    def N(t, k):
        return 0 if k > t else (t - k) // 2 + 1

    taps = sum(N(2 * m - 1, k) * N(2 * m - 1, l) for k in range(m + 1) for l in range(m + 1))
    taps += sum(N(2 * m - 1, k) * N(2 * m - 1, l) for k in range(m) for l in range(m))
    return (I(m, m, m + 1, m + 1) + I(m, m - 1, 2 * m, 2 * m) + I(m - 1, m, 2 * m, 2 * m)
            + I(m - 1, m - 1, 2 * m, 2 * m) + 3 * (2 * m) ** 2 + 4 * taps + (m + 1) ** 2)


def dof_per_node(m: int) -> int:
    return (m + 1) ** 2 + m * m


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for name, val in zip(names, r[3:7]):
                    if val.lower() == "active":
                        reasons.add(name)
            except Exception:
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ reference (CPU) arm

def cpu_sample(m: int, n: int, rows: int, lam: float = 0.9):
    """One half step of the numpy restatement of the reference (oracle/,
    step for step the reference's own numpy ops; pinned bitwise against the
    reference's golden vectors) on a `rows` x n window of the n x n workload.
    Returns (seconds, DOF-updates)."""
    import numpy as np

    from oracle import hermite_oracle as O

    h = 1.0 / n
    x = O.nodes(0.0, h, n, True, O.PRIMAL)
    xw = x[: rows + 1]
    u = O.planewave_data(xw, x, 0.0, m, m, 1, h, h)
    v = O.planewave_data(xw, x, 0.0, m - 1, m - 1, 1, h, h, tder=1)
    t0 = time.perf_counter()
    # rows+1 source rows are "primal with walls" along x locally -> rows targets
    a = O.gather(u, 0, "x", O.PRIMAL, False, None, None)
    du = np.moveaxis(O.gather(a, 2, "y", O.PRIMAL, True, None, None), 1, 2)
    a = O.gather(v, 0, "x", O.PRIMAL, False, None, None)
    dv = np.moveaxis(O.gather(a, 2, "y", O.PRIMAL, True, None, None), 1, 2)
    uo, vo = O._step_from_corners(du, dv, h, h, m, lam)
    dt = time.perf_counter() - t0
    assert uo.shape[0] == rows
    return dt, rows * n * dof_per_node(m)


def run_reference(args, rank, world):
    if rank != 0:
        return
    m, n = args.m, args.n
    rows = args.ref_rows
    for _ in range(args.warmup):
        cpu_sample(m, n, rows)
    tot_t = tot_d = 0.0
    for _ in range(args.steps):
        t, d = cpu_sample(m, n, rows)
        tot_t += t
        tot_d += d
    val = tot_d / tot_t / 1e9
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"2D periodic dissipative Hermite m={m}, {n}x{n}, lambda 0.9 (C2)",
                   "m": m, "n": n, "sample_rows": rows},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"one half step on a {rows}x{n} window of the {n}x{n} grid per step "
                                   f"(numpy restatement of hermwave.half_step_2d, OpenBLAS threads default)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--ref-rows", type=int, default=16)
    ap.add_argument("--cpu-rows", type=int, default=48)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200 import _lib as L
    from paper_1802_05246_b200.slab import SlabRing

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    m, n = args.m, args.n
    lam = 0.9
    nx_glob = n * world
    grid = hb.Grid2D(0.0, float(world), 0.0, 1.0, nx_glob, n, True)  # h = 1/n on both axes
    h = grid.hx
    cfg = hb.SchemeConfig(m=m, lam=lam)
    dt = cfg.dt(h)
    t0 = 0.1
    w = 2.0 * math.pi
    om = w * math.sqrt(2.0)
    ring = SlabRing(grid, rank, world)

    def init(parity, kx, tder):
        sub = ring.local_grid(parity)
        return hb.standing_wave_on_grid(sub, parity, t0, kx, kx, w, w, om, tder=tder)

    u = init(hb.PRIMAL, m, 0)
    v = init(hb.PRIMAL, m - 1, 1)
    ud = torch.empty_like(u)
    vd = torch.empty_like(v)
    stream = torch.cuda.current_stream()

    def step(src, dst, parity):
        ring.diss2d_step(src[0], src[1], dst[0], dst[1], parity, m, cfg, hb.BoundarySpec2D(), stream.cuda_stream)

    bufs = [(u, v), (ud, vd)]
    parity = hb.PRIMAL
    for i in range(args.warmup):
        step(bufs[i % 2], bufs[(i + 1) % 2], parity)
        parity = hb.flip(parity)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record()
        for i in range(args.steps):
            j = args.warmup + i
            ring.kernel_events = k_ev[i]
            step(bufs[j % 2], bufs[(j + 1) % 2], parity)
            parity = hb.flip(parity)
        stop.record()
        torch.cuda.synchronize()
    ring.kernel_events = None
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    kern_ms = sum(a.elapsed_time(b) for a, b in k_ev) / args.steps
    if world > 1:
        t = torch.tensor([ms, kern_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms = float(t[0]), float(t[1])
    sec = ms / 1e3
    cells_total = nx_glob * n
    dofs = cells_total * dof_per_node(m) * args.steps
    value = dofs / sec / 1e9

    # roofline of the dominant kernel (diss2d_kernel<m>): FP64-pipe bound for m >= 3
    cells_rank = ring.nrows * n
    flops = f_alg_diss(m) * cells_rank
    achieved_tf = flops / (kern_ms / 1e3) / 1e12
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    fp64 = load_json(os.path.join(ROOT, "profiles", "fp64_peak.json")) or {}
    p64 = fp64.get("dfma_tflops")
    p64_src = "measured DFMA microbenchmark (profiles/fp64_peak.json)" if p64 else \
        "datasheet-class 148 SM x 64 FMA x 2 x 1.965 GHz (no measurement found)"
    p64 = p64 or 37.2
    hbm = peaks.get("hbm_gbs", 6562.6)
    bytes_alg = 16 * cells_rank * dof_per_node(m)
    achieved_gbs = bytes_alg / (kern_ms / 1e3) / 1e9
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary_r01.json")) or {}
    traffic = None
    key = f"diss2d_m{m}_n{n}"
    if key in ncu.get("dram_bytes_per_launch", {}):
        traffic = ncu["dram_bytes_per_launch"][key]

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"2D periodic dissipative Hermite m={m}, {n}x{n} nodes per GPU, lambda 0.9 (C2)",
                   "m": m, "nodes_per_gpu": [n, n], "global_nodes": [nx_glob, n], "dof_per_node": dof_per_node(m),
                   "l2": "inputs larger than L2 (u+v = %.0f MB per parity, L2 126 MB)" % (
                       cells_rank * dof_per_node(m) * 8 / 1e6),
                   "parallelism": f"slab{world}" if world > 1 else "single"},
        "roofline": {"bound": "fp64", "achieved": achieved_tf, "peak": p64, "unit": "TFLOP/s",
                     "frac": achieved_tf / p64, "traffic": traffic, "peak_source": p64_src,
                     "flops_per_cell": f_alg_diss(m), "kernel_ms": kern_ms,
                     "hbm": {"achieved": achieved_gbs, "peak": hbm, "unit": "GB/s", "frac": achieved_gbs / hbm,
                             "bytes_per_dof": 16}},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }

    if rank == 0 and world == 1 and not args.no_e2e:
        result["e2e"] = e2e_bench(hb, torch, np, m, n, cfg, min(args.steps, 5))
    if rank == 0 and world == 1 and not args.no_cpu:
        t_cpu, d_cpu = cpu_sample(m, n, args.cpu_rows)
        result["cpu_baseline"] = {"value": d_cpu / t_cpu / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
                                  "sample": f"one half step on a {args.cpu_rows}x{n} window of the {n}x{n} "
                                            f"grid (numpy restatement of hermwave.half_step_2d)"}
    if rank == 0 and world == 1 and not args.no_sweep:
        result["sweep"] = sweep(hb, torch, p64)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_bench(hb, torch, np, m, n, cfg, steps):
    """Same metric through the public drop-in API with host buffers:
    hb.half_step_2d(FieldPair of numpy arrays) per step (H2D + kernel + D2H)."""
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0), tder=0)
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    hu = torch.empty(u.shape, dtype=torch.float64, pin_memory=True)
    hv = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
    hu.copy_(u)
    hv.copy_(v)
    pair = hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.1, hu.numpy()), hb.Field2D(grid, hb.PRIMAL, 0.1, hv.numpy()))
    bc = hb.BoundarySpec2D()
    hb.half_step_2d(pair, cfg, bc)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = pair
    for _ in range(steps):
        p = hb.half_step_2d(p, cfg, bc)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    nbytes = (hu.numel() + hv.numel()) * 8
    return {"value": n * n * dof_per_node(m) * steps / sec / 1e9, "unit": UNIT, "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "api": "paper_1802_05246_b200.half_step_2d(numpy FieldPair)",
            "steps": steps}


def sweep(hb, torch, p64):
    """Config C4: dissipative m = 4..8 at ~2^30 DOF per level (device resident)."""
    out = {}
    sizes = {2: 9088, 3: 6554, 4: 5118, 5: 4196, 6: 3554, 7: 3083, 8: 2721}
    for m in range(4, 9):
        n = sizes[m]
        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
        cfg = hb.SchemeConfig(m=m, lam=0.9)
        w = 2.0 * math.pi
        u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
        v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
        ud, vd = torch.empty_like(u), torch.empty_like(v)
        from paper_1802_05246_b200.stepping import diss2d_into

        bc = hb.BoundarySpec2D()
        bufs = [(u, v), (ud, vd)]
        par = hb.PRIMAL
        for i in range(3):
            diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, par, m, cfg, bc)
            par = hb.flip(par)
        torch.cuda.synchronize()
        k = 6
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(k):
            diss2d_into(*bufs[(i + 3) % 2], *bufs[(i + 4) % 2], grid, par, m, cfg, bc)
            par = hb.flip(par)
        b.record()
        torch.cuda.synchronize()
        sec = a.elapsed_time(b) / 1e3 / k
        g = n * n * dof_per_node(m) / sec / 1e9
        tf = f_alg_diss(m) * n * n / sec / 1e12
        out[f"m{m}"] = {"n": n, "gdof_per_s": g, "ms_per_step": sec * 1e3, "tflops_falg": tf,
                        "frac_fp64": tf / p64, "hbm_gbs": 16 * n * n * dof_per_node(m) / sec / 1e9}
        del u, v, ud, vd, bufs
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
