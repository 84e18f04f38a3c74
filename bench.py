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
row per half step with its ring neighbour (torch.distributed P2P over NCCL),
so the per-N values are the same per-GPU workload as N = 1.

Extra keys beside the contract's: "c5" at every N (BASELINE configs[4]:
m=6, strong scaling at 8192^2 and 16384^2 (N >= 4), weak at 2048N x 16384,
through the slab ring), and at N = 1 "c3" (conservative m=5, 2048^2,
Dirichlet/Neumann walls — configs[2], with its energy drift) and "sweep"
(dissipative m=2..8 at ~2^30 DOF per level — configs[3]), all device
resident.  --config c5 makes C5's weak-scaling slab the top-level workload.
"""

from __future__ import annotations

import argparse
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
SWEEP_N = {2: 9088, 3: 6554, 4: 5118, 5: 4196, 6: 3554, 7: 3083, 8: 2721}  # ~2^30 DOF


# --------------------------------------------------------------- roofline model

def _I(mux, muy, rx, ry):
    return 2 * (muy + 1) * (2 * (mux + 1) + rx * 2 * (mux + 1)) + rx * (2 * (muy + 1) + ry * 2 * (muy + 1))


def _N(t, k):
    return 0 if k > t else (t - k) // 2 + 1


def f_alg_diss(m: int) -> int:
    """Canonical symmetric-split live flop count per target cell, dissipative."""
    taps = sum(_N(2 * m - 1, k) * _N(2 * m - 1, l) for k in range(m + 1) for l in range(m + 1))
    taps += sum(_N(2 * m - 1, k) * _N(2 * m - 1, l) for k in range(m) for l in range(m))
    return (_I(m, m, m + 1, m + 1) + _I(m, m - 1, 2 * m, 2 * m) + _I(m - 1, m, 2 * m, 2 * m)
            + _I(m - 1, m - 1, 2 * m, 2 * m) + 3 * (2 * m) ** 2 + 4 * taps + (m + 1) ** 2)


def f_alg_cons(m: int) -> int:
    """Canonical flop count per target cell, conservative."""
    taps = sum(_N(2 * m + 1, k) * _N(2 * m + 1, l) for k in range(m + 1) for l in range(m + 1))
    return _I(m, m, 2 * m + 2, 2 * m + 2) + 2 * taps + 2 * (m + 1) ** 2


def dof_per_node(m: int, scheme: str = "diss") -> int:
    return (m + 1) ** 2 + m * m if scheme == "diss" else (m + 1) ** 2


# csrc/cellmap_shape.h cm_lmask: classes whose left-over outputs run on CUDA cores
HYBRID_MASK = {("cons", 5): 0xF, ("diss", 6): 0x1, ("diss", 8): 0x1, ("cons", 8): 0x1}


def cellmap_flops(m: int, scheme: str = "diss"):
    """(dense, issued) FP64 flops per target cell of the cell-map kernel:
    dense = 2 D_out D_in (the class maps, unpadded); issued = the DMMA tiles
    actually executed (outputs padded to 8 per class, inputs to 4 per field)
    plus, for hybrid-tile orders, the left-over outputs' CUDA-core FMAs."""
    w0, w1 = m + 1, (m if scheme == "diss" else 0)
    din, dout = w0 * w0 + w1 * w1, w0 * w0 + w1 * w1
    if scheme == "cons":
        din = dout = w0 * w0

    def cnt(w, p):
        return (w - 1 - p) // 2 + 1 if w > p else 0

    ncls = [cnt(w0, c >> 1) * cnt(w0, c & 1) + cnt(w1, c >> 1) * cnt(w1, c & 1) for c in range(4)]
    kslots = 4 * ((w0 * w0 + 3) // 4) + 4 * ((w1 * w1 + 3) // 4)
    mask = HYBRID_MASK.get((scheme, m), 0)
    left = [n % 8 if mask >> c & 1 else 0 for c, n in enumerate(ncls)]
    nslots = sum(8 * (n // 8) if left[c] else 8 * ((n + 7) // 8) for c, n in enumerate(ncls)) + sum(left)
    return 2 * din * dout, 2 * kslots * nslots


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def peaks():
    mp = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    fp = load_json(os.path.join(ROOT, "profiles", "fp64_peak.json")) or {}
    dmma = fp.get("dmma_tflops")
    return {"hbm_gbs": mp.get("hbm_gbs", 6650.0), "hbm_src": "measured" if "hbm_gbs" in mp else "fallback",
            "dmma_tflops": dmma or 37.2, "dmma_src": "measured (tools/fp64_peak.cu)" if dmma else "datasheet-class"}


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
#
# The reference is pure Python/numpy.  It is installed UNMODIFIED into
# baseline/_ref (pip install --no-index --target baseline/_ref
# of /root/reference/pkg); that copy travels to the GPU box with the repo.
# Each CPU sample runs the reference's own public hermwave.half_step_2d on a
# periodic n x R strip with the C2 spacing (h = 1/n on both axes), m, lambda
# and standing-wave data, i.e. R rows of the C2 grid's work: the per-node
# arithmetic is data-independent, so DOF-updates/s of the strip is C2's rate.
# A whole C2 half step would take the reference ~135 s and ~40 GiB (SURVEY
# §8a row 15).  Without baseline/_ref the numpy restatement in oracle/ stands
# in ("port").

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
STRIP_ROWS = 4


def _standing_blocks(xn, yn, t, k, h, tder):
    """Scaled blocks (h^a/a!)(h^b/b!) d_x^a d_y^b d_t^tder of
    sin(2 pi x) sin(2 pi y) cos(2 pi sqrt2 t) (the GPU arm's synthetic data)."""
    import numpy as np

    w = 2.0 * math.pi
    om = w * math.sqrt(2.0)
    out = np.empty((len(xn), len(yn), k + 1, k + 1))
    ft = om**tder * math.cos(om * t + 0.5 * math.pi * tder)
    for a in range(k + 1):
        fx = w**a * np.sin(w * xn + 0.5 * math.pi * a) * h**a / math.factorial(a)
        for b in range(k + 1):
            fy = w**b * np.sin(w * yn + 0.5 * math.pi * b) * h**b / math.factorial(b)
            out[:, :, a, b] = fx[:, None] * fy[None, :] * ft
    return out


def _strip_stepper(m: int, n: int, rows: int, kind: str):
    """A closure running one half step of the reference (or its port) on the
    n x rows periodic strip; returns (step, DOF-updates per step)."""
    import numpy as np

    h = 1.0 / n
    x = h * np.arange(n)
    y = h * np.arange(rows)
    u = _standing_blocks(x, y, 0.1, m, h, 0)
    v = _standing_blocks(x, y, 0.1, m - 1, h, 1)
    dof = n * rows * dof_per_node(m)
    if kind == "reference":
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import hermwave as hw  # the unmodified reference (baseline/_ref)
        from hermwave.boundary import BoundarySpec2D
        from hermwave.grid import PRIMAL, Field2D, FieldPair, Grid2D

        grid = Grid2D(0.0, 1.0, 0.0, rows * h, n, rows, True)
        pair = FieldPair(Field2D(grid, PRIMAL, 0.1, u), Field2D(grid, PRIMAL, 0.1, v))
        cfg, bc = hw.SchemeConfig(m=m, lam=0.9), BoundarySpec2D()
        return (lambda: hw.half_step_2d(pair, cfg, bc)), dof
    from oracle import hermite_oracle as O

    return (lambda: O.half_step_2d(u, v, O.PRIMAL, n, rows, True, h, h, m, 0.9)), dof


def ref_kind() -> str:
    return "reference" if os.path.isdir(os.path.join(REF_DIR, "hermwave")) else "port"


def _cpu_worker(m, n, rows, kind, rounds, bar, q):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):  # one BLAS thread per worker process
        step, _ = _strip_stepper(m, n, rows, kind)
        for _ in range(rounds):
            bar.wait()
            t0 = time.time()
            step()
            t1 = time.time()
            q.put((t0, t1))


def cpu_workers(m: int, n: int, rows: int) -> int:
    """Worker processes: every host core, capped so the reference's
    intermediates (~38 KiB per node at m = 4, scaling as the map size;
    SURVEY §8c) stay under a quarter of the host's available memory."""
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    per = n * rows * 40e3 * (dof_per_node(m) / 41.0) ** 2
    return max(1, min(os.cpu_count() or 1, 128, int(0.25 * avail / per)))


def cpu_sample(m: int, n: int, rows: int, rounds: int = 1, warm: int = 0, workers: int | None = None):
    """W processes (one BLAS thread each) each run the reference's half step on
    their own n x rows strip per round, all starting together (barrier).
    Returns (mean timed round wall seconds, DOF-updates per round, W, kind)."""
    import multiprocessing as mp

    kind = ref_kind()
    w = workers or cpu_workers(m, n, rows)
    ctx = mp.get_context("spawn")  # (the parent may hold CUDA state and threads)
    bar = ctx.Barrier(w)
    q = ctx.Queue()
    tot = warm + rounds
    procs = [ctx.Process(target=_cpu_worker, args=(m, n, rows, kind, tot, bar, q)) for _ in range(w)]
    for p in procs:
        p.start()
    spans = [q.get(timeout=900) for _ in range(w * tot)]
    for p in procs:
        p.join(timeout=60)
    spans.sort()  # rounds are barrier-separated: group the w reports of each round
    walls = []
    for r in range(tot):
        grp = spans[r * w:(r + 1) * w]
        walls.append(max(t1 for _, t1 in grp) - min(t0 for t0, _ in grp))
    walls = walls[warm:]
    return sum(walls) / len(walls), w * n * rows * dof_per_node(m), w, kind


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(m: int, n: int, rows: int, rounds: int, warm: int):
    """All-core rate and the single-core (1 process, 1 BLAS thread) rate."""
    sec, d, w, kind = cpu_sample(m, n, rows, rounds=rounds, warm=warm)
    sec1, d1, _, _ = cpu_sample(m, n, rows, rounds=max(1, min(rounds, 2)), warm=1, workers=1)
    what = "hermwave.half_step_2d, the unmodified reference (baseline/_ref)" if kind == "reference" else \
        "oracle/ numpy restatement of hermwave.half_step_2d"
    return {"value": d / sec / 1e9, "unit": UNIT, "cores": w, "kind": kind,
            "sample": f"{w} processes (1 BLAS thread each), each one half step of {what} on a periodic "
                      f"{n}x{rows} strip with the C2 spacing h=1/{n}, m={m}, lambda 0.9, standing-wave data, "
                      f"per round; {rounds} timed round(s) after {warm} warm-up",
            "single_core": {"value": d1 / sec1 / 1e9, "unit": UNIT, "cores": 1},
            "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}, sec, d


def run_reference(args, rank, world):
    if rank != 0:
        return
    m, n, rows = args.m, args.n, args.ref_rows
    # every requested step runs (each a bounded sample: one strip half step per
    # core, ~0.5 s at m = 4), up to 60 timed and 5 warm-up rounds
    n_warm, n_timed = min(max(args.warmup, 1), 5), min(max(args.steps, 1), 60)
    cb, sec, d = cpu_baseline(m, n, rows, n_timed, n_warm)
    val = cb["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": n_timed, "warmup": n_warm, "requested": {"steps": args.steps, "warmup": args.warmup},
        # one C2 half step (n^2 nodes) at the measured rate
        "ms_per_step": 1e3 * n * n * dof_per_node(m) / (val * 1e9),
        "ms_per_round": 1e3 * sec,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic standing wave (no dataset)",
        "config": {"workload": f"2D periodic dissipative Hermite m={m}, {n}x{n} nodes per GPU, lambda 0.9 (C2)",
                   "m": m, "n": n, "strip_rows_per_worker": rows, "workers": cb["cores"]},
        "cpu_baseline": cb,
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def slab_run(hb, torch, dist, ring, m, steps, warmup, stream, events=True):
    """Device-resident dissipative half steps of this rank's slab of ring.grid
    (standing wave from t0 = 0.1), timed with CUDA events on the
    launching stream between barriers; returns (ms total, mean kernel ms)."""
    grid = ring.grid
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    w = 2.0 * math.pi  # u = sin(2 pi x) sin(2 pi y) cos(2 pi sqrt2 t) (h = 1/ny, y extent 1)
    om = w * math.sqrt(2.0)

    def init(parity, k, tder):
        return hb.standing_wave_on_grid(grid, parity, 0.1, k, k, w, w, om, tder=tder,
                                        rows=(ring.row0, ring.nrows(parity)))

    u, v = init(hb.PRIMAL, m, 0), init(hb.PRIMAL, m - 1, 1)
    bufs = [(u, v), (torch.empty_like(u), torch.empty_like(v))]
    bc = hb.BoundarySpec2D()
    parity = hb.PRIMAL

    def step(i, par):
        ring.diss2d_step(*bufs[i % 2], *bufs[(i + 1) % 2], par, m, cfg, bc, stream.cuda_stream)

    for i in range(warmup):
        step(i, parity)
        parity = hb.flip(parity)
    torch.cuda.synchronize()
    if ring.world > 1:
        dist.barrier()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # the timed region: back-to-back steps, no per-step events (an event record between two
    # launches would break the programmatic dependent launch that chains them)
    start.record(stream)
    for i in range(steps):
        step(warmup + i, parity)
        parity = hb.flip(parity)
    stop.record(stream)
    torch.cuda.synchronize()
    if ring.world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    # then each step's launch(es) bracketed by events on the launching stream: the kernel's own
    # average duration (the roofline denominator), PDL overlap excluded
    kern_ms = float("nan")
    if events:
        nk = min(steps, 20)
        k_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nk)]
        for i in range(nk):
            ring.kernel_events = k_ev[i]
            step(warmup + steps + i, parity)
            parity = hb.flip(parity)
        torch.cuda.synchronize()
        ring.kernel_events = None
        kern_ms = sum(a.elapsed_time(b) for a, b in k_ev) / nk
    if ring.world > 1:  # the job's time is the slowest rank's
        t = torch.tensor([ms, kern_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms = float(t[0]), float(t[1])
    del u, v, bufs
    torch.cuda.empty_cache()
    return ms, kern_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c5"],
                    help="top-level workload: c2 (default; weak-scaled 1024^2 per GPU at N > 1) or c5 "
                         "(m=6, 2048 N x 16384 periodic, 2048 x 16384 per GPU: BASELINE configs[4] weak scaling)")
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--ref-rows", type=int, default=STRIP_ROWS)
    ap.add_argument("--cpu-rows", type=int, default=STRIP_ROWS)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        # NCCL's init lines (ranks, rings/NVLS, transports) to stderr: stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.slab import SlabRing

    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        chk = torch.ones(1, device="cuda")
        dist.all_reduce(chk)
        comm = {"backend": dist.get_backend(), "world": dist.get_world_size(),
                "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()),
                "allreduce_check": float(chk) == float(world)}
    stream = torch.cuda.current_stream()
    pk = peaks()
    if args.config == "c5":
        m, ny, rows_per = 6, 16384, 2048
        workload = f"C5 (BASELINE configs[4]) weak scaling: 2D periodic dissipative Hermite m=6, " \
                   f"{rows_per * world}x{ny} nodes ({rows_per}x{ny} per GPU), lambda 0.9"
    else:
        m, ny, rows_per = args.m, args.n, args.n
        workload = f"2D periodic dissipative Hermite m={m}, {rows_per}x{ny} nodes per GPU, lambda 0.9 (C2)"
    nx_glob = rows_per * world
    grid = hb.Grid2D(0.0, nx_glob / ny, 0.0, 1.0, nx_glob, ny, True)  # h = 1/ny on both axes
    ring = SlabRing(grid, rank, world)
    ms, kern_ms = 0.0, 0.0
    with ClockSampler(local) as clk:
        ms, kern_ms = slab_run(hb, torch, dist, ring, m, args.steps, args.warmup, stream)
    sec = ms / 1e3
    dofs = nx_glob * ny * dof_per_node(m) * args.steps
    value = dofs / sec / 1e9

    # roofline of the dominant kernel (cellmap_kernel<m, diss>): FP64 tensor
    # pipe (DMMA).  achieved = SURVEY §8d's canonical flops per cell x cells /
    # kernel time; "dense"/"issued" are what this kernel's cell maps execute.
    cells_rank = ring.nrows(hb.PRIMAL) * ny
    # the kernel's average launch duration over the timed region: at N = 1 a step is exactly one
    # launch (PDL chains them back to back); at N > 1 the event-bracketed pass (interior + halo row)
    kernel_ms_timed = ms / args.steps if world == 1 else kern_ms
    ksec = kernel_ms_timed / 1e3
    achieved = f_alg_diss(m) * cells_rank / ksec / 1e12
    dense, issued = cellmap_flops(m)
    bytes_alg = 16 * cells_rank * dof_per_node(m)
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {}
    traffic = (ncu.get("launches", {}).get(f"diss_m{m}_n{ny}") or {}).get("dram_bytes")
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": pk["dmma_tflops"], "unit": "TFLOP/s",
        "frac": achieved / pk["dmma_tflops"], "traffic": traffic,
        "peak_source": pk["dmma_src"] + ": FP64 DMMA (mma.sync m8n8k4 f64) — the tensor path this kernel runs on",
        "flops_per_cell_alg": f_alg_diss(m), "kernel_ms": kernel_ms_timed,
        "kernel_ms_standalone": kern_ms,
        "dense_map_tflops": dense * cells_rank / ksec / 1e12,
        "issued_dmma_tflops": issued * cells_rank / ksec / 1e12,
        "issued_frac": issued * cells_rank / ksec / 1e12 / pk["dmma_tflops"],
        "hbm": {"achieved": bytes_alg / ksec / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": bytes_alg / ksec / 1e9 / pk["hbm_gbs"], "bytes_per_dof": 16, "peak_source": pk["hbm_src"]},
    }
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic standing wave (no dataset)",
        "config": {"workload": workload, "m": m, "nodes_per_gpu": [ring.nrows(hb.PRIMAL), ny],
                   "global_nodes": [nx_glob, ny], "dof_per_node": dof_per_node(m),
                   "l2": "inputs larger than L2 (u+v = %.0f MB per parity, L2 126 MB); no flush" % (
                       cells_rank * dof_per_node(m) * 8 / 1e6),
                   "parallelism": f"slab{world} (x rows, one-row NCCL halo per half step)" if world > 1
                   else "single"},
        "roofline": roofline,
        # one cell-map launch per half step (interior + halo row: two at N > 1)
        "gpu_launches": args.steps * (1 if world == 1 else 2),
        "clocks": clk.summary(),
    }
    if comm is not None:
        result["comm"] = comm

    if not args.no_e2e:
        if world == 1:
            e2e = e2e_bench(hb, torch, np, m, ny, hb.SchemeConfig(m=m, lam=0.9), min(args.steps, 5))
        else:
            e2e = e2e_slab(hb, torch, dist, ring, m, min(args.steps, 5), stream)
        if rank == 0:
            result["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(m, ny, args.cpu_rows, rounds=2, warm=1)[0]
    if rank == 0 and world == 1 and not args.no_c3:
        result["c3"] = c3_bench(hb, torch, pk)
    if not args.no_c5:
        c5 = c5_scaling(hb, torch, dist, rank, world, stream, pk)
        if rank == 0:
            result["c5"] = c5
    if rank == 0 and world == 1 and not args.no_sweep:
        result["sweep"] = sweep(hb, torch, pk)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def c5_scaling(hb, torch, dist, rank, world, stream, pk):
    """BASELINE configs[4] (C5): 2D periodic dissipative m = 6 through the slab
    ring at this run's N: strong scaling at 8192^2 (45.6 GB per level, fits one
    GPU) and 16384^2 (182.5 GB per level: N >= 4), weak scaling at 2048 N x
    16384 (2048 x 16384 per GPU).  Device resident, 2 warm-up + 4 timed half
    steps each, max over ranks."""
    from paper_1802_05246_b200.slab import SlabRing

    m = 6
    cases = [("strong_8192", 8192, 8192), ("weak_2048Nx16384", 2048 * world, 16384)]
    if world >= 4:
        cases.append(("strong_16384", 16384, 16384))
    out = {"workload": "C5 (BASELINE configs[4]): 2D periodic dissipative Hermite m=6, lambda 0.9, standing wave; "
                       "strong scaling at 8192^2 (N=1/2/4/8) and 16384^2 (N=4/8), weak at 2048N x 16384",
           "n_gpus": world}
    for name, nx, ny in cases:
        grid = hb.Grid2D(0.0, nx / ny, 0.0, 1.0, nx, ny, True)
        ring = SlabRing(grid, rank, world)
        steps = 4
        ms, kern_ms = slab_run(hb, torch, dist, ring, m, steps, 2, stream)
        sec = ms / 1e3 / steps
        tf = f_alg_diss(m) * nx * ny / sec / 1e12
        out[name] = {"global_nodes": [nx, ny], "nodes_per_gpu": [ring.nrows(hb.PRIMAL), ny],
                     "gdof_per_s": nx * ny * dof_per_node(m) / sec / 1e9, "ms_per_step": sec * 1e3,
                     "kernel_ms_per_step": kern_ms, "tflops_falg": tf,
                     "frac_dmma_peak_per_gpu": tf / world / pk["dmma_tflops"], "steps": steps}
    return out


def e2e_slab(hb, torch, dist, ring, m, steps, stream):
    """End to end at N GPUs through the public slab API: every step each rank
    uploads its slab's (u, v) from pinned host memory, runs
    SlabRing.diss2d_step (NCCL halo + kernels) and reads the new state back;
    host wall clock, max over ranks."""
    grid = ring.grid
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    w = 2.0 * math.pi
    shp_u = ring.local_shape(hb.PRIMAL, m, m)
    shp_v = ring.local_shape(hb.PRIMAL, m - 1, m - 1)
    hu = torch.empty(shp_u, dtype=torch.float64, pin_memory=True)
    hv = torch.empty(shp_v, dtype=torch.float64, pin_memory=True)
    hu.copy_(hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0),
                                      rows=(ring.row0, ring.nrows(hb.PRIMAL))))
    hv.copy_(hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1,
                                      rows=(ring.row0, ring.nrows(hb.PRIMAL))))
    du, dv = torch.empty(shp_u, dtype=torch.float64, device="cuda"), torch.empty(shp_v, dtype=torch.float64,
                                                                                 device="cuda")
    ou, ov = torch.empty_like(du), torch.empty_like(dv)
    bc = hb.BoundarySpec2D()

    def one(par):
        du.copy_(hu, non_blocking=True)
        dv.copy_(hv, non_blocking=True)
        ring.diss2d_step(du, dv, ou, ov, par, m, cfg, bc, stream.cuda_stream)
        hu.copy_(ou, non_blocking=True)
        hv.copy_(ov, non_blocking=True)

    par = hb.PRIMAL
    one(par)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        par = hb.flip(par)
        one(par)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    t = torch.tensor([sec], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t[0])
    nbytes = (hu.numel() + hv.numel()) * 8
    return {"value": grid.nx * grid.ny * dof_per_node(m) * steps / sec / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "api": "paper_1802_05246_b200.slab.SlabRing.diss2d_step (pinned host slabs, per rank)",
            "steps": steps, "timer": "host wall clock around the steps, max over ranks"}


def e2e_bench(hb, torch, np, m, n, cfg, steps):
    """Same metric through the public drop-in API with host buffers:
    hb.half_step_2d(FieldPair of numpy arrays) per step — H2D of the step's
    inputs, the kernel, D2H of the new state.  Measured with the inputs in
    pinned host memory (the headline) and, as a hermwave caller passes them,
    in ordinary pageable numpy arrays ("pageable")."""
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0), tder=0)
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    bc = hb.BoundarySpec2D()
    nbytes = (u.numel() + v.numel()) * 8

    def timed(hu, hv):
        pair = hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.1, hu), hb.Field2D(grid, hb.PRIMAL, 0.1, hv))
        hb.half_step_2d(pair, cfg, bc)  # warm-up (also fills the pinned caching allocator)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):  # every step from the caller's own host arrays (outputs land pinned)
            hb.half_step_2d(pair, cfg, bc)
        torch.cuda.synchronize()
        return n * n * dof_per_node(m) * steps / (time.perf_counter() - t0) / 1e9

    pu = torch.empty(u.shape, dtype=torch.float64, pin_memory=True)
    pv = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
    pu.copy_(u)
    pv.copy_(v)
    pinned = timed(pu.numpy(), pv.numpy())
    pageable = timed(u.cpu().numpy().copy(), v.cpu().numpy().copy())
    return {"value": pinned, "unit": UNIT, "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "api": "paper_1802_05246_b200.half_step_2d(numpy FieldPair, pinned)",
            "steps": steps, "timer": "host wall clock around the API calls",
            "pageable": {"value": pageable, "unit": UNIT,
                         "api": "paper_1802_05246_b200.half_step_2d(numpy FieldPair, pageable numpy arrays)"}}


def _time_steps(torch, fn, k):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(k):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / k


def c3_bench(hb, torch, pk):
    """Config C3: conservative m=5 on 2048^2 with Dirichlet x / Neumann y walls
    (device resident, in place over `previous`)."""
    from paper_1802_05246_b200.stepping import cons2d_into

    m, n = 5, 2048
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0"), hb.BoundarySpec("neumann0", "neumann0"))
    pi = math.pi
    om = pi * math.sqrt(2.0)
    dt = cfg.dt(grid.hx)
    # u = sin(pi x) cos(pi y) cos(sqrt2 pi t) = sin(pi x) sin(pi y + pi/2) ...
    a = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.0, m, m, pi, pi, om, py=0.5 * pi)
    b = hb.standing_wave_on_grid(grid, hb.DUAL, -0.5 * dt, m, m, pi, pi, om, py=0.5 * pi)
    par = [hb.PRIMAL, hb.DUAL]
    state = {"a": a, "b": b, "pa": hb.PRIMAL}

    def one(i):
        cons2d_into(state["a"], state["b"], state["b"], grid, state["pa"], m, cfg, bc)
        state["a"], state["b"] = state["b"], state["a"]
        state["pa"] = hb.flip(state["pa"])

    for i in range(4):
        one(i)
    torch.cuda.synchronize()
    sec = _time_steps(torch, one, 10)
    cells = n * n  # targets alternate between 2048^2 (dual) and 2049^2 (primal); count the smaller
    g = cells * dof_per_node(m, "cons") / sec / 1e9
    tf = f_alg_cons(m) * cells / sec / 1e12
    del par
    # the conservation check: the defined 2D conservative energy (norms.py
    # conservative_energy_2d) sampled over NCONS further
    # steps.  At this h the exactly conserved mixed (m+1, m+1) form is below
    # round-off; the L2 / H1 adjoint forms are the physical
    # energy (conserved by the exact wave; L2 = sin^2(omega dt / 2) / 2 here)
    ncons, every = 1000, 250

    def energy():
        cur = hb.Field2D(grid, state["pa"], 0.0, state["a"])
        prev = hb.Field2D(grid, hb.flip(state["pa"]), 0.0, state["b"])
        return {s: hb.conservative_energy_2d(cur, prev, cfg.speed, dt, bc, s) for s in ("l2", "h1")}

    es = [energy()]
    for k in range(ncons):
        one(k)
        if (k + 1) % every == 0:
            es.append(energy())
    drift = {s: max(abs(e[s] - es[0][s]) for e in es) / es[0][s] for s in ("l2", "h1")}
    closed = 0.5 * math.sin(0.5 * om * dt) ** 2
    return {"workload": "2D conservative Hermite m=5, 2048^2, Dirichlet x / Neumann y walls (C3)",
            "gdof_per_s": g, "ms_per_step": sec * 1e3, "tflops_falg": tf, "frac_dmma_peak": tf / pk["dmma_tflops"],
            "hbm_gbs": 24 * cells * dof_per_node(m, "cons") / sec / 1e9,
            "conservation_check": {"kind": "2D conservative energy, adjoint form in the L2 and H1 seminorms "
                                           "(norms.conservative_energy_2d seminorm='l2'/'h1')",
                                   "steps": ncons, "samples": es, "max_rel_drift": drift,
                                   "l2_closed_form": closed, "l2_rel_err_vs_closed_form": abs(es[0]["l2"] - closed) / closed}}


def sweep(hb, torch, pk):
    """Config C4: dissipative m = 2..8 at ~2^30 DOF per level (device
    resident); each entry carries both roofline fractions (DMMA by SURVEY's
    F_alg, HBM by 16 B/DOF) and the binding one: SURVEY §8d puts the
    HBM / FP64 crossover between m = 2 and 3."""
    from paper_1802_05246_b200.stepping import diss2d_into

    out = {}
    for m in range(2, 9):
        n = SWEEP_N[m]
        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
        cfg = hb.SchemeConfig(m=m, lam=0.9)
        w = 2.0 * math.pi
        u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
        v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
        bufs = [(u, v), (torch.empty_like(u), torch.empty_like(v))]
        bc = hb.BoundarySpec2D()
        st = {"par": hb.PRIMAL}

        def one(i):
            diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, st["par"], m, cfg, bc)
            st["par"] = hb.flip(st["par"])

        for i in range(2):
            one(i)
        torch.cuda.synchronize()
        sec = _time_steps(torch, lambda i: one(i + 2), 6)
        g = n * n * dof_per_node(m) / sec / 1e9
        tf = f_alg_diss(m) * n * n / sec / 1e12
        dense, issued = cellmap_flops(m)
        out[f"m{m}"] = {"n": n, "gdof_per_s": g, "ms_per_step": sec * 1e3, "tflops_falg": tf,
                        "frac_dmma_peak": tf / pk["dmma_tflops"],
                        "issued_dmma_frac": issued * n * n / sec / 1e12 / pk["dmma_tflops"],
                        "hbm_frac": 16 * n * n * dof_per_node(m) / sec / 1e9 / pk["hbm_gbs"]}
        ai = f_alg_diss(m) / (16 * dof_per_node(m))  # flop / B
        out[f"m{m}"]["bound"] = "hbm" if ai < pk["dmma_tflops"] * 1e3 / pk["hbm_gbs"] else "tensor"
        del u, v, bufs
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    main()
