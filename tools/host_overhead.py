#!/usr/bin/env python
"""Host-side cost of one 2D half step through the Python / C-ABI path versus
the kernel's device time (does the launch path keep the GPU fed?)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import diss2d_into

    m, n = 4, 1024
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D()
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    bufs = [(u, v), (torch.empty_like(u), torch.empty_like(v))]
    par = hb.PRIMAL
    for i in range(5):
        diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, par, m, cfg, bc)
        par = hb.flip(par)
    torch.cuda.synchronize()
    K = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(K):
        diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, par, m, cfg, bc)
        par = hb.flip(par)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"back-to-back: device {e0.elapsed_time(e1) / K:.4f} ms/step, host issue {(t1 - t0) * 1e3 / K:.4f} ms/step")
    # host cost alone: launches into a stream blocked behind a long sleep kernel
    torch.cuda._sleep(int(2e9 * 0.05))
    t0 = time.perf_counter()
    for i in range(K):
        diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, par, m, cfg, bc)
        par = hb.flip(par)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host issue while GPU busy: {(t1 - t0) * 1e3 / K:.4f} ms/step")

    import subprocess

    def loop(K, smi):
        nonlocal par
        p = None
        if smi:
            p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "100"],
                                 stdout=subprocess.DEVNULL)
            time.sleep(0.25)
        torch.cuda.synchronize()
        e0.record()
        for i in range(K):
            diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, par, m, cfg, bc)
            par = hb.flip(par)
        e1.record()
        torch.cuda.synchronize()
        if p is not None:
            p.terminate()
            p.wait()
        return e0.elapsed_time(e1) / K

    for K, smi in ((20, False), (20, True), (20, False), (400, False), (400, True), (2000, False)):
        print(f"K={K} nvidia-smi={smi}: {loop(K, smi):.4f} ms/step")


if __name__ == "__main__":
    main()
