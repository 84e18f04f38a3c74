#!/usr/bin/env python
"""Timeline of one host-array half step (stepping._diss2d_host_pipelined):
event times of each chunk's upload, kernel and download relative to the call
start, plus the host issue time, to see what bounds the e2e number."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200 import stepping as S

    m, n = 4, 1024
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D()
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    hu = torch.empty(u.shape, dtype=torch.float64, pin_memory=True)
    hv = torch.empty(v.shape, dtype=torch.float64, pin_memory=True)
    hu.copy_(u)
    hv.copy_(v)
    a, b, par = hu.numpy(), hv.numpy(), hb.PRIMAL
    for it in range(4):
        marks = []
        t0 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        h0 = time.perf_counter()
        _, a, b = S._diss2d_host_pipelined(a, b, grid, par, m, cfg, bc, _marks=marks)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        h2 = time.perf_counter()
        print(f"iter {it} parity {par}: host issue {1e3 * (h1 - h0):.2f} ms (includes the final wait), "
              f"total {1e3 * (h2 - h0):.2f} ms")
        for lab, e in marks:
            print(f"   {lab:14s} {t0.elapsed_time(e):7.3f}")
        par = hb.flip(par)


if __name__ == "__main__":
    main()
