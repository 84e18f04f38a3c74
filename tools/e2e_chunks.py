#!/usr/bin/env python
"""e2e half step (host arrays in/out) versus the pipeline's chunk count."""
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
    dof = n * n * ((m + 1) ** 2 + m * m)
    geo = lambda *f: [0.0, *f, 1.0]  # noqa: E731
    for nch in (8, 16, geo(0.02, 0.1, 0.25, 0.45, 0.65, 0.85, 0.96), geo(0.015, 0.06, 0.2, 0.4, 0.6, 0.8, 0.92, 0.98),
                geo(0.03, 0.2, 0.4, 0.6, 0.8, 0.97), geo(0.01, 0.05, 0.15, 0.35, 0.55, 0.75, 0.9, 0.97, 0.99)):
        a, b, par = hu.numpy(), hv.numpy(), hb.PRIMAL
        ts = []
        for i in range(8):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, a, b = S._diss2d_host_pipelined(a, b, grid, par, m, cfg, bc, nchunks=nch)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            par = hb.flip(par)
        best = sorted(ts[2:])
        print(f"chunks={nch if isinstance(nch, int) else len(nch) - 1}: median {1e3 * best[len(best) // 2]:.2f} ms, best {1e3 * best[0]:.2f} ms "
              f"-> {dof / best[len(best) // 2] / 1e9:.2f} GDOF/s")


if __name__ == "__main__":
    main()
