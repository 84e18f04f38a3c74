#!/usr/bin/env python
"""Small driver for profiling: a few device-resident 2D half steps (or
conservative steps) of one configuration, timed with CUDA events.

  python tools/prof_step.py --scheme diss --m 4 --n 1024 --steps 5
"""

import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scheme", default="diss", choices=["diss", "cons"])
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--walls", action="store_true")
    args = ap.parse_args()

    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import cons2d_into, diss2d_into

    m, n = args.m, args.n
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, not args.walls)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    if args.walls:
        bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0"), hb.BoundarySpec("neumann0", "neumann0"))
    else:
        bc = hb.BoundarySpec2D()
    w = 2.0 * math.pi
    par = hb.PRIMAL
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if args.scheme == "diss":
        u = hb.standing_wave_on_grid(grid, par, 0.1, m, m, w, w, w * math.sqrt(2.0))
        v = hb.standing_wave_on_grid(grid, par, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
        bufs = [(u, v), None]
        shp = lambda p, k: (grid.axis(0).n_nodes(p), grid.axis(1).n_nodes(p), k + 1, k + 1)  # noqa: E731
        other = {hb.DUAL: (torch.empty(shp(hb.DUAL, m), dtype=torch.float64, device="cuda"),
                           torch.empty(shp(hb.DUAL, m - 1), dtype=torch.float64, device="cuda")),
                 hb.PRIMAL: (u, v)}
        times = []
        for i in range(args.steps):
            tp = hb.flip(par)
            ev[0].record()
            diss2d_into(*other[par], *other[tp], grid, par, m, cfg, bc)
            ev[1].record()
            torch.cuda.synchronize()
            times.append(ev[0].elapsed_time(ev[1]))
            par = tp
        dof = n * n * ((m + 1) ** 2 + m * m)
    else:
        a = hb.standing_wave_on_grid(grid, par, 0.1, m, m, w, w, w * math.sqrt(2.0))
        nd = grid.axis(0).n_nodes(hb.DUAL)
        b = torch.zeros((nd, grid.axis(1).n_nodes(hb.DUAL), m + 1, m + 1), dtype=torch.float64, device="cuda")
        times = []
        for i in range(args.steps):
            ev[0].record()
            cons2d_into(a, b, b, grid, par, m, cfg, bc)
            ev[1].record()
            torch.cuda.synchronize()
            times.append(ev[0].elapsed_time(ev[1]))
            a, b = b, a
            par = hb.flip(par)
        dof = n * n * (m + 1) ** 2
    best = min(times[1:] or times)
    print(f"{args.scheme} m={m} n={n}: best {best:.4f} ms, {dof / best / 1e6:.2f} GDOF/s; all {['%.3f' % t for t in times]}")


if __name__ == "__main__":
    main()
