#!/usr/bin/env python
"""Small driver for profiling and A/B timing: device-resident 2D half steps
(or conservative steps) of one configuration.

  python tools/prof_step.py --scheme diss --m 4 --n 1024 --steps 20

Times `--steps` back-to-back launches (alternating parity, as a time loop
runs) between two CUDA events after 3 warm-up steps, `--reps` times, and
prints the best and median per-step time.  HERMB200_LIB selects an
alternative build of the library (tools/build_variant.sh).
"""

import argparse
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scheme", default="diss", choices=["diss", "cons"])
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--walls", action="store_true")
    ap.add_argument("--tag", default=os.environ.get("HERMB200_LIB", "default"))
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
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    shp = lambda p, k: (grid.axis(0).n_nodes(p), grid.axis(1).n_nodes(p), k + 1, k + 1)  # noqa: E731
    if args.scheme == "diss":
        u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
        v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
        bufs = {hb.PRIMAL: (u, v),
                hb.DUAL: (torch.empty(shp(hb.DUAL, m), dtype=torch.float64, device="cuda"),
                          torch.empty(shp(hb.DUAL, m - 1), dtype=torch.float64, device="cuda"))}

        def step(par):
            diss2d_into(*bufs[par], *bufs[hb.flip(par)], grid, par, m, cfg, bc)

        dof = n * n * ((m + 1) ** 2 + m * m)
    else:
        lv = {hb.PRIMAL: hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0)),
              hb.DUAL: torch.zeros(shp(hb.DUAL, m), dtype=torch.float64, device="cuda")}

        def step(par):  # current on `par`, previous (overwritten in place) on the other parity
            cons2d_into(lv[par], lv[hb.flip(par)], lv[hb.flip(par)], grid, par, m, cfg, bc)

        dof = n * n * (m + 1) ** 2
    par = hb.PRIMAL
    for _ in range(3):
        step(par)
        par = hb.flip(par)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        ev[0].record()
        for _ in range(args.steps):
            step(par)
            par = hb.flip(par)
        ev[1].record()
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]) / args.steps)
    best, med = min(times), statistics.median(times)
    print(f"{args.scheme} m={m} n={n}{' walls' if args.walls else ''} [{os.path.basename(os.path.dirname(args.tag)) or args.tag}]: "
          f"best {best:.4f} ms, median {med:.4f} ms, {dof / best / 1e6:.2f} GDOF/s")


if __name__ == "__main__":
    main()
