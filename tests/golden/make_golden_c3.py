"""Golden vectors for BASELINE config C3's exact setup, produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c3.py

C3 is the 2D conservative scheme (conservative.py:139-157) with Dirichlet
walls in x and Neumann walls in y (boundary.py:56-98, 124-130).  For odd
orders (m = 3, 5 = C3's order, 7) and BOTH starting parities this records:

  * the standing wave u = sin(pi x) cos(pi y) cos(sqrt(2) pi t) on the unit
    square (the C3 throughput input), current level at t = 0 and previous
    level at t = -dt/2 on the opposite parity, stepped NSTEPS full steps;
  * seeded random levels with nonzero Dirichlet data, stepped NSTEPS steps;
  * bootstrap_first_half (conservative.py:166-195) from the wave at t = 0;
  * sigma: the reference's own sensitivity to a 1-ulp relative perturbation
    of its inputs on the same run, per coefficient (k, l)
    as the max over the nodes, which the
    GPU tests use as the tolerance scale.

Output: tests/golden/c3walls.npz (numpy version stamped).  Nothing at test
time reads /root/reference.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import hermwave as hw  # noqa: E402
from hermwave.boundary import BoundarySpec, BoundarySpec2D  # noqa: E402
from hermwave.grid import DUAL, PRIMAL, Field2D, Grid2D, TwoLevelState  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(OUT))

from cases import C3_CASES as CASES, C3_LAM as LAM, C3_RAND_BC as RAND_BC, C3_WAVE_BC as WAVE_BC  # noqa: E402



def standing_wave(nodes_x, nodes_y, t, m, h, tder=0):
    """Scaled blocks (h^k/k!)(h^l/l!) d_x^k d_y^l d_t^tder of
    sin(pi x) cos(pi y) cos(sqrt(2) pi t)."""
    w = math.pi
    om = math.sqrt(2.0) * math.pi
    out = np.empty((len(nodes_x), len(nodes_y), m + 1, m + 1))
    for k in range(m + 1):
        fx = w**k * np.sin(w * nodes_x + 0.5 * math.pi * k) * h**k / math.factorial(k)
        for l in range(m + 1):
            fy = w**l * np.cos(w * nodes_y + 0.5 * math.pi * l) * h**l / math.factorial(l)
            ft = om**tder * math.cos(om * t + 0.5 * math.pi * tder)
            out[:, :, k, l] = fx[:, None] * fy[None, :] * ft
    return out


def run(grid, par, cur, prev, cfg, bc, steps, t_prev):
    st = TwoLevelState(Field2D(grid, par, 0.0, cur), Field2D(grid, hw.grid.flip(par), t_prev, prev))
    for _ in range(steps):
        st = hw.full_step_conservative(st, cfg, bc)
    return st


def main():
    A = {}
    for idx, (name, m, n, par, steps, kind) in enumerate(CASES):
        rng = np.random.default_rng(1300 + idx)
        grid = Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
        bcx, bcy = WAVE_BC if kind == "wave" else RAND_BC
        bc = BoundarySpec2D(BoundarySpec(*bcx), BoundarySpec(*bcy))
        cfg = hw.SchemeConfig(m=m, lam=LAM)
        h = grid.hx
        dt = cfg.dt(h)
        tp = hw.grid.flip(par)
        if kind == "wave":
            cur = standing_wave(grid.axis(0).nodes(par), grid.axis(1).nodes(par), 0.0, m, h)
            prev = standing_wave(grid.axis(0).nodes(tp), grid.axis(1).nodes(tp), -0.5 * dt, m, h)
            g1 = standing_wave(grid.axis(0).nodes(par), grid.axis(1).nodes(par), 0.0, m, h, tder=1)
        else:
            shp = lambda p: (grid.axis(0).n_nodes(p), grid.axis(1).n_nodes(p), m + 1, m + 1)  # noqa: E731
            cur, prev, g1 = rng.standard_normal(shp(par)), rng.standard_normal(shp(tp)), rng.standard_normal(shp(par))
        st = run(grid, par, cur, prev, cfg, bc, steps, -0.5 * dt)
        # the reference's own 1-ulp sensitivity on the same run
        pert = [x * (1.0 + 2.2e-16 * rng.standard_normal(x.shape)) for x in (cur, prev)]
        sp = run(grid, par, pert[0], pert[1], cfg, bc, steps, -0.5 * dt)
        b = hw.bootstrap_first_half(Field2D(grid, par, 0.0, cur), Field2D(grid, par, 0.0, g1), cfg, bc)
        bp = hw.bootstrap_first_half(Field2D(grid, par, 0.0, pert[0]),
                                     Field2D(grid, par, 0.0, g1 * (1.0 + 2.2e-16 * rng.standard_normal(g1.shape))),
                                     cfg, bc)
        A[f"{name}/cur0"], A[f"{name}/prev0"], A[f"{name}/g1"] = cur, prev, g1
        A[f"{name}/cur"] = np.ascontiguousarray(st.current.values)
        A[f"{name}/t"] = np.array(st.current.time)
        # per coefficient (k, l): max over the nodes
        A[f"{name}/sigma"] = np.abs(np.ascontiguousarray(sp.current.values) - A[f"{name}/cur"]).max(axis=(0, 1))
        A[f"{name}/boot"] = np.ascontiguousarray(b.current.values)
        A[f"{name}/boot_sigma"] = np.abs(np.ascontiguousarray(bp.current.values) - A[f"{name}/boot"]).max(axis=(0, 1))
        print(name, st.current.parity, f"sigma/max {A[f'{name}/sigma'].max() / np.abs(A[f'{name}/cur']).max():.2e}",
              flush=True)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "c3walls.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
