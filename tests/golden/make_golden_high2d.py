"""Golden vectors for the 2D steps at the top of the reference's order range
(m = 9..12; interp.py:30 MAX_ORDER = 12), produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_high2d.py

For each order: one dissipative half step (dissipative.py:215-247), one
conservative step (conservative.py:139-157) and bootstrap_first_half
(conservative.py:166-195) on a few-node grid, periodic and with walls, from
seeded random data; plus sigma, the reference's own per-coefficient
sensitivity to a 1-ulp relative perturbation of its inputs (max over nodes),
which scales the GPU tolerance (cond(M_mu) grows to ~1e10 at
mu = 12).  Output: tests/golden/high2d.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(OUT))

import hermwave as hw  # noqa: E402
from hermwave.boundary import BoundarySpec, BoundarySpec2D  # noqa: E402
from hermwave.grid import Field2D, FieldPair, Grid2D, TwoLevelState  # noqa: E402

from cases import HIGH2D_CASES  # noqa: E402


def spec(walls):
    if not walls:
        return BoundarySpec2D()
    return BoundarySpec2D(BoundarySpec("dirichlet0", "neumann0", 0.3, 0.0), BoundarySpec("neumann0", "dirichlet0",
                                                                                         0.0, -0.2))


def main():
    A = {}
    for idx, (name, m, nx, ny, walls, par) in enumerate(HIGH2D_CASES):
        rng = np.random.default_rng(1500 + idx)
        grid = Grid2D(0.0, 1.0, -0.5, 0.7, nx, ny, not walls)
        bc = spec(walls)
        cfg = hw.SchemeConfig(m=m, lam=0.9)
        tp = hw.grid.flip(par)
        shp = lambda p, k: (grid.axis(0).n_nodes(p), grid.axis(1).n_nodes(p), k + 1, k + 1)  # noqa: E731
        u, v = rng.standard_normal(shp(par, m)), rng.standard_normal(shp(par, m - 1))
        cur, prev, g1 = rng.standard_normal(shp(par, m)), rng.standard_normal(shp(tp, m)), rng.standard_normal(
            shp(par, m))

        def run(u, v, cur, prev, g1):
            d = hw.half_step_2d(FieldPair(Field2D(grid, par, 0.0, u), Field2D(grid, par, 0.0, v)), cfg, bc)
            c = hw.full_step_conservative(TwoLevelState(Field2D(grid, par, 0.0, cur), Field2D(grid, tp, -0.1, prev)),
                                          cfg, bc)
            b = hw.bootstrap_first_half(Field2D(grid, par, 0.0, cur), Field2D(grid, par, 0.0, g1), cfg, bc)
            return [np.ascontiguousarray(x) for x in (d.u.values, d.v.values, c.current.values, b.current.values)]

        outs = run(u, v, cur, prev, g1)
        pert = [x * (1.0 + 2.2e-16 * rng.standard_normal(x.shape)) for x in (u, v, cur, prev, g1)]
        outp = run(*pert)
        for key, x in zip(("u0", "v0", "cur0", "prev0", "g1"), (u, v, cur, prev, g1)):
            A[f"{name}/{key}"] = x
        for key, o, p in zip(("u", "v", "cons", "boot"), outs, outp):
            A[f"{name}/{key}"] = o
            A[f"{name}/{key}_sigma"] = np.abs(o - p).max(axis=(0, 1))
        print(name, [float(np.abs(o).max()) for o in outs], flush=True)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "high2d.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
