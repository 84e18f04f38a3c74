"""Observed-order ladders of SURVEY App. A.5 as the REFERENCE measures them.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ladders.py

  * "c2": config C2's scheme and CFL (2D periodic dissipative m=4, lambda 0.9),
    kappa = 1 plane wave (driver.py:241-256) to t ~ 0.5, n = 6..15 (rate 7.04);
  * "walls_m2" / "walls_m3": C3's setting (conservative, Dirichlet x /
    Neumann y) with u = sin(3 pi x) cos(3 pi y) cos(3 sqrt2 pi t), lambda 0.9,
    t ~ 0.5, an EVEN number of half steps so every level ends on the primal
    grid (App. A.5/A.6: an odd count flips the final parity and the dual-wall
    L2 quirk integrates a larger domain), n = 8..18.
Per level: n, nhalf, the L2 error (diagnostics.py:118-135) and the fitted rate
(diagnostics.py:267-278).  Output: tests/golden/ladders.npz.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
OUT = os.path.dirname(os.path.abspath(__file__))

import hermwave as hw  # noqa: E402
from hermwave.boundary import BoundarySpec, BoundarySpec2D  # noqa: E402
from hermwave.diagnostics import fit_rate, l2_error_field_2d  # noqa: E402
from hermwave.driver import planewave_data  # noqa: E402
from hermwave.grid import DUAL, PRIMAL, Field2D, FieldPair, Grid2D, TwoLevelState  # noqa: E402

sys.path.insert(0, OUT)
from make_golden_c3 import standing_wave  # noqa: E402


def c2_ladder():
    m, lam = 4, 0.9
    cfg = hw.SchemeConfig(m=m, lam=lam)
    rows = []
    for n in range(6, 16):
        grid = Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
        h = grid.hx
        dt = cfg.dt(h)
        nhalf = round(1.0 / dt)  # t ~ 0.5
        x = grid.axis(0).nodes(PRIMAL)
        pair = FieldPair(Field2D(grid, PRIMAL, 0.0, planewave_data(x, x, 0.0, m, m, 1, h, h)),
                         Field2D(grid, PRIMAL, 0.0, planewave_data(x, x, 0.0, m - 1, m - 1, 1, h, h, tder=1)))
        for _ in range(nhalf):
            pair = hw.half_step_2d(pair, cfg, BoundarySpec2D())
        t = pair.u.time
        w = 2.0 * math.pi

        def exact(X, Y, t=t):
            return np.sin(w * (X + Y + math.sqrt(2.0) * t))

        rows.append((n, nhalf, h, l2_error_field_2d(pair.u, exact, BoundarySpec2D())))
    return rows


def wall_ladder(m):
    lam = 0.9
    cfg = hw.SchemeConfig(m=m, lam=lam)
    bc = BoundarySpec2D(BoundarySpec("dirichlet0", "dirichlet0"), BoundarySpec("neumann0", "neumann0"))
    rows = []
    for n in range(8, 19):
        grid = Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
        h = grid.hx
        dt = cfg.dt(h)
        nhalf = 2 * round(0.5 / dt)  # even: the last level lands on the primal grid
        xp, xd = grid.axis(0).nodes(PRIMAL), grid.axis(0).nodes(DUAL)
        st = TwoLevelState(Field2D(grid, PRIMAL, 0.0, wave3(xp, 0.0, m, h)),
                           Field2D(grid, DUAL, -0.5 * dt, wave3(xd, -0.5 * dt, m, h)))
        for _ in range(nhalf):
            st = hw.full_step_conservative(st, cfg, bc)
        assert st.current.parity == PRIMAL
        t = st.current.time
        k = 3.0 * math.pi

        def exact(X, Y, t=t):
            return np.sin(k * X) * np.cos(k * Y) * math.cos(math.sqrt(2.0) * k * t)

        rows.append((n, nhalf, h, l2_error_field_2d(st.current, exact, bc)))
    return rows


def wave3(nodes, t, m, h):
    """Scaled blocks of sin(3 pi x) cos(3 pi y) cos(3 sqrt2 pi t) (standing_wave with k = 3 pi)."""
    k = 3.0 * math.pi
    om = math.sqrt(2.0) * k
    out = np.empty((len(nodes), len(nodes), m + 1, m + 1))
    for a in range(m + 1):
        fx = k**a * np.sin(k * nodes + 0.5 * math.pi * a) * h**a / math.factorial(a)
        for b in range(m + 1):
            fy = k**b * np.cos(k * nodes + 0.5 * math.pi * b) * h**b / math.factorial(b)
            out[:, :, a, b] = fx[:, None] * fy[None, :] * math.cos(om * t)
    return out


def main():
    A = {}
    for name, rows in (("c2", c2_ladder()), ("walls_m2", wall_ladder(2)), ("walls_m3", wall_ladder(3))):
        n, nhalf, h, err = (np.array(c) for c in zip(*rows))
        A[f"{name}/n"], A[f"{name}/nhalf"], A[f"{name}/h"], A[f"{name}/err"] = n, nhalf, h, err
        A[f"{name}/rate"] = np.array(fit_rate(h, err))
        print(name, "rate", float(A[f"{name}/rate"]), "err", err[0], err[-1], flush=True)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "ladders.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
