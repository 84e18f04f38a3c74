"""Golden run of BASELINE config C1 by the REFERENCE: 1D periodic dissipative
Hermite m=3, CFL 0.9, the standing wave sin(x) cos(t) on [0, 2 pi] to t ~ 1,
on a refinement ladder plus n_x = 200.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_c1.py

Imports hermwave read-only from /root/reference/pkg/src; records per level the
(u, u_x, v) L2 errors (diagnostics.py:103-115), the fitted orders
(diagnostics.py:241-278) and, at n_x = 200, the final state itself.
Output: tests/golden/c1.npz (numpy version stamped).
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import hermwave as hw  # noqa: E402
from hermwave.driver import _scale_cols, sine_derivs  # noqa: E402
from hermwave.grid import PRIMAL, Field1D, FieldPair, Grid1D  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
M, LAM, T = 3, 0.9, 1.0
LADDER = (6, 8, 10, 13, 16, 20, 27)


def run(n):
    grid = Grid1D(0.0, 2.0 * math.pi, n, True)
    h = grid.h
    cfg = hw.SchemeConfig(m=M, lam=LAM)
    dt = cfg.dt(h)
    x = grid.nodes(PRIMAL)
    u0 = _scale_cols(sine_derivs(x, M, 0.0), h)
    v0 = np.zeros((n, M))  # u_t = -sin(x) sin(t) = 0 at t = 0
    pair = FieldPair(Field1D(grid, PRIMAL, 0.0, u0), Field1D(grid, PRIMAL, 0.0, v0))
    bc = hw.BoundarySpec()
    nhalf = round(2.0 * T / dt)
    for _ in range(nhalf):
        pair = hw.half_step_1d(pair, cfg, bc)
    t = pair.u.time
    eu, edux, ev = hw.l2_errors_pair(pair, lambda x: np.sin(x) * math.cos(t), lambda x: np.cos(x) * math.cos(t),
                                     lambda x: -np.sin(x) * math.sin(t), bc)
    return pair, nhalf, (eu, edux, ev)


def main():
    A = {}
    errs, hs = [], []
    for n in LADDER:
        pair, nhalf, e = run(n)
        errs.append(e)
        hs.append(pair.u.grid.h)
        A[f"n{n}/nhalf"] = np.array(nhalf)
        A[f"n{n}/time"] = np.array(pair.u.time)
    errs = np.array(errs)
    A["ladder"] = np.array(LADDER)
    A["errors"] = errs  # (levels, 3): u, u_x, v
    A["rates"] = np.array([hw.fit_rate(np.array(hs), errs[:, j]) for j in range(3)])
    pair, nhalf, e = run(200)
    A["n200/u"], A["n200/v"] = np.ascontiguousarray(pair.u.values), np.ascontiguousarray(pair.v.values)
    A["n200/errors"], A["n200/nhalf"], A["n200/time"] = np.array(e), np.array(nhalf), np.array(pair.u.time)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "c1.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path), "rates", A["rates"], "nhalf200", nhalf)


if __name__ == "__main__":
    main()
