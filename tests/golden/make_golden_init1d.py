"""Golden vectors for the 1D closed-form initial data, produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_init1d.py

Records hermwave.driver's gaussian_derivs, gaussian_box_u / _v, sine_derivs
and _scale_cols (driver.py:195-238) on the node sets the driver's own
experiments use (run_gaussian_1d's Grid1D(-1.5, 1.5, n), both parities, the
box times 0 and -dt/2; run_conservation_1d's Grid1D(-pi, pi, n)) and on a
spread of points, for orders up to 12.  Output: tests/golden/init1d.npz.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import hermwave as hw  # noqa: E402
from hermwave.driver import _scale_cols, gaussian_box_u, gaussian_box_v, gaussian_derivs, sine_derivs  # noqa: E402
from hermwave.grid import DUAL, PRIMAL, Grid1D  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    A = {}
    pts = np.linspace(-1.7, 1.7, 41)
    for k in (0, 1, 4, 8, 12):
        A[f"pts/gauss/{k}"] = gaussian_derivs(pts, k)
        A[f"pts/gauss_a3/{k}"] = gaussian_derivs(pts, k, a=-3.0)
        A[f"pts/box_u/{k}"] = gaussian_box_u(pts, 0.37, k)
        A[f"pts/box_v/{k}"] = gaussian_box_v(pts, 0.37, k)
        A[f"pts/sine/{k}"] = sine_derivs(pts, k, 0.8)
    A["pts/x"] = pts
    for m, n, lam in ((3, 10, 0.8), (4, 17, 1.0), (6, 12, 0.8)):
        g = Grid1D(-1.5, 1.5, n, False)
        h = g.h
        dt = lam * h
        for par in (PRIMAL, DUAL):
            x = g.nodes(par)
            A[f"grid/{m}/{n}/{par}/gauss"] = _scale_cols(gaussian_derivs(x, m), h)
            A[f"grid/{m}/{n}/{par}/box_u"] = _scale_cols(gaussian_box_u(x, -0.5 * dt, m), h)
            A[f"grid/{m}/{n}/{par}/box_v"] = _scale_cols(gaussian_box_v(x, 0.0, m), h)
        gp = Grid1D(-math.pi, math.pi, n, True)
        for par in (PRIMAL, DUAL):
            A[f"grid/{m}/{n}/{par}/sine"] = _scale_cols(sine_derivs(gp.nodes(par), m, -0.5 * lam * gp.h), gp.h)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "init1d.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
