"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports hermwave read-only from /root/reference/pkg/src, feeds it seeded
inputs and stores inputs + outputs in tests/golden/*.npz, stamped with the
numpy version.  The fixtures travel with the repo; nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import hermwave as hw  # noqa: E402
from hermwave.boundary import BoundarySpec, BoundarySpec2D  # noqa: E402
from hermwave.diagnostics import l2_error_field, l2_error_field_2d, l2_errors_pair  # noqa: E402
from hermwave.driver import planewave_data  # noqa: E402
from hermwave.grid import DUAL, PRIMAL, Field1D, Field2D, FieldPair, Grid1D, Grid2D, TwoLevelState  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(OUT))

from cases import CASES_1D, CASES_2D, exact2d, forcing_fn  # noqa: E402


def bc1(kind_l, kind_r, gl=0.0, gr=0.0):
    return BoundarySpec(kind_l, kind_r, gl, gr)


def bc_tuple(spec):
    return (spec.left, spec.right, spec.left_value, spec.right_value)


def rand_field2d(rng, grid, parity, kx, ky):
    nx, ny = grid.axis(0).n_nodes(parity), grid.axis(1).n_nodes(parity)
    return rng.standard_normal((nx, ny, kx + 1, ky + 1))


def spec2d(bcx, bcy):
    if bcx is None:
        return BoundarySpec2D()
    return BoundarySpec2D(BoundarySpec(*bcx), BoundarySpec(*bcy))


def make_2d():
    arrays = {}
    for idx, (name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps) in enumerate(CASES_2D):
        rng = np.random.default_rng(500 + idx)
        grid = Grid2D(0.0, 1.0, -0.5, 0.7, nx, ny, per)
        bc = spec2d(bcx, bcy)
        cfg = hw.SchemeConfig(m=m, speed=c, lam=lam, stage_cap=cap)
        # dissipative
        u0 = rand_field2d(rng, grid, par, m, m)
        v0 = rand_field2d(rng, grid, par, m - 1, m - 1)
        pair = FieldPair(Field2D(grid, par, 0.0, u0), Field2D(grid, par, 0.0, v0))
        for _ in range(steps):
            pair = hw.half_step_2d(pair, cfg, bc)
        arrays[f"d2/{name}/u0"] = u0
        arrays[f"d2/{name}/v0"] = v0
        arrays[f"d2/{name}/u"] = np.ascontiguousarray(pair.u.values)
        arrays[f"d2/{name}/v"] = np.ascontiguousarray(pair.v.values)
        arrays[f"d2/{name}/t"] = np.array(pair.time)
        # conservative (one full step from random levels; then bootstrap)
        cur = rand_field2d(rng, grid, par, m, m)
        prev = rand_field2d(rng, grid, hw.grid.flip(par), m, m)
        st = TwoLevelState(Field2D(grid, par, 0.0, cur), Field2D(grid, hw.grid.flip(par), -0.1, prev))
        for _ in range(steps):
            st = hw.full_step_conservative(st, cfg, bc)
        arrays[f"c2/{name}/cur0"] = cur
        arrays[f"c2/{name}/prev0"] = prev
        arrays[f"c2/{name}/cur"] = np.ascontiguousarray(st.current.values)
        arrays[f"c2/{name}/prev"] = np.ascontiguousarray(st.previous.values)
        arrays[f"c2/{name}/t"] = np.array(st.current.time)
        g1 = rand_field2d(rng, grid, par, m, m)
        b = hw.bootstrap_first_half(Field2D(grid, par, 0.0, cur), Field2D(grid, par, 0.0, g1), cfg, bc)
        arrays[f"b2/{name}/g1"] = g1
        arrays[f"b2/{name}/out"] = np.ascontiguousarray(b.current.values)
        # L2 error of u0 against a smooth function (dual-wall quirk included)
        arrays[f"e2/{name}/u"] = np.array(l2_error_field_2d(Field2D(grid, par, 0.0, u0), exact2d, bc))
        arrays[f"e2/{name}/v"] = np.array(l2_error_field_2d(Field2D(grid, par, 0.0, v0), exact2d, bc))
    # plane-wave initial data (driver.py:241-256)
    grid = Grid2D(0.0, 1.0, 0.0, 1.0, 7, 7, True)
    xp = grid.axis(0).nodes(DUAL)
    arrays["init/planewave_u"] = planewave_data(xp, xp, 0.3, 4, 4, 5, grid.hx, grid.hy)
    arrays["init/planewave_v"] = planewave_data(xp, xp, 0.3, 3, 3, 5, grid.hx, grid.hy, tder=1)
    return arrays


def make_1d():
    arrays = {}
    for idx, (name, m, n, per, par, bcs, lam, c, cap, steps, forced) in enumerate(CASES_1D):
        rng = np.random.default_rng(700 + idx)
        grid = Grid1D(-0.4, 1.1, n, per)
        bc = BoundarySpec() if bcs is None else BoundarySpec(*bcs)
        cfg = hw.SchemeConfig(m=m, speed=c, lam=lam, stage_cap=cap)
        nn = grid.n_nodes(par)
        u0 = rng.standard_normal((nn, m + 1))
        v0 = rng.standard_normal((nn, m))
        pair = FieldPair(Field1D(grid, par, 0.0, u0), Field1D(grid, par, 0.0, v0))
        for _ in range(steps):
            pair = hw.half_step_1d(pair, cfg, bc, forcing=forcing_fn if forced else None)
        arrays[f"d1/{name}/u0"] = u0
        arrays[f"d1/{name}/v0"] = v0
        arrays[f"d1/{name}/u"] = np.ascontiguousarray(pair.u.values)
        arrays[f"d1/{name}/v"] = np.ascontiguousarray(pair.v.values)
        arrays[f"d1/{name}/t"] = np.array(pair.time)
        if forced:
            continue
        cur = rng.standard_normal((nn, m + 1))
        prev = rng.standard_normal((grid.n_nodes(hw.grid.flip(par)), m + 1))
        st = TwoLevelState(Field1D(grid, par, 0.0, cur), Field1D(grid, hw.grid.flip(par), -0.1, prev))
        for _ in range(steps):
            st = hw.full_step_conservative(st, cfg, bc)
        arrays[f"c1/{name}/cur0"] = cur
        arrays[f"c1/{name}/prev0"] = prev
        arrays[f"c1/{name}/cur"] = np.ascontiguousarray(st.current.values)
        arrays[f"c1/{name}/prev"] = np.ascontiguousarray(st.previous.values)
        g1 = rng.standard_normal((nn, m + 1))
        b = hw.bootstrap_first_half(Field1D(grid, par, 0.0, cur), Field1D(grid, par, 0.0, g1), cfg, bc)
        arrays[f"b1/{name}/g1"] = g1
        arrays[f"b1/{name}/out"] = np.ascontiguousarray(b.current.values)
        # errors (u, u_x, v) against smooth functions; walls clip, periodic does not
        eu, edux, ev = l2_errors_pair(FieldPair(Field1D(grid, par, 0.0, u0), Field1D(grid, par, 0.0, v0)),
                                      np.sin, np.cos, lambda x: -np.sin(2 * x), bc)
        arrays[f"e1/{name}/pair"] = np.array([eu, edux, ev])
        arrays[f"e1/{name}/field"] = np.array(l2_error_field(Field1D(grid, par, 0.0, u0), np.sin, bc))
    return arrays


def main():
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    mats = {f"interp/{mu}": np.array(hw.interp_matrix(mu)) for mu in range(0, 13)}
    np.savez_compressed(os.path.join(OUT, "interp.npz"), **mats, **stamp)
    np.savez_compressed(os.path.join(OUT, "steps2d.npz"), **make_2d(), **stamp)
    np.savez_compressed(os.path.join(OUT, "steps1d.npz"), **make_1d(), **stamp)
    for f in ("interp.npz", "steps2d.npz", "steps1d.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
