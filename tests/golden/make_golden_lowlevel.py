"""Golden vectors for the lower-level batched API, produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_lowlevel.py

Imports hermwave read-only from /root/reference/pkg/src and records
apply_interp(_2d), expand_taylor(_2d) (with forcing / with d1), eval_series,
conservative_update_1d/2d, pascal_table, ghost_data(_2d), pair_sources and
corner_sources on seeded inputs.  Output: tests/golden/lowlevel.npz (numpy
version stamped).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import hermwave as hw  # noqa: E402
from hermwave.boundary import BoundarySpec, BoundarySpec2D, corner_sources, pair_sources  # noqa: E402
from hermwave.grid import DUAL, PRIMAL, Field1D, Field2D, Grid1D, Grid2D  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def forcing(l, s, x, t):  # smooth, depends on every argument
    return np.cos(0.7 * x + 0.3 * t) * (l + 1.0) / (s + 2.0)


def main():
    rng = np.random.default_rng(2024)
    A = {}
    for mu in (0, 2, 5):
        d = rng.standard_normal((3, 4, 2, mu + 1))
        A[f"ai1/{mu}/in"] = d
        A[f"ai1/{mu}/out"] = hw.apply_interp(d)
    for mux, muy in ((1, 1), (3, 2), (4, 4)):
        d = rng.standard_normal((5, 2, 2, mux + 1, muy + 1))
        A[f"ai2/{mux}{muy}/in"] = d
        A[f"ai2/{mux}{muy}/out"] = hw.apply_interp_2d(d)
    # expand_taylor: (dt, h, speed, smax) per case; forcing on the second
    for name, (lu, lv, smax, forced) in {"a": (6, 5, 6, False), "b": (8, 7, 9, True)}.items():
        cu = rng.standard_normal((4, lu))
        cv = rng.standard_normal((4, lv))
        centers = np.linspace(-0.3, 0.8, 4)
        dt, h, c, t = 0.037, 0.05, 1.3, 0.21
        tu, tv = hw.expand_taylor(cu, cv, dt, h, c, smax, forcing if forced else None, centers, t)
        A.update({f"et1/{name}/cu": cu, f"et1/{name}/cv": cv, f"et1/{name}/tu": tu, f"et1/{name}/tv": tv,
                  f"et1/{name}/centers": centers})
    for name, (k, lv, smax, with_d1) in {"a": (8, 6, 10, False), "b": (10, 8, 14, True)}.items():
        c0 = rng.standard_normal((3, k, k))
        d0 = rng.standard_normal((3, lv, lv))
        d1 = rng.standard_normal((3, k - 2, k - 2)) if with_d1 else None
        ct, dtab = hw.expand_taylor_2d(c0, d0, 0.02, 0.05, 0.07, 1.1, smax, d1)
        A.update({f"et2/{name}/c0": c0, f"et2/{name}/d0": d0, f"et2/{name}/ct": ct, f"et2/{name}/dt": dtab})
        if with_d1:
            A[f"et2/{name}/d1"] = d1
    tab = rng.standard_normal((6, 5, 11))
    A["es/in"] = tab
    A["es/out"] = hw.eval_series(tab, 0.5)
    A["es/out07"] = hw.eval_series(tab, 0.7)
    for m in (1, 3, 6):
        cfg = hw.SchemeConfig(m=m, lam=0.8, speed=1.2)
        c1 = rng.standard_normal((7, 2 * m + 2))
        p1 = rng.standard_normal((7, m + 1))
        A[f"cu1/{m}/c"], A[f"cu1/{m}/p"] = c1, p1
        A[f"cu1/{m}/out"] = hw.conservative_update_1d(c1, p1, cfg, 0.05)
        c2 = rng.standard_normal((3, 2, 2 * m + 2, 2 * m + 2))
        p2 = rng.standard_normal((3, 2, m + 1, m + 1))
        A[f"cu2/{m}/c"], A[f"cu2/{m}/p"] = c2, p2
        A[f"cu2/{m}/out"] = hw.conservative_update_2d(c2, p2, cfg, 0.05, 0.07)
        pt = hw.pascal_table(m, 0.31, 0.27)
        A[f"pt/{m}/base"], A[f"pt/{m}/scaled"] = pt.base, pt.scaled
    blk = rng.standard_normal((4, 5))
    for kind in ("dirichlet0", "neumann0"):
        A[f"g1/{kind}"] = hw.ghost_data(blk, kind, 0.7 if kind == "dirichlet0" else 0.0)
    blk2 = rng.standard_normal((3, 4, 5))
    for kind in ("dirichlet0", "neumann0"):
        for ax in (0, 1):
            A[f"g2/{kind}/{ax}"] = hw.ghost_data_2d(blk2, kind, ax, -0.4 if kind == "dirichlet0" else 0.0)
    A["g1/in"], A["g2/in"] = blk, blk2
    # gathers: periodic / walls, both parities
    cases1 = {"per_p": (True, PRIMAL, BoundarySpec()), "per_d": (True, DUAL, BoundarySpec()),
              "wall_p": (False, PRIMAL, BoundarySpec("dirichlet0", "neumann0", 0.3, 0.0)),
              "wall_d": (False, DUAL, BoundarySpec("dirichlet0", "neumann0", 0.3, 0.0))}
    for name, (per, par, spec) in cases1.items():
        g = Grid1D(-0.2, 1.1, 7, per)
        v = rng.standard_normal((g.n_nodes(par), 4))
        d, cen = pair_sources(Field1D(g, par, 0.0, v), spec)
        A[f"ps/{name}/in"], A[f"ps/{name}/out"], A[f"ps/{name}/cen"] = v, d, cen
        if name == "wall_d":
            d2, _ = pair_sources(Field1D(g, par, 0.0, v), spec, (0.0, 0.0))
            A["ps/wall_d/out_zero"] = d2
    sx = BoundarySpec("dirichlet0", "neumann0", 0.5, 0.0)
    sy = BoundarySpec("neumann0", "dirichlet0", 0.0, -0.25)
    cases2 = {"per_p": (True, PRIMAL, BoundarySpec2D()), "per_d": (True, DUAL, BoundarySpec2D()),
              "wall_p": (False, PRIMAL, BoundarySpec2D(sx, sy)), "wall_d": (False, DUAL, BoundarySpec2D(sx, sy))}
    for name, (per, par, spec) in cases2.items():
        g = Grid2D(-0.2, 1.1, 0.1, 0.9, 5, 4, per)
        v = rng.standard_normal((g.axis(0).n_nodes(par), g.axis(1).n_nodes(par), 3, 3))
        d, cx, cy = corner_sources(Field2D(g, par, 0.0, v), spec)
        A[f"cs/{name}/in"], A[f"cs/{name}/out"], A[f"cs/{name}/cx"], A[f"cs/{name}/cy"] = v, d, cx, cy
        if name == "wall_d":
            d2, _, _ = corner_sources(Field2D(g, par, 0.0, v), spec, (0.0, 0.0))
            A["cs/wall_d/out_zero"] = d2
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "lowlevel.npz")
    np.savez_compressed(path, **A, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
