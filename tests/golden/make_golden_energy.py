"""Golden vectors for the 1D energy reductions, produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_energy.py

Imports hermwave read-only from /root/reference/pkg/src and records
dissipative_energy / conservative_energy (diagnostics.py:220-234) on seeded
random fields, plus a short conservative trace whose energy the scheme
preserves.  Output: tests/golden/energy.npz (numpy version stamped).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

import hermwave as hw  # noqa: E402
from hermwave.boundary import BoundarySpec  # noqa: E402
from hermwave.diagnostics import conservative_energy, dissipative_energy  # noqa: E402
from hermwave.grid import DUAL, PRIMAL, Field1D, FieldPair, Grid1D, TwoLevelState  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, m, n, periodic, parity, bc, speed)
DISS_CASES = [
    ("p_m1", 1, 9, True, PRIMAL, None, 1.0),
    ("p_m2_dual", 2, 8, True, DUAL, None, 1.7),
    ("p_m3", 3, 12, True, PRIMAL, None, 0.6),
    ("p_m5", 5, 7, True, DUAL, None, 1.0),
    ("w_m3_primal", 3, 8, False, PRIMAL, ("dirichlet0", "neumann0", 0.3, 0.0), 1.0),
    ("w_m4_dual", 4, 6, False, DUAL, ("neumann0", "dirichlet0", 0.0, -0.5), 2.0),
]
# (name, m, n, parity_cur, lam, speed)
CONS_CASES = [
    ("m1", 1, 10, PRIMAL, 0.9, 1.0),
    ("m2_dual", 2, 9, DUAL, 0.5, 1.3),
    ("m3_lam1", 3, 8, PRIMAL, 1.0, 1.0),
    ("m4", 4, 11, DUAL, 0.7, 0.8),
    ("m6", 6, 6, PRIMAL, 0.9, 1.0),
]
X1D = (-0.4, 1.1)


def main():
    arrays = {}
    for idx, (name, m, n, per, par, bcs, speed) in enumerate(DISS_CASES):
        rng = np.random.default_rng(900 + idx)
        grid = Grid1D(*X1D, n, per)
        bc = BoundarySpec() if bcs is None else BoundarySpec(*bcs)
        nn = grid.n_nodes(par)
        u = rng.standard_normal((nn, m + 1))
        v = rng.standard_normal((nn, m))
        pair = FieldPair(Field1D(grid, par, 0.0, u), Field1D(grid, par, 0.0, v))
        arrays[f"ed/{name}/u"] = u
        arrays[f"ed/{name}/v"] = v
        arrays[f"ed/{name}/e"] = np.array(dissipative_energy(pair, speed, bc))
    for idx, (name, m, n, par, lam, speed) in enumerate(CONS_CASES):
        rng = np.random.default_rng(950 + idx)
        grid = Grid1D(*X1D, n, True)
        bc = BoundarySpec()
        cfg = hw.SchemeConfig(m=m, speed=speed, lam=lam)
        dt = cfg.dt(grid.h)
        cur = rng.standard_normal((grid.n_nodes(par), m + 1))
        prev = rng.standard_normal((grid.n_nodes(hw.grid.flip(par)), m + 1))
        c = Field1D(grid, par, 0.0, cur)
        p = Field1D(grid, hw.grid.flip(par), -0.5 * dt, prev)
        arrays[f"ec/{name}/cur"] = cur
        arrays[f"ec/{name}/prev"] = prev
        arrays[f"ec/{name}/e"] = np.array(conservative_energy(c, p, speed, dt, bc))
        # a short conservative trace: the scheme preserves this energy
        st = TwoLevelState(c, p)
        trace = [conservative_energy(st.current, st.previous, speed, dt, bc)]
        for _ in range(4):
            st = hw.full_step_conservative(st, cfg, bc)
            trace.append(conservative_energy(st.current, st.previous, speed, dt, bc))
        arrays[f"ec/{name}/trace"] = np.array(trace)
    stamp = {"meta/numpy": np.array(np.__version__), "meta/reference": np.array(hw.__version__)}
    path = os.path.join(OUT, "energy.npz")
    np.savez_compressed(path, **arrays, **stamp)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
