"""Every 2D kernel configuration on grids large enough for interior tiles.

The golden cases (test_gpu_parity.py) are a few nodes per axis, so each is a
single edge tile and only the kernels' general staging path runs.  Here every
order of every scheme runs one step on a 40 x 70 grid — interior tiles take
the fast 8-/16-byte staging paths, edge tiles the wrap / ghost path — with
random data, walls (nonzero Dirichlet data) or periodic, both parities,
against the oracle at the same per-order tolerances as the golden tests.
"""

import numpy as np
import pytest

import paper_1802_05246_b200 as hb
from oracle import hermite_oracle as O
from test_gpu_parity import ALL_TOL, VALUE_TOL, rel, value_rel

pytestmark = pytest.mark.gpu

NX, NY, LAM, C = 40, 70, 0.9, 1.1
X2D = (-0.3, 0.9, 0.2, 2.3)
BCX = ("dirichlet0", "neumann0", 0.4, 0.0)
BCY = ("neumann0", "dirichlet0", 0.0, -0.3)


def setup(m, walls, par, seed):
    grid = hb.Grid2D(*X2D, NX, NY, not walls)
    bc = hb.BoundarySpec2D(hb.BoundarySpec(*BCX), hb.BoundarySpec(*BCY)) if walls else hb.BoundarySpec2D()
    obx, oby = (BCX, BCY) if walls else (O.PERIODIC_BC, O.PERIODIC_BC)
    rng = np.random.default_rng(seed)
    shp = (grid.axis(0).n_nodes(par), grid.axis(1).n_nodes(par))
    return grid, bc, obx, oby, rng, shp


CASES = [(m, walls, par) for m in range(1, 9) for walls, par in ((False, O.PRIMAL), (True, O.DUAL), (True, O.PRIMAL))]


@pytest.mark.parametrize("m,walls,par", CASES)
def test_dissipative_interior(m, walls, par):
    grid, bc, obx, oby, rng, shp = setup(m, walls, par, 100 + m)
    u = rng.standard_normal(shp + (m + 1, m + 1))
    v = rng.standard_normal(shp + (m, m))
    cfg = hb.SchemeConfig(m=m, lam=LAM, speed=C)
    out = hb.half_step_2d(hb.FieldPair(hb.Field2D(grid, par, 0.0, u), hb.Field2D(grid, par, 0.0, v)), cfg, bc)
    wu, wv = O.half_step_2d(u, v, par, NX, NY, not walls, grid.hx, grid.hy, m, LAM, C, obx, oby)
    for got, want in ((out.u.values, wu), (out.v.values, wv)):
        assert got.shape == want.shape
        assert value_rel(got, want) <= VALUE_TOL[m]
        assert rel(got, want) <= ALL_TOL[m]


@pytest.mark.parametrize("m,walls,par", CASES)
def test_conservative_and_bootstrap_interior(m, walls, par):
    grid, bc, obx, oby, rng, shp = setup(m, walls, par, 200 + m)
    tp = hb.flip(par)
    cur = rng.standard_normal(shp + (m + 1, m + 1))
    prev = rng.standard_normal((grid.axis(0).n_nodes(tp), grid.axis(1).n_nodes(tp), m + 1, m + 1))
    cfg = hb.SchemeConfig(m=m, lam=LAM, speed=C)
    st = hb.full_step_conservative(hb.TwoLevelState(hb.Field2D(grid, par, 0.0, cur),
                                                    hb.Field2D(grid, tp, -0.1, prev)), cfg, bc)
    want = O.cons_step_2d(cur, prev, par, not walls, grid.hx, grid.hy, m, LAM, C, obx, oby)
    assert rel(st.current.values, want) <= ALL_TOL[m]
    g1 = rng.standard_normal(shp + (m + 1, m + 1))
    b = hb.bootstrap_first_half(hb.Field2D(grid, par, 0.0, cur), hb.Field2D(grid, par, 0.0, g1), cfg, bc)
    wb = O.bootstrap_2d(cur, g1, par, not walls, grid.hx, grid.hy, m, LAM, C, obx, oby)
    assert rel(b.current.values, wb) <= ALL_TOL[m]
