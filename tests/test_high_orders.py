"""2D steps at the top of the reference's order range, m = 9..12 (interp.py:30
MAX_ORDER = 12; round 1 raised HW_EUNSUPPORTED above m = 8).  They run on the
generic runtime-order SIMT kernel (csrc/simt2d.cuh) — coverage, not a
throughput path.  Goldens: tests/golden/high2d.npz, produced by the reference
(tests/golden/make_golden_high2d.py) with its own 1-ulp sensitivity sigma per
coefficient; cond(M_mu) reaches ~1e10 here, so the tolerance is 10 sigma plus
a 1e-13 floor of the output scale (value coefficients: 1e-11)."""

import os

import numpy as np
import pytest

from cases import HIGH2D_CASES
from oracle import hermite_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "high2d.npz")
BCX = ("dirichlet0", "neumann0", 0.3, 0.0)
BCY = ("neumann0", "dirichlet0", 0.0, -0.2)


@pytest.fixture(scope="module")
def hg():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def _bcs(walls):
    return (BCX, BCY) if walls else (O.PERIODIC_BC, O.PERIODIC_BC)


@pytest.mark.parametrize("case", HIGH2D_CASES, ids=[c[0] for c in HIGH2D_CASES])
def test_oracle_high_orders_match_reference(hg, case):
    name, m, nx, ny, walls, par = case
    bx, by = _bcs(walls)
    hx, hy = 1.0 / nx, 1.2 / ny
    u, v = O.half_step_2d(hg[f"{name}/u0"], hg[f"{name}/v0"], par, nx, ny, not walls, hx, hy, m, 0.9, 1.0, bx, by)
    for got, key in ((u, "u"), (v, "v")):
        np.testing.assert_allclose(got, hg[f"{name}/{key}"], rtol=0, atol=1e-12 * np.max(np.abs(hg[f"{name}/{key}"])))
    c = O.cons_step_2d(hg[f"{name}/cur0"], hg[f"{name}/prev0"], par, not walls, hx, hy, m, 0.9, 1.0, bx, by)
    np.testing.assert_allclose(c, hg[f"{name}/cons"], rtol=0, atol=1e-12 * np.max(np.abs(hg[f"{name}/cons"])))


def _within(got, want, sigma):
    scale = float(np.max(np.abs(want)))
    d = np.abs(got - want).max(axis=(0, 1))
    ok = np.all(d <= 10.0 * sigma + 1e-13 * scale)
    d00 = float(np.max(np.abs(got[..., 0, 0] - want[..., 0, 0])))
    return bool(ok) and d00 <= max(10.0 * float(sigma[0, 0]), 1e-11 * scale), float(np.max(d / scale))


@pytest.mark.gpu
@pytest.mark.parametrize("case", HIGH2D_CASES, ids=[c[0] for c in HIGH2D_CASES])
def test_device_high_orders_vs_reference(hg, case):
    import paper_1802_05246_b200 as hb

    name, m, nx, ny, walls, par = case
    grid = hb.Grid2D(0.0, 1.0, -0.5, 0.7, nx, ny, not walls)
    bc = hb.BoundarySpec2D(hb.BoundarySpec(*BCX), hb.BoundarySpec(*BCY)) if walls else hb.BoundarySpec2D()
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    d = hb.half_step_2d(hb.FieldPair(hb.Field2D(grid, par, 0.0, hg[f"{name}/u0"]),
                                     hb.Field2D(grid, par, 0.0, hg[f"{name}/v0"])), cfg, bc)
    for got, key in ((d.u.values, "u"), (d.v.values, "v")):
        ok, rel = _within(got, hg[f"{name}/{key}"], hg[f"{name}/{key}_sigma"])
        assert ok, (key, rel)
    c = hb.full_step_conservative(hb.TwoLevelState(hb.Field2D(grid, par, 0.0, hg[f"{name}/cur0"]),
                                                   hb.Field2D(grid, hb.flip(par), -0.1, hg[f"{name}/prev0"])), cfg, bc)
    ok, rel = _within(c.current.values, hg[f"{name}/cons"], hg[f"{name}/cons_sigma"])
    assert ok, ("cons", rel)
    b = hb.bootstrap_first_half(hb.Field2D(grid, par, 0.0, hg[f"{name}/cur0"]),
                                hb.Field2D(grid, par, 0.0, hg[f"{name}/g1"]), cfg, bc)
    ok, rel = _within(b.current.values, hg[f"{name}/boot"], hg[f"{name}/boot_sigma"])
    assert ok, ("boot", rel)


@pytest.mark.gpu
def test_device_order_limit():
    import paper_1802_05246_b200 as hb

    m = 13  # beyond MAX_ORDER: the reference's interp_matrix raises ValueError (interp.py:62-63)
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, 3, 3, True)
    u = np.zeros((3, 3, m + 1, m + 1))
    v = np.zeros((3, 3, m, m))
    with pytest.raises(ValueError):
        hb.half_step_2d(hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, u), hb.Field2D(grid, hb.PRIMAL, 0.0, v)),
                        hb.SchemeConfig(m=m, lam=0.9), hb.BoundarySpec2D())
