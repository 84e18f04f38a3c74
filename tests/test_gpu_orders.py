"""Parity depth on the device:

  * observed convergence orders: C2's scheme and CFL (periodic dissipative
    m=4, lambda 0.9, kappa 1 plane wave to t ~ 0.5, n = 6..15) and C3's wall
    setting (conservative, Dirichlet x / Neumann y, sin(3 pi x) cos(3 pi y)
    cos(3 sqrt2 pi t), an even half-step count so every level ends primal,
    m = 2, 3, n = 8..18) against the reference's own ladders
    (tests/golden/ladders.npz from tests/golden/make_golden_ladders.py):
    per-level errors to 1e-9 relative (1e-14 absolute floor), fitted orders
    to 1e-4;
  * a grown-window check at C2's full size: 8 half steps of the 1024^2 grid on
    the device, then the oracle steps a window grown by the 8-step dependency
    cone (one node per side per two half steps) and must agree on the
    interior window within 10x its own 1-ulp sensitivity.
"""

import math
import os

import numpy as np
import pytest

from oracle import hermite_oracle as O

pytestmark = pytest.mark.gpu
# The finest levels' errors (~1e-10 of an O(1) field) carry the state's rounding
# (summation order differs from the reference's BLAS): ~1e-15 absolute, which
# moves the fitted order by ~1e-5.  "Identical observed orders": 4 decimals.
ATOL, RATE_TOL = 1e-14, 1e-4
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ladders.npz")


@pytest.fixture(scope="module")
def lad():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def test_c2_ladder_orders_match_reference(lad):
    import paper_1802_05246_b200 as hb

    m, lam = 4, 0.9
    cfg = hb.SchemeConfig(m=m, lam=lam)
    errs, hs = [], []
    for n, nhalf in zip(lad["c2/n"], lad["c2/nhalf"]):
        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, int(n), int(n), True)
        dt = cfg.dt(grid.hx)
        assert round(1.0 / dt) == nhalf
        pair = hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, hb.planewave_on_grid(grid, hb.PRIMAL, 0.0, m, m, 1)),
                            hb.Field2D(grid, hb.PRIMAL, 0.0,
                                       hb.planewave_on_grid(grid, hb.PRIMAL, 0.0, m - 1, m - 1, 1, tder=1)))
        pair = hb.advance_2d(pair, cfg, hb.BoundarySpec2D(), int(nhalf))
        errs.append(hb.l2_error_field_2d(pair.u, hb.PlaneWave2D(kappa=1, t=pair.u.time), hb.BoundarySpec2D()))
        hs.append(grid.hx)
    np.testing.assert_allclose(errs, lad["c2/err"], rtol=1e-9, atol=ATOL)
    assert hb.fit_rate(hs, errs) == pytest.approx(float(lad["c2/rate"]), abs=RATE_TOL)


@pytest.mark.parametrize("m", [2, 3])
def test_c3_wall_ladder_orders_match_reference(lad, m):
    import paper_1802_05246_b200 as hb

    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0"), hb.BoundarySpec("neumann0", "neumann0"))
    k = 3.0 * math.pi
    errs, hs = [], []
    for n, nhalf in zip(lad[f"walls_m{m}/n"], lad[f"walls_m{m}/nhalf"]):
        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, int(n), int(n), False)
        dt = cfg.dt(grid.hx)

        def wave(par, t):
            return hb.standing_wave_on_grid(grid, par, t, m, m, k, k, math.sqrt(2.0) * k, py=0.5 * math.pi)

        st = hb.TwoLevelState(hb.Field2D(grid, hb.PRIMAL, 0.0, wave(hb.PRIMAL, 0.0)),
                              hb.Field2D(grid, hb.DUAL, -0.5 * dt, wave(hb.DUAL, -0.5 * dt)))
        st = hb.advance_conservative(st, cfg, bc, int(nhalf))
        assert st.current.parity == hb.PRIMAL
        t = st.current.time

        def exact(X, Y, t=t):
            return np.sin(k * X) * np.cos(k * Y) * math.cos(math.sqrt(2.0) * k * t)

        errs.append(hb.l2_error_field_2d(st.current, exact, bc))
        hs.append(grid.hx)
    np.testing.assert_allclose(errs, lad[f"walls_m{m}/err"], rtol=1e-9, atol=ATOL)
    assert hb.fit_rate(hs, errs) == pytest.approx(float(lad[f"walls_m{m}/rate"]), abs=RATE_TOL)


def _grown_window_steps(u, v, nsteps, h, m, lam):
    """The oracle's half steps on a window: every step gathers consecutive node
    pairs (targets t <- t, t+1 from primal; p <- p-1, p from dual), so the
    window shrinks by one node per axis per step."""
    for _ in range(nsteps):
        def corners(f):
            a = O.gather(f, 0, "x", O.PRIMAL, False, None, None)
            return np.moveaxis(O.gather(a, 2, "y", O.PRIMAL, False, None, None), 1, 2)

        u, v = O._step_from_corners(corners(u), corners(v), h, h, m, lam)
    return u, v


def test_c2_full_size_grown_window_after_8_half_steps():
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import diss2d_into

    m, n, lam, steps = 4, 1024, 0.9, 8
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    cfg = hb.SchemeConfig(m=m, lam=lam)
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    bufs = [(u.clone(), v.clone()), (torch.empty_like(u), torch.empty_like(v))]
    par = hb.PRIMAL
    for i in range(steps):
        diss2d_into(*bufs[i % 2], *bufs[(i + 1) % 2], grid, par, m, cfg, hb.BoundarySpec2D())
        par = hb.flip(par)
    ud, vd = bufs[steps % 2]
    torch.cuda.synchronize()
    # after 8 half steps (4 primal->dual->primal pairs) primal target p depends on
    # primal sources p-4 .. p+4: a W-node window needs the W + 8 source nodes around it
    W = 12
    rng = np.random.default_rng(11)
    for r0, c0 in [(0, 0), (500, 260), (n - 6, n - 6)]:  # corner (periodic wrap), middle, far edge
        ridx = np.arange(r0 - 4, r0 + W + 4) % n
        cidx = np.arange(c0 - 4, c0 + W + 4) % n
        us = u.cpu().numpy()[ridx][:, cidx]
        vs = v.cpu().numpy()[ridx][:, cidx]
        wu, wv = _grown_window_steps(us, vs, steps, grid.hx, m, lam)
        pu, pv = _grown_window_steps(us * (1.0 + 2.2e-16 * rng.standard_normal(us.shape)),
                                     vs * (1.0 + 2.2e-16 * rng.standard_normal(vs.shape)), steps, grid.hx, m, lam)
        assert wu.shape[:2] == (W, W)
        ti, tj = np.arange(r0, r0 + W) % n, np.arange(c0, c0 + W) % n
        gu = ud.cpu().numpy()[ti][:, tj]
        gv = vd.cpu().numpy()[ti][:, tj]
        for got, want, pert in ((gu, wu, pu), (gv, wv, pv)):
            sig = np.abs(pert - want)
            scale = np.max(np.abs(want))
            assert np.max(np.abs(got - want)) <= 10.0 * np.max(sig) + 1e-15 * scale
            assert np.max(np.abs(got[..., 0, 0] - want[..., 0, 0])) <= max(10.0 * np.max(sig[..., 0, 0]),
                                                                             1e-13 * scale)
