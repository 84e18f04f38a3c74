"""Parity at BASELINE.json's full sizes through windowed oracle checks and
size-independent properties (the oracle cannot step a whole 16384^2 grid):

  * C2 (periodic m=4, 1024^2) and C5 at its single-GPU size (m=6, 8192^2): one device half step,
    then oracle windows (rows x columns, periodic wrap) at the grid's
    corners and middle;
  * C3 (conservative m=5, 2048^2, Dirichlet x / Neumann y): reversibility —
    N steps forward, swap the levels, N steps back returns the start.  Any
    update new = F(cur) - prev has this property, so it checks the in-place
    two-level bookkeeping, not the operator: the operator at full size is
    pinned by tests/test_c3.py's wall-corner oracle windows and the energy by
    tests/test_energy_cons2d.py;
  * 2D -> 1D reduction on y-independent data (test_dissipative.py:266-302,
    test_conservative.py:212-238).
"""

import math

import numpy as np
import pytest

from oracle import hermite_oracle as O

pytestmark = pytest.mark.gpu


def window_2d(u, v, parity, r0, nr, c0, nc, h, m, lam):
    """Oracle half step for target rows [r0, r0+nr) x cols [c0, c0+nc) of a
    periodic grid (host arrays u, v of the whole grid)."""
    off = 0 if parity == O.PRIMAL else -1
    nx, ny = u.shape[:2]
    rows = (np.arange(r0 + off, r0 + off + nr + 1)) % nx
    cols = (np.arange(c0 + off, c0 + off + nc + 1)) % ny

    def corners(f):
        w = f[rows][:, cols]
        a = O.gather(w, 0, "x", O.PRIMAL, False, None, None)
        return np.moveaxis(O.gather(a, 2, "y", O.PRIMAL, False, None, None), 1, 2)

    return O._step_from_corners(corners(u), corners(v), h, h, m, lam)


def rel(got, want):
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))


def noise_floor(us, vs, r0, nr, c0, nc, h, m, lam, seed=0):
    """The oracle's own rounding sensitivity on this window: max change of
    every output under a 1-ulp relative perturbation of the inputs (SURVEY
    App. A.4's sigma_ref)."""
    rng = np.random.default_rng(seed)
    wu, wv = window_2d(us, vs, O.PRIMAL, r0, nr, c0, nc, h, m, lam)
    up = us * (1.0 + 2.2e-16 * rng.standard_normal(us.shape))
    vp = vs * (1.0 + 2.2e-16 * rng.standard_normal(vs.shape))
    pu, pv = window_2d(up, vp, O.PRIMAL, r0, nr, c0, nc, h, m, lam)
    return wu, wv, np.abs(pu - wu), np.abs(pv - wv)


@pytest.mark.parametrize("m,n", [(4, 1024), (6, 8192)])
def test_full_size_windows_match_oracle(m, n):
    """C2 (m=4, 1024^2) and C5's single-GPU size (m=6, 8192^2, 45.6 GB per level):
    one device half step; 5 x 40 target windows at the corner, the middle and
    the far edge (periodic wrap) agree with the oracle to within 10x the
    oracle's own 1-ulp sensitivity on the same window."""
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import diss2d_into

    lam = 0.9
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    try:
        ud, vd = torch.empty_like(u), torch.empty_like(v)
        diss2d_into(u, v, ud, vd, grid, hb.PRIMAL, m, hb.SchemeConfig(m=m, lam=lam), hb.BoundarySpec2D())
        torch.cuda.synchronize()
        hb.require_finite(ud, vd)
        nr, nc = 5, 40
        for r0, c0 in [(0, 0), (n // 2 - 3, n // 2 - 17), (n - 5, n - 40)]:
            # the source window (rows r0..r0+nr, cols c0..c0+nc, periodic) as a small array
            ridx = torch.as_tensor(np.arange(r0, r0 + nr + 1) % n, device="cuda")
            cidx = torch.as_tensor(np.arange(c0, c0 + nc + 1) % n, device="cuda")
            us = u.index_select(0, ridx).index_select(1, cidx).cpu().numpy()
            vs = v.index_select(0, ridx).index_select(1, cidx).cpu().numpy()
            wu, wv, su, sv = noise_floor(us, vs, 0, nr, 0, nc, grid.hx, m, lam)
            gu = ud[r0:r0 + nr, c0:c0 + nc].cpu().numpy()
            gv = vd[r0:r0 + nr, c0:c0 + nc].cpu().numpy()
            for got, want, sig in ((gu, wu, su), (gv, wv, sv)):
                floor = 1e-15 * np.max(np.abs(want))
                assert np.max(np.abs(got - want)) <= 10.0 * np.max(sig) + floor
                d00 = np.max(np.abs(got[..., 0, 0] - want[..., 0, 0]))
                assert d00 <= max(10.0 * np.max(sig[..., 0, 0]), 1e-13 * np.max(np.abs(want[..., 0, 0])))
    finally:
        del u, v
        torch.cuda.empty_cache()


def test_c3_time_reversal_full_size():
    import torch

    import paper_1802_05246_b200 as hb

    m, n, nsteps = 5, 2048, 20
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0"), hb.BoundarySpec("neumann0", "neumann0"))
    dt = cfg.dt(grid.hx)
    pi = math.pi
    om = pi * math.sqrt(2.0)
    a0 = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.0, m, m, pi, pi, om, py=0.5 * pi)
    b0 = hb.standing_wave_on_grid(grid, hb.DUAL, -0.5 * dt, m, m, pi, pi, om, py=0.5 * pi)
    st = hb.TwoLevelState(hb.Field2D(grid, hb.PRIMAL, 0.0, a0.clone()),
                          hb.Field2D(grid, hb.DUAL, -0.5 * dt, b0.clone()))
    fwd = hb.advance_conservative(st, cfg, bc, nsteps)
    back = hb.advance_conservative(hb.TwoLevelState(fwd.previous, fwd.current), cfg, bc, nsteps)
    # after the swap, N steps back land on (previous0, current0)
    gb = back.current.values
    ga = back.previous.values
    torch.cuda.synchronize()
    assert back.current.parity == hb.DUAL and back.previous.parity == hb.PRIMAL
    for got, want in ((gb, b0), (ga, a0)):
        d = (got - want).abs()
        assert float(d[..., 0, 0].max()) <= 1e-12 * float(want[..., 0, 0].abs().max())
        assert float(d.max()) <= 1e-8 * float(want.abs().max())


@pytest.mark.parametrize("m", [2, 4, 6])
def test_2d_reduces_to_1d_on_y_independent_data(m):
    """test_dissipative.py:266-302 / test_conservative.py:212-238 on the device."""
    import paper_1802_05246_b200 as hb

    n = 9
    rng = np.random.default_rng(40 + m)
    g2 = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    g1 = hb.Grid1D(0.0, 1.0, n, True)
    cfg = hb.SchemeConfig(m=m, lam=0.85)
    u1 = rng.standard_normal((n, m + 1))
    v1 = rng.standard_normal((n, m))
    u2 = np.zeros((n, n, m + 1, m + 1))
    v2 = np.zeros((n, n, m, m))
    u2[:, :, :, 0] = u1[:, None, :]
    v2[:, :, :, 0] = v1[:, None, :]
    p2 = hb.half_step_2d(hb.FieldPair(hb.Field2D(g2, hb.PRIMAL, 0.0, u2), hb.Field2D(g2, hb.PRIMAL, 0.0, v2)),
                         cfg, hb.BoundarySpec2D())
    p1 = hb.half_step_1d(hb.FieldPair(hb.Field1D(g1, hb.PRIMAL, 0.0, u1), hb.Field1D(g1, hb.PRIMAL, 0.0, v1)),
                         cfg, hb.BoundarySpec())
    # high orders amplify rounding by cond(M_mu): 1e-12 at m <= 3 as in the
    # reference test, 1e-11 / 1e-9 of the output scale at m = 4 / 6
    scale = {2: 1e-12, 4: 1e-11, 6: 1e-9}[m] * max(np.abs(p1.u.values).max(), np.abs(p1.v.values).max()) / 1e-12
    np.testing.assert_allclose(p2.u.values[:, :, :, 0], np.broadcast_to(p1.u.values[:, None, :], (n, n, m + 1)),
                               rtol=0, atol=1e-12 * scale)
    np.testing.assert_allclose(p2.u.values[:, :, :, 1:], 0.0, atol=1e-12 * scale)
    np.testing.assert_allclose(p2.v.values[:, :, :, 0], np.broadcast_to(p1.v.values[:, None, :], (n, n, m)),
                               rtol=0, atol=1e-12 * scale)
    cur1 = rng.standard_normal((n, m + 1))
    prev1 = rng.standard_normal((n, m + 1))
    cur2 = np.zeros((n, n, m + 1, m + 1))
    prev2 = np.zeros((n, n, m + 1, m + 1))
    cur2[:, :, :, 0] = cur1[:, None, :]
    prev2[:, :, :, 0] = prev1[:, None, :]
    o1 = hb.full_step_conservative(hb.TwoLevelState(hb.Field1D(g1, hb.PRIMAL, 0.0, cur1),
                                                    hb.Field1D(g1, hb.DUAL, -0.1, prev1)), cfg, hb.BoundarySpec())
    o2 = hb.full_step_conservative(hb.TwoLevelState(hb.Field2D(g2, hb.PRIMAL, 0.0, cur2),
                                                    hb.Field2D(g2, hb.DUAL, -0.1, prev2)), cfg, hb.BoundarySpec2D())
    sc = {2: 1e-12, 4: 1e-11, 6: 1e-9}[m] * np.abs(o1.current.values).max() / 1e-12
    np.testing.assert_allclose(o2.current.values[:, :, :, 0],
                               np.broadcast_to(o1.current.values[:, None, :], (n, n, m + 1)), rtol=0, atol=1e-12 * sc)
    np.testing.assert_allclose(o2.current.values[:, :, :, 1:], 0.0, atol=1e-12 * sc)
