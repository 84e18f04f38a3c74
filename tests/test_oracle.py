"""Pin the CPU oracle (oracle/hermite_oracle.py) against the golden vectors the
reference itself produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from cases import CASES_1D, CASES_2D, PERIODIC_BC, X1D, X2D, exact2d, forcing_fn
from oracle import hermite_oracle as O


def _bcs(bcx, bcy):
    return (PERIODIC_BC, PERIODIC_BC) if bcx is None else (tuple(bcx), tuple(bcy))


def _h2d(nx, ny):
    return (X2D[1] - X2D[0]) / nx, (X2D[3] - X2D[2]) / ny


def assert_same(got, want, rtol=0.0):
    """Bitwise unless rtol given (then relative to the array's max norm)."""
    if rtol == 0.0:
        np.testing.assert_array_equal(got, want)
    else:
        scale = max(1.0, float(np.max(np.abs(want))))
        np.testing.assert_allclose(got, want, rtol=0, atol=rtol * scale)


@pytest.mark.parametrize("mu", range(13))
def test_interp_matrix_exact(golden, mu):
    assert_same(O.hermite_matrix(mu), golden[f"interp/{mu}"])


@pytest.mark.parametrize("case", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_oracle_half_step_2d(golden, case):
    name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps = case
    bx, by = _bcs(bcx, bcy)
    hx, hy = _h2d(nx, ny)
    u, v = golden[f"d2/{name}/u0"], golden[f"d2/{name}/v0"]
    p = par
    for _ in range(steps):
        u, v = O.half_step_2d(u, v, p, nx, ny, per, hx, hy, m, lam, c, bx, by, cap)
        p = O.flip(p)
    assert_same(u, golden[f"d2/{name}/u"])
    assert_same(v, golden[f"d2/{name}/v"])


@pytest.mark.parametrize("case", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_oracle_conservative_2d(golden, case):
    name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps = case
    bx, by = _bcs(bcx, bcy)
    hx, hy = _h2d(nx, ny)
    cur, prev = golden[f"c2/{name}/cur0"], golden[f"c2/{name}/prev0"]
    p = par
    for _ in range(steps):
        cur, prev = O.cons_step_2d(cur, prev, p, per, hx, hy, m, lam, c, bx, by), cur
        p = O.flip(p)
    assert_same(cur, golden[f"c2/{name}/cur"])
    assert_same(prev, golden[f"c2/{name}/prev"])
    boot = O.bootstrap_2d(golden[f"c2/{name}/cur0"], golden[f"b2/{name}/g1"], par, per, hx, hy, m, lam, c,
                          bx, by)
    assert_same(boot, golden[f"b2/{name}/out"])


@pytest.mark.parametrize("case", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_oracle_l2_2d(golden, case):
    name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps = case
    bx, by = _bcs(bcx, bcy)
    hx, hy = _h2d(nx, ny)
    for fld in ("u", "v"):
        vals = golden[f"d2/{name}/{fld}0"]
        e = O.l2_error_2d(vals, par, nx, ny, per, X2D[0], X2D[2], hx, hy, exact2d, bcx=bx, bcy=by)
        assert_same(e, golden[f"e2/{name}/{fld}"])


def test_oracle_planewave(golden):
    h = 1.0 / 7
    xp = O.nodes(0.0, h, 7, True, O.DUAL)
    assert_same(O.planewave_data(xp, xp, 0.3, 4, 4, 5, h, h), golden["init/planewave_u"])
    assert_same(O.planewave_data(xp, xp, 0.3, 3, 3, 5, h, h, tder=1), golden["init/planewave_v"])


@pytest.mark.parametrize("case", CASES_1D, ids=[c[0] for c in CASES_1D])
def test_oracle_1d(golden, case):
    name, m, n, per, par, bcs, lam, c, cap, steps, forced = case
    bc = PERIODIC_BC if bcs is None else tuple(bcs)
    h = (X1D[1] - X1D[0]) / n
    u, v = golden[f"d1/{name}/u0"], golden[f"d1/{name}/v0"]
    p, t = par, 0.0
    for _ in range(steps):
        u, v = O.half_step_1d(u, v, p, n, per, X1D[0], h, m, lam, c, bc, cap,
                              forcing_fn if forced else None, t)
        t = t + 0.5 * lam * h / c
        p = O.flip(p)
    assert_same(u, golden[f"d1/{name}/u"])
    assert_same(v, golden[f"d1/{name}/v"])
    if forced:
        return
    cur, prev = golden[f"c1/{name}/cur0"], golden[f"c1/{name}/prev0"]
    p = par
    for _ in range(steps):
        cur, prev = O.cons_step_1d(cur, prev, p, n, per, m, lam, bc), cur
        p = O.flip(p)
    assert_same(cur, golden[f"c1/{name}/cur"])
    assert_same(prev, golden[f"c1/{name}/prev"])
    boot = O.bootstrap_1d(golden[f"c1/{name}/cur0"], golden[f"b1/{name}/g1"], par, n, per, h, m, lam, c, bc)
    assert_same(boot, golden[f"b1/{name}/out"])
    u0, v0 = golden[f"d1/{name}/u0"], golden[f"d1/{name}/v0"]
    eu = O.l2_error_1d(u0, par, n, per, X1D[0], h, np.sin, bc=bc)
    ed = O.l2_error_1d(u0, par, n, per, X1D[0], h, np.cos, bc=bc, deriv=1, npts=2 * m + 2)
    ev = O.l2_error_1d(v0, par, n, per, X1D[0], h, lambda x: -np.sin(2 * x), bc=bc, npts=2 * m + 2)
    assert_same(np.array([eu, ed, ev]), golden[f"e1/{name}/pair"])
    assert_same(eu, golden[f"e1/{name}/field"])
