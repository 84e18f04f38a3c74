"""1D energies (diagnostics.py:190-234): the oracle restatement against the
reference's own values (tests/golden/energy.npz, tests/golden/make_golden_energy.py)
on the CPU, and the device reductions against both on a B200."""

import os

import numpy as np
import pytest

from oracle import hermite_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "energy.npz")
X1D = (-0.4, 1.1)
DISS = [("p_m1", 1, 9, True, O.PRIMAL, None, 1.0), ("p_m2_dual", 2, 8, True, O.DUAL, None, 1.7),
        ("p_m3", 3, 12, True, O.PRIMAL, None, 0.6), ("p_m5", 5, 7, True, O.DUAL, None, 1.0),
        ("w_m3_primal", 3, 8, False, O.PRIMAL, ("dirichlet0", "neumann0", 0.3, 0.0), 1.0),
        ("w_m4_dual", 4, 6, False, O.DUAL, ("neumann0", "dirichlet0", 0.0, -0.5), 2.0)]
CONS = [("m1", 1, 10, O.PRIMAL, 0.9, 1.0), ("m2_dual", 2, 9, O.DUAL, 0.5, 1.3), ("m3_lam1", 3, 8, O.PRIMAL, 1.0, 1.0),
        ("m4", 4, 11, O.DUAL, 0.7, 0.8), ("m6", 6, 6, O.PRIMAL, 0.9, 1.0)]


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def _h(n):
    return (X1D[1] - X1D[0]) / n


@pytest.mark.parametrize("case", DISS, ids=[c[0] for c in DISS])
def test_oracle_dissipative_energy(gold, case):
    name, m, n, per, par, bcs, speed = case
    bc = O.PERIODIC_BC if bcs is None else bcs
    e = O.dissipative_energy_1d(gold[f"ed/{name}/u"], gold[f"ed/{name}/v"], par, n, per, _h(n), speed, bc)
    assert e == pytest.approx(float(gold[f"ed/{name}/e"]), rel=1e-13)


@pytest.mark.parametrize("case", CONS, ids=[c[0] for c in CONS])
def test_oracle_conservative_energy(gold, case):
    name, m, n, par, lam, speed = case
    h = _h(n)
    dt = lam * h / speed
    e = O.conservative_energy_1d(gold[f"ec/{name}/cur"], gold[f"ec/{name}/prev"], par, n, h, 0.5 * speed * dt)
    assert e == pytest.approx(float(gold[f"ec/{name}/e"]), rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("case", DISS, ids=[c[0] for c in DISS])
def test_device_dissipative_energy(gold, case):
    import paper_1802_05246_b200 as hb

    name, m, n, per, par, bcs, speed = case
    grid = hb.Grid1D(*X1D, n, per)
    bc = hb.BoundarySpec() if bcs is None else hb.BoundarySpec(*bcs)
    pair = hb.FieldPair(hb.Field1D(grid, par, 0.0, gold[f"ed/{name}/u"]),
                        hb.Field1D(grid, par, 0.0, gold[f"ed/{name}/v"]))
    assert hb.dissipative_energy(pair, speed, bc) == pytest.approx(float(gold[f"ed/{name}/e"]), rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CONS, ids=[c[0] for c in CONS])
def test_device_conservative_energy_and_invariance(gold, case):
    import paper_1802_05246_b200 as hb

    name, m, n, par, lam, speed = case
    grid = hb.Grid1D(*X1D, n, True)
    cfg = hb.SchemeConfig(m=m, speed=speed, lam=lam)
    dt = cfg.dt(grid.h)
    bc = hb.BoundarySpec()
    cur = hb.Field1D(grid, par, 0.0, gold[f"ec/{name}/cur"])
    prev = hb.Field1D(grid, hb.flip(par), -0.5 * dt, gold[f"ec/{name}/prev"])
    e0 = hb.conservative_energy(cur, prev, speed, dt, bc)
    assert e0 == pytest.approx(float(gold[f"ec/{name}/e"]), rel=1e-12)
    # the conservative scheme preserves it (test_diagnostics.py:232-251), here
    # through the device stepper, against the reference's own trace
    st = hb.TwoLevelState(cur, prev)
    for k in range(1, 5):
        st = hb.full_step_conservative(st, cfg, bc)
        e = hb.conservative_energy(st.current, st.previous, speed, dt, bc)
        assert e == pytest.approx(float(gold[f"ec/{name}/trace"][k]), rel=1e-11)
        assert e == pytest.approx(e0, rel=1e-11)


@pytest.mark.gpu
def test_device_energy_errors():
    import paper_1802_05246_b200 as hb

    grid = hb.Grid1D(0.0, 1.0, 6, False)
    bc = hb.BoundarySpec("dirichlet0", "dirichlet0")
    f = hb.Field1D(grid, hb.PRIMAL, 0.0, np.zeros((7, 3)))
    g = hb.Field1D(grid, hb.DUAL, 0.0, np.zeros((6, 3)))
    with pytest.raises(ValueError, match="periodic"):
        hb.conservative_energy(f, g, 1.0, 0.1, bc)
    gp = hb.Grid1D(0.0, 1.0, 6, True)
    f = hb.Field1D(gp, hb.PRIMAL, 0.0, np.zeros((6, 3)))
    g = hb.Field1D(gp, hb.DUAL, 0.0, np.zeros((6, 3)))
    with pytest.raises(ValueError, match="shift distance"):
        hb.conservative_energy(f, g, 1.0, 2.0 * gp.h, hb.BoundarySpec())
    assert hb.dissipative_energy(hb.FieldPair(f, hb.Field1D(gp, hb.PRIMAL, 0.0, np.zeros((6, 2)))), 2.0,
                                 hb.BoundarySpec()) == 0.0


# ------------------------------------------------------------ the defined 2D energy
# No reference counterpart exists (the reference's energies are 1D).  It is
# pinned by (i) reduction to the REFERENCE's 1D dissipative energy on
# y-independent data, (ii) an oracle that integrates the interpolants in
# closed form (monomial Gram matrices) rather than by the device's Gauss rule.
PERIODIC_DISS = [c for c in DISS if c[3]]
LY, NY = 0.7, 5


def _extend_y(u1, v1):
    """y-independent 2D fields whose x-profile is the 1D pair (l = 0 blocks)."""
    n, m = u1.shape[0], u1.shape[1] - 1
    u2 = np.zeros((n, NY, m + 1, m + 1))
    v2 = np.zeros((n, NY, m, m))
    u2[:, :, :, 0] = u1[:, None, :]
    v2[:, :, :, 0] = v1[:, None, :]
    return u2, v2


@pytest.mark.parametrize("case", PERIODIC_DISS, ids=[c[0] for c in PERIODIC_DISS])
def test_oracle_energy_2d_reduces_to_reference_1d(gold, case):
    name, m, n, per, par, bcs, speed = case
    u2, v2 = _extend_y(gold[f"ed/{name}/u"], gold[f"ed/{name}/v"])
    e2 = O.dissipative_energy_2d(u2, v2, par, _h(n), LY / NY, speed)
    assert e2 == pytest.approx(LY * float(gold[f"ed/{name}/e"]), rel=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("case", PERIODIC_DISS, ids=[c[0] for c in PERIODIC_DISS])
def test_device_energy_2d_reduces_to_reference_1d(gold, case):
    import paper_1802_05246_b200 as hb

    name, m, n, per, par, bcs, speed = case
    u2, v2 = _extend_y(gold[f"ed/{name}/u"], gold[f"ed/{name}/v"])
    grid = hb.Grid2D(X1D[0], X1D[1], 0.0, LY, n, NY, True)
    pair = hb.FieldPair(hb.Field2D(grid, par, 0.0, u2), hb.Field2D(grid, par, 0.0, v2))
    assert hb.dissipative_energy_2d(pair, speed) == pytest.approx(LY * float(gold[f"ed/{name}/e"]), rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("m,par", [(1, O.PRIMAL), (2, O.DUAL), (4, O.PRIMAL), (6, O.DUAL), (8, O.PRIMAL)])
def test_device_energy_2d_matches_closed_form_oracle(m, par):
    import paper_1802_05246_b200 as hb

    rng = np.random.default_rng(300 + m)
    nx, ny = 9, 7
    grid = hb.Grid2D(-0.2, 0.9, 0.1, 1.3, nx, ny, True)
    u = rng.standard_normal((nx, ny, m + 1, m + 1))
    v = rng.standard_normal((nx, ny, m, m))
    pair = hb.FieldPair(hb.Field2D(grid, par, 0.0, u), hb.Field2D(grid, par, 0.0, v))
    want = O.dissipative_energy_2d(u, v, par, grid.hx, grid.hy, 1.3)
    # Gauss vs closed form: the rounding of a sum of O(cells * npts^2) squares
    # of interpolants amplified by cond(M_mu)
    assert hb.dissipative_energy_2d(pair, 1.3) == pytest.approx(want, rel={8: 1e-9, 6: 1e-11}.get(m, 1e-12))


@pytest.mark.gpu
@pytest.mark.parametrize("m", [2, 4])
def test_device_energy_2d_does_not_grow_under_the_dissipative_step(m):
    """Observed (not proven) analogue of test_dissipative.py:196-230: the
    defined 2D energy of random data is non-increasing over half steps."""
    import paper_1802_05246_b200 as hb

    rng = np.random.default_rng(20 + m)
    n = 16
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    p = hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, rng.standard_normal((n, n, m + 1, m + 1))),
                     hb.Field2D(grid, hb.PRIMAL, 0.0, rng.standard_normal((n, n, m, m))))
    es = [hb.dissipative_energy_2d(p, 1.0)]
    for _ in range(6):
        p = hb.half_step_2d(p, cfg, hb.BoundarySpec2D())
        es.append(hb.dissipative_energy_2d(p, 1.0))
    assert all(b <= a * (1 + 1e-12) for a, b in zip(es, es[1:]))
    assert es[-1] < 0.5 * es[0]


@pytest.mark.gpu
def test_device_energy_2d_errors():
    import paper_1802_05246_b200 as hb

    m = 2
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, 4, 4, False)
    u = np.zeros((5, 5, m + 1, m + 1))
    v = np.zeros((5, 5, m, m))
    with pytest.raises(ValueError, match="periodic"):
        hb.dissipative_energy_2d(hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, u), hb.Field2D(grid, hb.PRIMAL, 0.0, v)), 1.0)
