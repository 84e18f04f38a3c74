"""The reference's long-horizon acceptance criteria on the device
(test_acceptance.py:107-135 criterion 4, :262-297 criterion 7): 10^4
conservative steps keep the exact 1D energy to 1e-8 (smooth data, and below
random data's drift), 10^4 dissipative half steps stay bounded by twice the
initial sup norm.  Same configurations and thresholds as the reference."""

import math
from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _drift(m, mode, steps=10_000, lam=0.5, n0=30, seed=123):
    from paper_1802_05246_b200 import studies as S

    cfg = replace(S.default_config("conserve1d"), m=m, mode=mode, steps=steps, lam=lam, n0=n0, seed=seed).validate()
    _, _, deltas, e0 = S.run_conservation_1d(cfg)
    return float(np.max(np.abs(deltas)) / e0)


@pytest.mark.parametrize("m", [1, 3])
def test_criterion4_smooth_energy_drift(m):
    assert _drift(m, "smooth") <= 1e-8


def test_criterion4_smooth_below_random():
    assert _drift(1, "smooth") < _drift(1, "random")


@pytest.mark.parametrize("m", [1, 2, 3, 4])
def test_criterion7_conservative_long_run(m):
    assert _drift(m, "smooth", lam=1.0, n0=10) <= 1e-8


@pytest.mark.parametrize("m", [1, 2, 3, 4])
def test_criterion7_dissipative_long_run(m):
    import torch

    import paper_1802_05246_b200 as hb

    n = 10
    grid = hb.Grid1D(-math.pi, math.pi, n, True)
    cfg = hb.SchemeConfig(m=m, lam=1.0)
    bc = hb.BoundarySpec()
    xs = grid.nodes(hb.PRIMAL)
    h = grid.h
    u = np.stack([np.sin(xs + l * math.pi / 2) * h**l / math.factorial(l) for l in range(m + 1)], axis=-1)
    v = np.stack([-np.cos(xs + l * math.pi / 2) * h**l / math.factorial(l) for l in range(m)], axis=-1)
    pair = hb.FieldPair(hb.Field1D(grid, hb.PRIMAL, 0.0, torch.from_numpy(u).cuda()),
                        hb.Field1D(grid, hb.PRIMAL, 0.0, torch.from_numpy(v).cuda()))
    sup0 = float(np.abs(u[:, 0]).max())
    sup = sup0
    for k in range(10_000):
        pair = hb.half_step_1d(pair, cfg, bc)
        if (k + 1) % 100 == 0:
            vals = pair.u.values.cpu().numpy()
            assert np.all(np.isfinite(vals))
            sup = max(sup, float(np.abs(vals[:, 0]).max()))
    assert sup <= 2.0 * sup0


# criteria 1-3 (test_acceptance.py:53-100): the refinement studies of both
# schemes in 1D and 2D on the driver's default ladders; the device runs must
# reproduce the reference's own errors and fitted rates (tests/golden/acceptance.npz,
# tests/golden/make_golden_acceptance.py) — including the cells the reference
# itself reports outside the design-order window at these resolutions.
ACC = ([("gaussian1d", "dissipative", m, lam) for m in (1, 2, 3, 4) for lam in (0.8, 1.0)]
       + [("gaussian1d", "conservative", m, lam) for m in (1, 2, 3) for lam in (0.8, 1.0)]
       + [("planewave2d", "dissipative", m, lam) for m in (1, 2, 3) for lam in (0.8, 1.0)]
       + [("planewave2d", "conservative", m, lam) for m in (1, 2, 3) for lam in (0.8, 1.0)])


@pytest.fixture(scope="module")
def acc_gold():
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "acceptance.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("exp,scheme,m,lam", ACC, ids=[f"{e}-{s[:4]}-m{m}-{lam}" for e, s, m, lam in ACC])
def test_criteria_1_to_3_rates_match_reference(acc_gold, exp, scheme, m, lam):
    from paper_1802_05246_b200 import studies as S

    cfg = replace(S.default_config(exp), scheme=scheme, m=m, lam=lam).validate()
    rep = S.run_experiment(cfg)
    k = f"{exp}/{scheme[:4]}/m{m}/lam{lam}"
    np.testing.assert_array_equal(rep.ns, acc_gold[f"{k}/ns"])
    # initial data come from the device generators (ulp-level differences from the reference's numpy
    # evaluation, tests/test_init1d.py), so errors near round-off carry an absolute floor
    np.testing.assert_allclose(rep.err_u, acc_gold[f"{k}/err_u"], rtol=1e-9, atol=1e-14)
    assert rep.rate() == pytest.approx(float(acc_gold[f"{k}/rate"]), abs=1e-6)


# criterion 5 (test_acceptance.py:141-203): one step is exact for the cell
# interpolant — the d'Alembert centre value of the interpolated pair, and the
# conservative average of the interpolant at +-rho h — to 1e-12.
@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("lam", [0.5, 1.0])
def test_criterion5_dissipative_polynomial_exactness(m, lam):
    from numpy.polynomial import Polynomial as Poly

    import paper_1802_05246_b200 as hb
    from oracle import hermite_oracle as O

    rng = np.random.default_rng(500 + m)
    n = 6
    grid = hb.Grid1D(0.0, 3.0, n, True)
    u = rng.standard_normal((n, m + 1))
    v = rng.standard_normal((n, m))
    out = hb.half_step_1d(hb.FieldPair(hb.Field1D(grid, hb.PRIMAL, 0.0, u), hb.Field1D(grid, hb.PRIMAL, 0.0, v)),
                          hb.SchemeConfig(m=m, lam=lam), hb.BoundarySpec())
    ud = O.pair_data(u, O.PRIMAL, True, O.PERIODIC_BC)
    vd = O.pair_data(v, O.PRIMAL, True, O.PERIODIC_BC)
    scale = np.abs(ud).max()
    h, s0 = grid.h, 0.5 * lam
    worst = 0.0
    for i in range(n):
        pu, pv = Poly(O.interp_1d(ud[i])), Poly(O.interp_1d(vd[i]))
        qint, dp = pv.integ(), pu.deriv()
        uref = 0.5 * (pu(s0) + pu(-s0)) + (h / 2.0) * (qint(s0) - qint(-s0))
        vref = (1.0 / (2 * h)) * (dp(s0) - dp(-s0)) + 0.5 * (pv(s0) + pv(-s0))
        worst = max(worst, abs(out.u.values[i, 0] - uref) / scale, abs(out.v.values[i, 0] - vref) / scale)
    assert worst <= 1e-12


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("lam", [0.5, 1.0])
def test_criterion5_conservative_polynomial_exactness(m, lam):
    from numpy.polynomial import Polynomial as Poly

    import paper_1802_05246_b200 as hb
    from oracle import hermite_oracle as O

    rng = np.random.default_rng(520 + m)
    n = 6
    grid = hb.Grid1D(0.0, 3.0, n, True)
    cur = rng.standard_normal((n, m + 1))
    prev = rng.standard_normal((n, m + 1))
    out = hb.full_step_conservative(hb.TwoLevelState(hb.Field1D(grid, hb.PRIMAL, 0.0, cur),
                                                     hb.Field1D(grid, hb.DUAL, -0.1, prev)),
                                    hb.SchemeConfig(m=m, lam=lam), hb.BoundarySpec())
    coeffs = O.interp_1d(O.pair_data(cur, O.PRIMAL, True, O.PERIODIC_BC))
    scale = np.abs(coeffs).max()
    rho = 0.5 * lam
    worst = 0.0
    for i in range(n):
        p = Poly(coeffs[i])  # in the cell's scaled variable (x - centre) / h
        ref = 2.0 * (0.5 * (p(rho) + p(-rho))) - prev[i, 0]
        worst = max(worst, abs(out.current.values[i, 0] - ref) / scale)
    assert worst <= 1e-12


# criterion 8 (test_acceptance.py:298-322): reflections are involutions, and a
# Dirichlet (Neumann) wall suppresses the even (odd) interpolant coefficients.
@pytest.mark.parametrize("m", [1, 2, 3, 4])
def test_criterion8_reflections(m):
    import paper_1802_05246_b200 as hb

    rng = np.random.default_rng(800 + m)
    data = rng.standard_normal((6, m + 1))
    for kind in ("dirichlet0", "neumann0"):
        assert np.array_equal(hb.ghost_data(hb.ghost_data(data, kind), kind), data)
    b = np.random.default_rng(810 + m).standard_normal(m + 1)
    scale = np.abs(b).max()
    even = hb.apply_interp(np.stack([hb.ghost_data(b[None], "dirichlet0")[0], b]))
    odd = hb.apply_interp(np.stack([hb.ghost_data(b[None], "neumann0")[0], b]))
    assert np.abs(even[0::2]).max() / scale <= 1e-13
    assert np.abs(odd[1::2]).max() / scale <= 1e-13
