"""Refinement studies and conservation traces on the device (studies.py),
against the reference driver's own results on the same configurations
(tests/golden/studies.npz from tests/golden/make_golden_studies.py).  The
config/CSV plumbing is checked on the CPU, mirroring test_driver.py."""

import os

import numpy as np
import pytest

from paper_1802_05246_b200 import studies as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "studies.npz")
STUDIES = {
    "pw2d_diss_m3": ("planewave2d", dict(m=3, lam=0.9, levels=4, n0=6)),
    "pw2d_cons_m2_exact": ("planewave2d", dict(scheme="conservative", m=2, lam=0.9, levels=4, n0=6)),
    "pw2d_cons_m2_boot": ("planewave2d", dict(scheme="conservative", m=2, lam=0.7, levels=3, n0=6,
                                              init="bootstrap")),
    "g1d_diss_m3": ("gaussian1d", dict(m=3, levels=4, n0=10)),
    "g1d_cons_m2_boot": ("gaussian1d", dict(scheme="conservative", m=2, levels=4, n0=12, init="bootstrap",
                                            boundary="neumann0")),
    "g1d_diss_m2_per": ("gaussian1d", dict(m=2, levels=3, n0=12, boundary="periodic", lam=0.9)),
    "c1d_smooth_m2": ("conserve1d", dict(m=2, steps=300, sample_every=100)),
    # the driver's default ladders: observed orders in the asymptotic range
    "pw2d_default_m4": ("planewave2d", dict(m=4)),
    "g1d_default_m3": ("gaussian1d", dict(m=3)),
    "c1d_random_m3": ("conserve1d", dict(m=3, steps=200, sample_every=50, mode="random", seed=7)),
}


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def test_level_ladder_and_defaults():
    cfg = S.default_config("planewave2d")
    assert (cfg.levels, cfg.n0, cfg.lam) == (5, 10, 0.8)
    assert S.make_config("gaussian1d", None, dict(levels=4, n0=10)).level_sizes() == [10, 12, 15, 18]


@pytest.mark.parametrize("over,msg", [(dict(m=0), "m must be"), (dict(lam=1.5), "lambda"),
                                      (dict(boundary="neumann0"), "periodic domain"),
                                      (dict(init="warm"), "init must")])
def test_config_validation(over, msg):
    with pytest.raises(S.ConfigError, match=msg):
        S.make_config("planewave2d", None, over)
    with pytest.raises(S.ConfigError, match="set scheme=conservative"):
        S.make_config("conserve1d", None, dict(scheme="dissipative"))


def test_csv_schemas():
    from paper_1802_05246_b200 import ErrorReport

    rep = ErrorReport(ns=np.array([4, 5, 6]), hs=np.array([0.25, 0.2, 1 / 6]), dts=np.array([0.2, 0.16, 0.13]),
                      err_u=np.array([1e-2, 4e-3, 2e-3]))
    lines = S.rates_csv(rep).splitlines()
    assert lines[0] == "level,n,h,dt,error_u,rate"
    assert lines[1].endswith(",") and len(lines) == 4
    assert S.energy_csv([0, 5], [0.0, 0.5], [0.0, 1.5e-12]).splitlines()[0] == "step,time,energy_delta"


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(STUDIES))
def test_study_matches_reference(gold, name):
    exp, over = STUDIES[name]
    res = S.run_experiment(S.make_config(exp, None, over))
    if exp == "conserve1d":
        steps, times, deltas, e0 = res
        np.testing.assert_array_equal(steps, gold[f"{name}/steps"])
        np.testing.assert_allclose(times, gold[f"{name}/times"], rtol=0, atol=1e-12)
        assert e0 == pytest.approx(float(gold[f"{name}/e0"]), rel=1e-12)
        # the invariant holds to rounding on both sides
        assert np.max(np.abs(deltas)) <= 1e-12 * abs(e0)
        return
    np.testing.assert_array_equal(res.ns, gold[f"{name}/ns"])
    np.testing.assert_allclose(res.err_u, gold[f"{name}/err_u"], rtol=1e-9)
    if f"{name}/err_dux" in gold:
        np.testing.assert_allclose(res.err_dux, gold[f"{name}/err_dux"], rtol=1e-9)
        np.testing.assert_allclose(res.err_v, gold[f"{name}/err_v"], rtol=1e-9)
    if f"{name}/rate" in gold:
        assert res.rate() == pytest.approx(float(gold[f"{name}/rate"]), abs=1e-6)
