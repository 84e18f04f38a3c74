"""1D closed-form initial data on the device
against the reference's own values (tests/golden/init1d.npz, made by
tests/golden/make_golden_init1d.py from hermwave.driver:195-238).

The device evaluates the Gaussian derivatives by the Leibniz recurrence
G^(k+1) = 2a (x G^(k) + k G^(k-1)) instead of the reference's polynomial
coefficients + polyval, so the two agree to rounding: per derivative column,
relative to the column's largest magnitude (sin(x + k pi/2) is CUDA's sin of a
shifted argument vs numpy's: a few ulp of the column max).
"""

import math
import os

import numpy as np
import pytest

from oracle import hermite_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "init1d.npz")
GRIDS = [(3, 10, 0.8), (4, 17, 1.0), (6, 12, 0.8)]


@pytest.fixture(scope="module")
def g1():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def _cols_close(got, want, rtol=1e-13):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    scale = np.maximum(np.max(np.abs(want), axis=tuple(range(want.ndim - 1))), 1e-300)
    err = np.max(np.abs(got - want), axis=tuple(range(want.ndim - 1))) / scale
    assert np.all(err <= rtol), err


def test_oracle_sine_and_scaling_match_reference(g1):
    x = g1["pts/x"]
    for k in (0, 1, 4, 8, 12):
        np.testing.assert_array_equal(O.sine_derivs(x, k, 0.8), g1[f"pts/sine/{k}"])
    for m, n, lam in GRIDS:
        h = 2.0 * math.pi / n
        for par in ("primal", "dual"):
            xs = O.nodes(-math.pi, h, n, True, par)
            np.testing.assert_array_equal(O.scale_cols(O.sine_derivs(xs, m, -0.5 * lam * h), h),
                                          g1[f"grid/{m}/{n}/{par}/sine"])


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 4, 8, 12])
def test_device_generators_at_points(g1, k):
    import paper_1802_05246_b200 as hb

    x = g1["pts/x"]
    _cols_close(hb.gaussian_derivs(x, k), g1[f"pts/gauss/{k}"])
    _cols_close(hb.gaussian_derivs(x, k, a=-3.0), g1[f"pts/gauss_a3/{k}"])
    _cols_close(hb.gaussian_box_u(x, 0.37, k), g1[f"pts/box_u/{k}"])
    _cols_close(hb.gaussian_box_v(x, 0.37, k), g1[f"pts/box_v/{k}"])
    _cols_close(hb.sine_derivs(x, k, 0.8), g1[f"pts/sine/{k}"], 1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,lam", GRIDS)
def test_device_scaled_data_on_grids(g1, m, n, lam):
    """The driver experiments' node sets, scaled (the blocks the steppers take)."""
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.initdata import data_on_grid_1d

    g = hb.Grid1D(-1.5, 1.5, n, False)
    dt = lam * g.h
    gp = hb.Grid1D(-math.pi, math.pi, n, True)
    for par in ("primal", "dual"):
        _cols_close(data_on_grid_1d(g, par, "gaussian", m, host=True), g1[f"grid/{m}/{n}/{par}/gauss"])
        _cols_close(data_on_grid_1d(g, par, "gaussian_box", m, t=-0.5 * dt, host=True),
                    g1[f"grid/{m}/{n}/{par}/box_u"])
        _cols_close(data_on_grid_1d(g, par, "gaussian_box", m, t=0.0, tder=1, host=True),
                    g1[f"grid/{m}/{n}/{par}/box_v"])
        _cols_close(data_on_grid_1d(gp, par, "sine", m, t=-0.5 * lam * gp.h, host=True),
                    g1[f"grid/{m}/{n}/{par}/sine"], 1e-14)
        # scale_cols on the device == the reference's _scale_cols of the same columns
        x = g.nodes(par)
        raw = hb.gaussian_derivs(torch.as_tensor(x, device="cuda"), m)
        _cols_close(hb.scale_cols(raw, g.h).cpu().numpy(), g1[f"grid/{m}/{n}/{par}/gauss"])


@pytest.mark.gpu
def test_device_init1d_errors():
    import paper_1802_05246_b200 as hb

    with pytest.raises(ValueError, match="derivative count"):
        hb.gaussian_derivs(np.zeros(3), 13)
    assert hb.sine_derivs(np.zeros(0), 3, 0.0).shape == (0, 4)
