"""The lower-level batched API (lowlevel.py, csrc/lowlevel.cuh) against the
reference's own outputs (tests/golden/lowlevel.npz from
tests/golden/make_golden_lowlevel.py).  Element-wise functions (Taylor
recursions, Horner, ghosts, gathers) are bit-identical; the contractions
(interpolation, conservative update) agree to rounding — numpy routes them
through BLAS in its own summation order."""

import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lowlevel.npz")


@pytest.fixture(scope="module")
def g():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def close(got, want, rel=1e-14):
    scale = max(float(np.max(np.abs(want))), 1e-300)
    assert got.shape == want.shape
    assert float(np.max(np.abs(got - want))) <= rel * scale


@pytest.mark.parametrize("m", [1, 3, 6])
def test_pascal_table_matches_reference(g, m):
    """A host table, as in the reference (conservative.py:59-75)."""
    import paper_1802_05246_b200 as hb

    pt = hb.pascal_table(m, 0.31, 0.27)
    assert np.array_equal(pt.base, g[f"pt/{m}/base"])
    assert np.array_equal(pt.scaled, g[f"pt/{m}/scaled"])


@pytest.mark.gpu
def test_apply_interp(g):
    import paper_1802_05246_b200 as hb

    for mu in (0, 2, 5):
        close(hb.apply_interp(g[f"ai1/{mu}/in"]), g[f"ai1/{mu}/out"])
    for mm in ("11", "32", "44"):
        close(hb.apply_interp_2d(g[f"ai2/{mm}/in"]), g[f"ai2/{mm}/out"])


@pytest.mark.gpu
def test_expand_taylor_bitwise(g):
    import paper_1802_05246_b200 as hb

    def forcing(l, s, x, t):  # tests/golden/make_golden_lowlevel.py
        return np.cos(0.7 * x + 0.3 * t) * (l + 1.0) / (s + 2.0)

    for name, smax, f in (("a", 6, None), ("b", 9, forcing)):
        tu, tv = hb.expand_taylor(g[f"et1/{name}/cu"], g[f"et1/{name}/cv"], 0.037, 0.05, 1.3, smax, f,
                                  g[f"et1/{name}/centers"], 0.21)
        assert np.array_equal(tu, g[f"et1/{name}/tu"]) and np.array_equal(tv, g[f"et1/{name}/tv"])
    for name, smax in (("a", 10), ("b", 14)):
        d1 = g.get(f"et2/{name}/d1")
        ct, dt = hb.expand_taylor_2d(g[f"et2/{name}/c0"], g[f"et2/{name}/d0"], 0.02, 0.05, 0.07, 1.1, smax, d1)
        assert np.array_equal(ct, g[f"et2/{name}/ct"]) and np.array_equal(dt, g[f"et2/{name}/dt"])


@pytest.mark.gpu
def test_eval_series_bitwise(g):
    import paper_1802_05246_b200 as hb

    assert np.array_equal(hb.eval_series(g["es/in"], 0.5), g["es/out"])
    assert np.array_equal(hb.eval_series(g["es/in"], 0.7), g["es/out07"])


@pytest.mark.gpu
@pytest.mark.parametrize("m", [1, 3, 6])
def test_conservative_updates(g, m):
    import paper_1802_05246_b200 as hb

    cfg = hb.SchemeConfig(m=m, lam=0.8, speed=1.2)
    close(hb.conservative_update_1d(g[f"cu1/{m}/c"], g[f"cu1/{m}/p"], cfg, 0.05), g[f"cu1/{m}/out"])
    close(hb.conservative_update_2d(g[f"cu2/{m}/c"], g[f"cu2/{m}/p"], cfg, 0.05, 0.07), g[f"cu2/{m}/out"], 1e-13)


@pytest.mark.gpu
def test_ghosts_bitwise(g):
    import paper_1802_05246_b200 as hb

    for kind in ("dirichlet0", "neumann0"):
        assert np.array_equal(hb.ghost_data(g["g1/in"], kind, 0.7 if kind == "dirichlet0" else 0.0), g[f"g1/{kind}"])
        for ax in (0, 1):
            got = hb.ghost_data_2d(g["g2/in"], kind, ax, -0.4 if kind == "dirichlet0" else 0.0)
            assert np.array_equal(got, g[f"g2/{kind}/{ax}"])
    with pytest.raises(ValueError):
        hb.ghost_data(g["g1/in"], "periodic")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["per_p", "per_d", "wall_p", "wall_d"])
def test_gathers_bitwise(g, name):
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.lowlevel import corner_sources, pair_sources

    par = hb.PRIMAL if name.endswith("_p") else hb.DUAL
    per = name.startswith("per")
    g1 = hb.Grid1D(-0.2, 1.1, 7, per)
    spec = hb.BoundarySpec() if per else hb.BoundarySpec("dirichlet0", "neumann0", 0.3, 0.0)
    f1 = hb.Field1D(g1, par, 0.0, g[f"ps/{name}/in"])
    d, cen = pair_sources(f1, spec)
    assert np.array_equal(d, g[f"ps/{name}/out"]) and np.array_equal(cen, g[f"ps/{name}/cen"])
    g2 = hb.Grid2D(-0.2, 1.1, 0.1, 0.9, 5, 4, per)
    spec2 = hb.BoundarySpec2D() if per else hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "neumann0", 0.5, 0.0),
                                                              hb.BoundarySpec("neumann0", "dirichlet0", 0.0, -0.25))
    f2 = hb.Field2D(g2, par, 0.0, g[f"cs/{name}/in"])
    d, cx, cy = corner_sources(f2, spec2)
    assert np.array_equal(d, g[f"cs/{name}/out"])
    assert np.array_equal(cx, g[f"cs/{name}/cx"]) and np.array_equal(cy, g[f"cs/{name}/cy"])
    if name == "wall_d":  # the velocity override: reflect around zero
        assert np.array_equal(pair_sources(f1, spec, (0.0, 0.0))[0], g["ps/wall_d/out_zero"])
        assert np.array_equal(corner_sources(f2, spec2, (0.0, 0.0))[0], g["cs/wall_d/out_zero"])


@pytest.mark.gpu
def test_device_tensors_stay_on_device(g):
    import torch

    import paper_1802_05246_b200 as hb

    x = torch.from_numpy(g["es/in"]).cuda()
    out = hb.eval_series(x, 0.5)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert np.array_equal(out.cpu().numpy(), g["es/out"])
