"""CUDA path (through the C ABI) vs the reference's golden vectors and vs the
pinned CPU oracle.  Requires a B200.

Tolerances (FP64).  The kernels sum in a different order
than the reference's BLAS einsum + stage recursion, so parity is measured
against the reference's own rounding sensitivity:
  * value coefficients (u_00, v_00): max|d| / max|ref| <= VALUE_TOL[m]
  * all coefficients: max|d| / max|ref| <= ALL_TOL[m]  (high-order scaled
    coefficients of random data are amplified by cond(M_mu) up to 1e7)
"""

import math

import numpy as np
import pytest

import paper_1802_05246_b200 as hb
from cases import CASES_1D, CASES_2D, X1D, X2D, exact2d, forcing_fn
from oracle import hermite_oracle as O

pytestmark = pytest.mark.gpu

VALUE_TOL = {1: 1e-13, 2: 1e-13, 3: 1e-13, 4: 1e-13, 5: 1e-12, 6: 1e-12, 7: 1e-11, 8: 1e-11, 12: 1e-9}
ALL_TOL = {1: 1e-13, 2: 1e-13, 3: 1e-12, 4: 1e-12, 5: 1e-11, 6: 1e-10, 7: 1e-9, 8: 1e-8, 12: 1e-5}


def rel(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-300))


def value_rel(got, want):
    return rel(got[..., 0, 0] if got.ndim == 4 else got[..., 0], want[..., 0, 0] if want.ndim == 4 else want[..., 0])


def spec2d(bcx, bcy):
    if bcx is None:
        return hb.BoundarySpec2D()
    return hb.BoundarySpec2D(hb.BoundarySpec(*bcx), hb.BoundarySpec(*bcy))


@pytest.mark.parametrize("case", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_half_step_2d_vs_reference(golden, case):
    name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps = case
    grid = hb.Grid2D(*X2D, nx, ny, per)
    cfg = hb.SchemeConfig(m=m, speed=c, lam=lam, stage_cap=cap)
    bc = spec2d(bcx, bcy)
    pair = hb.FieldPair(hb.Field2D(grid, par, 0.0, golden[f"d2/{name}/u0"]),
                        hb.Field2D(grid, par, 0.0, golden[f"d2/{name}/v0"]))
    for _ in range(steps):
        pair = hb.half_step_2d(pair, cfg, bc)
    assert isinstance(pair.u.values, np.ndarray)
    wu, wv = golden[f"d2/{name}/u"], golden[f"d2/{name}/v"]
    assert pair.u.values.shape == wu.shape and pair.v.values.shape == wv.shape
    assert pair.time == float(golden[f"d2/{name}/t"])
    tv = VALUE_TOL[m] * (10 if steps > 1 else 1)
    ta = ALL_TOL[m] * (10 if steps > 1 else 1)
    assert value_rel(pair.u.values, wu) <= tv
    assert value_rel(pair.v.values, wv) <= tv
    assert rel(pair.u.values, wu) <= ta
    assert rel(pair.v.values, wv) <= ta


@pytest.mark.parametrize("case", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_conservative_2d_vs_reference(golden, case):
    name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps = case
    grid = hb.Grid2D(*X2D, nx, ny, per)
    cfg = hb.SchemeConfig(m=m, speed=c, lam=lam, stage_cap=cap)
    bc = spec2d(bcx, bcy)
    st = hb.TwoLevelState(hb.Field2D(grid, par, 0.0, golden[f"c2/{name}/cur0"]),
                          hb.Field2D(grid, hb.flip(par), -0.1, golden[f"c2/{name}/prev0"]))
    for _ in range(steps):
        st = hb.full_step_conservative(st, cfg, bc)
    tol = ALL_TOL[m] * (10 if steps > 1 else 1)
    assert rel(st.current.values, golden[f"c2/{name}/cur"]) <= tol
    assert np.array_equal(st.previous.values, golden[f"c2/{name}/prev"]) or steps > 1
    assert st.current.time == float(golden[f"c2/{name}/t"])
    b = hb.bootstrap_first_half(hb.Field2D(grid, par, 0.0, golden[f"c2/{name}/cur0"]),
                                hb.Field2D(grid, par, 0.0, golden[f"b2/{name}/g1"]), cfg, bc)
    assert rel(b.current.values, golden[f"b2/{name}/out"]) <= ALL_TOL[m]
    assert b.current.parity == hb.flip(par)


@pytest.mark.parametrize("case", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_l2_error_2d_vs_reference(golden, case):
    name, m, nx, ny, per, par, bcx, bcy, lam, c, cap, steps = case
    grid = hb.Grid2D(*X2D, nx, ny, per)
    bc = spec2d(bcx, bcy)
    for fld in ("u", "v"):
        f = hb.Field2D(grid, par, 0.0, golden[f"d2/{name}/{fld}0"])
        got = hb.l2_error_field_2d(f, exact2d, bc)
        assert abs(got - float(golden[f"e2/{name}/{fld}"])) <= 1e-12 * float(golden[f"e2/{name}/{fld}"])


@pytest.mark.parametrize("case", CASES_1D, ids=[c[0] for c in CASES_1D])
def test_1d_vs_reference(golden, case):
    name, m, n, per, par, bcs, lam, c, cap, steps, forced = case
    grid = hb.Grid1D(*X1D, n, per)
    bc = hb.BoundarySpec() if bcs is None else hb.BoundarySpec(*bcs)
    cfg = hb.SchemeConfig(m=m, speed=c, lam=lam, stage_cap=cap)
    pair = hb.FieldPair(hb.Field1D(grid, par, 0.0, golden[f"d1/{name}/u0"]),
                        hb.Field1D(grid, par, 0.0, golden[f"d1/{name}/v0"]))
    for _ in range(steps):
        pair = hb.half_step_1d(pair, cfg, bc, forcing=forcing_fn if forced else None)
    tol = ALL_TOL[m] * (10 if steps > 1 else 1)
    assert rel(pair.u.values, golden[f"d1/{name}/u"]) <= tol
    assert rel(pair.v.values, golden[f"d1/{name}/v"]) <= tol
    assert pair.time == float(golden[f"d1/{name}/t"])
    if forced:
        return
    st = hb.TwoLevelState(hb.Field1D(grid, par, 0.0, golden[f"c1/{name}/cur0"]),
                          hb.Field1D(grid, hb.flip(par), -0.1, golden[f"c1/{name}/prev0"]))
    for _ in range(steps):
        st = hb.full_step_conservative(st, cfg, bc)
    assert rel(st.current.values, golden[f"c1/{name}/cur"]) <= tol
    b = hb.bootstrap_first_half(hb.Field1D(grid, par, 0.0, golden[f"c1/{name}/cur0"]),
                                hb.Field1D(grid, par, 0.0, golden[f"b1/{name}/g1"]), cfg, bc)
    assert rel(b.current.values, golden[f"b1/{name}/out"]) <= ALL_TOL[m]
    u0 = hb.Field1D(grid, par, 0.0, golden[f"d1/{name}/u0"])
    v0 = hb.Field1D(grid, par, 0.0, golden[f"d1/{name}/v0"])
    errs = hb.l2_errors_pair(hb.FieldPair(u0, v0), np.sin, np.cos, lambda x: -np.sin(2 * x), bc)
    np.testing.assert_allclose(errs, golden[f"e1/{name}/pair"], rtol=1e-12)
    assert abs(hb.l2_error_field(u0, np.sin, bc) - float(golden[f"e1/{name}/field"])) <= \
        1e-12 * float(golden[f"e1/{name}/field"])


@pytest.mark.parametrize("m,n,nhalf", [(2, 48, 64), (4, 64, 32), (6, 32, 32), (8, 24, 16)])
def test_planewave_multistep_vs_oracle(m, n, nhalf):
    """Config-2 style run (periodic plane wave, lam 0.9) against the oracle."""
    lam = 0.9
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    h = grid.hx
    xp = grid.axis(0).nodes(hb.PRIMAL)
    u0 = O.planewave_data(xp, xp, 0.0, m, m, 1, h, h)
    v0 = O.planewave_data(xp, xp, 0.0, m - 1, m - 1, 1, h, h, tder=1)
    cfg = hb.SchemeConfig(m=m, lam=lam)
    out = hb.advance_2d(hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, u0),
                                     hb.Field2D(grid, hb.PRIMAL, 0.0, v0)), cfg, hb.BoundarySpec2D(), nhalf)
    u, v, p = u0, v0, hb.PRIMAL
    for _ in range(nhalf):
        u, v = O.half_step_2d(u, v, p, n, n, True, h, h, m, lam)
        p = O.flip(p)
    noise = {2: 1e-14, 4: 1e-13, 6: 5e-12, 8: 5e-11}[m]  # ~10x the reference's 1-ulp sensitivity
    assert value_rel(out.u.values, u) <= max(1e-12, noise)
    assert value_rel(out.v.values, v) <= max(1e-12, noise)


def test_device_resident_path_keeps_tensors():
    import torch

    m, n = 4, 40
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    u0 = hb.planewave_on_grid(grid, hb.PRIMAL, 0.0, m, m, 1)
    v0 = hb.planewave_on_grid(grid, hb.PRIMAL, 0.0, m - 1, m - 1, 1, tder=1)
    assert isinstance(u0, torch.Tensor) and u0.is_cuda
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    pair = hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, u0), hb.Field2D(grid, hb.PRIMAL, 0.0, v0))
    a = hb.half_step_2d(pair, cfg, hb.BoundarySpec2D())
    assert isinstance(a.u.values, torch.Tensor) and a.u.values.is_cuda
    b = hb.half_step_2d(hb.FieldPair(hb.Field2D(grid, hb.PRIMAL, 0.0, u0.cpu().numpy()),
                                     hb.Field2D(grid, hb.PRIMAL, 0.0, v0.cpu().numpy())), cfg, hb.BoundarySpec2D())
    assert np.array_equal(a.u.values.cpu().numpy(), b.u.values)
    # device init equals the reference's planewave_data to rounding
    h = grid.hx
    xp = grid.axis(0).nodes(hb.PRIMAL)
    assert rel(u0.cpu().numpy(), O.planewave_data(xp, xp, 0.0, m, m, 1, h, h)) <= 1e-14


def test_finite_check():
    a = np.zeros((5, 5, 3, 3))
    hb.require_finite(a)
    a[2, 3, 1, 1] = np.nan
    with pytest.raises(hb.NumericalError):
        hb.require_finite(a)


def test_builtin_exact_matches_callable():
    m, n = 3, 12
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    h = grid.hx
    xp = grid.axis(0).nodes(hb.PRIMAL)
    u0 = O.planewave_data(xp, xp, 0.1, m, m, 2, h, h)
    f = hb.Field2D(grid, hb.PRIMAL, 0.0, u0)
    pw = hb.PlaneWave2D(kappa=2, t=0.2)
    e_dev = hb.l2_error_field_2d(f, pw, hb.BoundarySpec2D())
    e_host = hb.l2_error_field_2d(f, lambda x, y: pw(x, y), hb.BoundarySpec2D())
    e_ref = O.l2_error_2d(u0, hb.PRIMAL, n, n, True, 0.0, 0.0, h, h, pw)
    assert abs(e_dev - e_ref) <= 1e-12 * e_ref
    assert abs(e_host - e_ref) <= 1e-12 * e_ref
    assert math.isfinite(e_dev)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("per,par", [(True, hb.PRIMAL), (True, hb.DUAL), (False, hb.PRIMAL), (False, hb.DUAL)])
def test_host_pipelined_path_equals_device_path(per, par, pinned):
    """numpy in/out of >= 64 rows goes through the chunked, copy-overlapped path
    (stepping._diss2d_host_pipelined; pageable inputs through pinned staging,
    pinned ones straight); every cell's arithmetic is the same, so it must
    equal the device-resident path bit for bit."""
    import torch

    m, nx, ny = 3, 150, 37
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.3, nx, ny, per)
    bc = hb.BoundarySpec2D() if per else hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "neumann0", 0.2, 0.0),
                                                           hb.BoundarySpec("neumann0", "dirichlet0", 0.0, -0.3))
    rng = np.random.default_rng(11)
    shp = (grid.axis(0).n_nodes(par), grid.axis(1).n_nodes(par))
    u0 = rng.standard_normal(shp + (m + 1, m + 1))
    v0 = rng.standard_normal(shp + (m, m))
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    uh, vh = (torch.from_numpy(u0).pin_memory().numpy(), torch.from_numpy(v0).pin_memory().numpy()) if pinned \
        else (u0, v0)
    a = hb.half_step_2d(hb.FieldPair(hb.Field2D(grid, par, 0.0, uh), hb.Field2D(grid, par, 0.0, vh)), cfg, bc)
    b = hb.half_step_2d(hb.FieldPair(hb.Field2D(grid, par, 0.0, torch.from_numpy(u0).cuda()),
                                     hb.Field2D(grid, par, 0.0, torch.from_numpy(v0).cuda())), cfg, bc)
    assert isinstance(a.u.values, np.ndarray) and a.time == b.time and a.parity == b.parity
    assert np.array_equal(a.u.values, b.u.values.cpu().numpy())
    assert np.array_equal(a.v.values, b.v.values.cpu().numpy())


@pytest.mark.parametrize("m", [3, 5])
def test_unaligned_field_bases_equal_aligned(m):
    """Fields whose records have even length are staged with 16-byte copies
    when their base is 16-byte aligned; a view starting one double into its
    storage must take the 8-byte path and give the same bits."""
    import torch

    from paper_1802_05246_b200.stepping import diss2d_into

    n = 64
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    g = torch.Generator().manual_seed(m)
    u = torch.randn((n, n, m + 1, m + 1), generator=g, dtype=torch.float64).cuda()
    v = torch.randn((n, n, m, m), generator=g, dtype=torch.float64).cuda()

    def shifted(x):  # same values, base address 8 bytes past a 16-byte boundary
        buf = torch.empty(x.numel() + 1, dtype=x.dtype, device=x.device)
        y = buf[1:].view(x.shape)
        y.copy_(x)
        assert y.data_ptr() % 16 == 8
        return y

    outs = []
    for uu, vv in ((u, v), (shifted(u), shifted(v))):
        ud, vd = torch.empty_like(u), torch.empty_like(v)
        diss2d_into(uu, vv, ud, vd, grid, hb.PRIMAL, m, cfg, hb.BoundarySpec2D())
        outs.append((ud, vd))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
