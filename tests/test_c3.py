"""BASELINE config C3 (2D conservative, m=5, Dirichlet x / Neumann y walls,
2048^2) against the reference.

  * CPU: the oracle reproduces the reference's own C3-setup runs
    (tests/golden/c3walls.npz, made by tests/golden/make_golden_c3.py) for
    odd orders 3, 5, 7 from BOTH parities, 6-8 full steps, and bootstrap.
  * GPU: the device path through the C ABI matches the same goldens within
    10x the reference's own 1-ulp sensitivity (per coefficient), and at the
    full 2048^2 size one step from each parity matches oracle windows at the
    four wall corners (where the Dirichlet/Neumann ghosts and the corner
    double reflection act) and in the middle.
"""

import math

import numpy as np
import pytest

from cases import C3_CASES, C3_LAM, C3_RAND_BC, C3_WAVE_BC
from oracle import hermite_oracle as O


@pytest.fixture(scope="module")
def c3g():
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c3walls.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def _bc(kind):
    return C3_WAVE_BC if kind == "wave" else C3_RAND_BC


def _oracle_run(g, name, m, n, par, steps, kind):
    bx, by = _bc(kind)
    h = 1.0 / n
    cur, prev, p = g[f"{name}/cur0"], g[f"{name}/prev0"], par
    for _ in range(steps):
        cur, prev = O.cons_step_2d(cur, prev, p, False, h, h, m, C3_LAM, 1.0, bx, by), cur
        p = O.flip(p)
    return cur


@pytest.mark.parametrize("case", C3_CASES, ids=[c[0] for c in C3_CASES])
def test_oracle_matches_reference_c3(c3g, case):
    name, m, n, par, steps, kind = case
    cur = _oracle_run(c3g, name, m, n, par, steps, kind)
    want = c3g[f"{name}/cur"]
    # the oracle restates the reference op for op: equal to its rounding
    assert np.max(np.abs(cur - want)) <= 1e-14 * np.max(np.abs(want))
    bx, by = _bc(kind)
    b = O.bootstrap_2d(c3g[f"{name}/cur0"], c3g[f"{name}/g1"], par, False, 1.0 / n, 1.0 / n, m, C3_LAM, 1.0, bx, by)
    assert np.max(np.abs(b - c3g[f"{name}/boot"])) <= 1e-14 * np.max(np.abs(c3g[f"{name}/boot"]))


def _within_sigma(got, want, sigma, rel_floor=1e-15):
    """Per coefficient (k, l): max over nodes of |got - want| <= 10 sigma[k, l]
    + rel_floor * max|want|; value coefficients also <= 1e-12 relative."""
    scale = float(np.max(np.abs(want)))
    d = np.abs(got - want).max(axis=(0, 1))
    ok = d <= 10.0 * sigma + rel_floor * scale
    d00 = float(np.max(np.abs(got[..., 0, 0] - want[..., 0, 0])))
    return bool(ok.all()) and d00 <= max(10.0 * float(sigma[0, 0]), 1e-12 * scale), (d / scale, sigma / scale)


@pytest.mark.gpu
@pytest.mark.parametrize("case", C3_CASES, ids=[c[0] for c in C3_CASES])
def test_device_c3_vs_reference(c3g, case):
    import paper_1802_05246_b200 as hb

    name, m, n, par, steps, kind = case
    bx, by = _bc(kind)
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
    bc = hb.BoundarySpec2D(hb.BoundarySpec(*bx), hb.BoundarySpec(*by))
    cfg = hb.SchemeConfig(m=m, lam=C3_LAM)
    dt = cfg.dt(grid.hx)
    st = hb.TwoLevelState(hb.Field2D(grid, par, 0.0, c3g[f"{name}/cur0"]),
                          hb.Field2D(grid, hb.flip(par), -0.5 * dt, c3g[f"{name}/prev0"]))
    for _ in range(steps):
        st = hb.full_step_conservative(st, cfg, bc)
    want = c3g[f"{name}/cur"]
    assert st.current.values.shape == want.shape
    assert st.current.time == float(c3g[f"{name}/t"])
    ok, info = _within_sigma(st.current.values, want, c3g[f"{name}/sigma"])
    assert ok, info
    b = hb.bootstrap_first_half(hb.Field2D(grid, par, 0.0, c3g[f"{name}/cur0"]),
                                hb.Field2D(grid, par, 0.0, c3g[f"{name}/g1"]), cfg, bc)
    ok, info = _within_sigma(b.current.values, c3g[f"{name}/boot"], c3g[f"{name}/boot_sigma"])
    assert ok, info


# ---------------------------------------------------------------- full size (2048^2) windows

def cons_window(cur_w, prev_t, par, lo_wall, hi_wall, h, m, lam, bcx, bcy):
    """Oracle conservative step for the targets of a source window.

    cur_w: source nodes [r0, r1) x [c0, c1) of the current level (parity par);
    lo_wall / hi_wall: (x, y) flags, whether the window starts / ends at the
    physical wall on that axis.  From PRIMAL every target uses two real
    sources; from DUAL the gather pads ghosts on both sides of the window
    (boundary.py:124-130), so targets next to a window edge that is not a
    wall are dropped.  prev_t: the previous level on the kept targets."""
    d = O.corner_data(cur_w, par, False, bcx, bcy)
    if par == O.DUAL:
        sx = slice(0 if lo_wall[0] else 1, None if hi_wall[0] else -1)
        sy = slice(0 if lo_wall[1] else 1, None if hi_wall[1] else -1)
        d = d[sx, sy]
    c = O.interp_2d(d)
    dt = lam * h
    wt = O.update_tensor_2d(m, 0.5 * dt / h, 0.5 * dt / h)
    return 2.0 * np.einsum("klab,...ab->...kl", wt, c, optimize=True) - prev_t


def _windows(n, par, k=8):
    """(source rows, target rows, lo_wall, hi_wall) per axis for a k-target window
    at the low wall, the middle and the high wall."""
    ns = n + 1 if par == O.PRIMAL else n          # source nodes per axis
    out = []
    if par == O.PRIMAL:                            # target t <- sources t, t+1
        for t0 in (0, n // 2 - 3, n - k):
            out.append((np.arange(t0, t0 + k + 1), np.arange(t0, t0 + k), t0 == 0, t0 + k + 1 == ns))
    else:                                          # target t <- sources t-1, t (ghosts at -1, n)
        out.append((np.arange(0, k), np.arange(0, k), True, False))
        t0 = n // 2 - 3
        out.append((np.arange(t0 - 1, t0 + k), np.arange(t0, t0 + k), False, False))
        out.append((np.arange(n - k, n), np.arange(n - k + 1, n + 1), False, True))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("par", ["primal", "dual"])
def test_device_c3_full_size_wall_corners(par):
    """One C3 step at 2048^2 from each parity; 8x8-target oracle windows at the
    four wall corners, the four wall midpoints and the centre agree with the
    oracle within 10x the oracle's own 1-ulp sensitivity on the same window."""
    import torch

    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import cons2d_into

    m, n, lam = 5, 2048, C3_LAM
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
    bx, by = C3_WAVE_BC
    bc = hb.BoundarySpec2D(hb.BoundarySpec(*bx), hb.BoundarySpec(*by))
    cfg = hb.SchemeConfig(m=m, lam=lam)
    dt = cfg.dt(grid.hx)
    pi, om = math.pi, math.pi * math.sqrt(2.0)
    tp = hb.flip(par)
    cur = hb.standing_wave_on_grid(grid, par, 0.0, m, m, pi, pi, om, py=0.5 * pi)
    prev = hb.standing_wave_on_grid(grid, tp, -0.5 * dt, m, m, pi, pi, om, py=0.5 * pi)
    try:
        out = torch.empty_like(prev)
        cons2d_into(cur, prev, out, grid, par, m, cfg, bc)
        torch.cuda.synchronize()
        hb.require_finite(out)
        rng = np.random.default_rng(7)
        wins = _windows(n, par)
        for sr, tr, xlo, xhi in wins:
            for sc, tc, ylo, yhi in wins:
                cw = cur[torch.as_tensor(sr, device="cuda")][:, torch.as_tensor(sc, device="cuda")].cpu().numpy()
                pw = prev[torch.as_tensor(tr, device="cuda")][:, torch.as_tensor(tc, device="cuda")].cpu().numpy()
                got = out[torch.as_tensor(tr, device="cuda")][:, torch.as_tensor(tc, device="cuda")].cpu().numpy()
                want = cons_window(cw, pw, par, (xlo, ylo), (xhi, yhi), grid.hx, m, lam, bx, by)
                cp = cw * (1.0 + 2.2e-16 * rng.standard_normal(cw.shape))
                pp = pw * (1.0 + 2.2e-16 * rng.standard_normal(pw.shape))
                sig = np.abs(cons_window(cp, pp, par, (xlo, ylo), (xhi, yhi), grid.hx, m, lam, bx, by) - want)
                assert got.shape == want.shape
                scale = float(np.max(np.abs(want)))
                assert np.max(np.abs(got - want)) <= 10.0 * np.max(sig) + 1e-15 * scale
                d00 = float(np.max(np.abs(got[..., 0, 0] - want[..., 0, 0])))
                assert d00 <= max(10.0 * float(np.max(sig[..., 0, 0])), 1e-13 * scale)
    finally:
        del cur, prev
        torch.cuda.empty_cache()


def test_window_oracle_matches_whole_grid_oracle():
    """CPU self-check of cons_window: on a 24^2 C3 grid its windows reproduce
    the whole-grid oracle step, from both parities (to BLAS blocking-order
    rounding: einsum sums in a batch-shape dependent order)."""
    m, n, lam = 5, 24, C3_LAM
    bx, by = C3_RAND_BC
    rng = np.random.default_rng(3)
    for par in (O.PRIMAL, O.DUAL):
        tp = O.flip(par)
        ns, nt = (n + 1, n) if par == O.PRIMAL else (n, n + 1)
        cur = rng.standard_normal((ns, ns, m + 1, m + 1))
        prev = rng.standard_normal((nt, nt, m + 1, m + 1))
        full = O.cons_step_2d(cur, prev, par, False, 1.0 / n, 1.0 / n, m, lam, 1.0, bx, by)
        assert full.shape[0] == nt and tp
        for sr, tr, xlo, xhi in _windows(n, par, k=5):
            for sc, tc, ylo, yhi in _windows(n, par, k=5):
                w = cons_window(cur[sr][:, sc], prev[tr][:, tc], par, (xlo, ylo), (xhi, yhi), 1.0 / n, m, lam, bx, by)
                want = full[tr][:, tc]
                np.testing.assert_allclose(w, want, rtol=0, atol=1e-13 * np.max(np.abs(want)))
