"""The multi-GPU slab path with the real kernels, on one GPU (SURVEY §8e:
"the multi-GPU result must equal the single-GPU result bitwise").

A world of W slab ranks is simulated in one process: each rank's SlabRing
launches the C-ABI kernels on its own rows exactly as under torchrun
(interior rows first, then the halo-dependent edge row with the halo passed
as the Rows2D lo/hi pointer; wall ghosts built by the end slabs); only the
transport is replaced — `exchange` hands over a copy of the neighbour's row
(every rank's rows are views of one global tensor) instead of an NCCL
send/recv.  No rank's kernel waits on another's.  The gathered slabs must
equal the one-launch whole-grid step bit for bit, over several steps of both
parities: periodic dissipative (C2/C5) and C3's conservative wall grid plus
bootstrap.  The per-rank partial reductions (hw_l2err2d / hw_inner2d on a
target-row window with halos) must sum to the whole-grid values.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ring(grid, rank, world):
    from paper_1802_05246_b200.slab import SlabRing

    class Ring(SlabRing):
        def exchange(self, fields, parity_src, tag=0):
            side, _, _, frm = self.halo_plan(parity_src)
            if side is None:
                return None, [None] * len(fields), []
            r = self.row0 - 1 if side == "lo" else self.row0 + self.nrows(parity_src)
            bufs = [None if frm is None else f._base[r % f._base.shape[0]].clone() for f in fields]
            return side, bufs, []

        def _allreduce(self, vals):  # partials are summed by the test
            return list(vals)

    return Ring(grid, rank, world)


def _views(g, rings, parity):
    return [g[r.row0: r.row0 + r.nrows(parity)] for r in rings]


@pytest.mark.parametrize("m,world", [(1, 4), (2, 2), (3, 2), (4, 4), (6, 2), (6, 4)])
def test_slab_ranks_equal_whole_grid_bitwise(m, world):
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import diss2d_into

    nx, ny, steps = 64, 40, 4
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, nx, ny, True)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D()
    w = 2.0 * math.pi
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, w * math.sqrt(2.0), tder=1)
    g = torch.Generator(device="cpu").manual_seed(7 + m)
    u = u + 1e-3 * torch.randn(u.shape, generator=g, dtype=torch.float64).to(u.device)
    v = v + 1e-3 * torch.randn(v.shape, generator=g, dtype=torch.float64).to(v.device)
    # slab init: the row window of the init kernel equals the whole grid's rows bitwise
    rings = [_ring(grid, r, world) for r in range(world)]
    r1 = rings[-1]
    w0 = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0))
    ws = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, w * math.sqrt(2.0),
                                  rows=(r1.row0, r1.nrows(hb.PRIMAL)))
    assert torch.equal(ws, w0[r1.row0:])

    wu, wv, par = u.clone(), v.clone(), hb.PRIMAL
    for _ in range(steps):
        nu, nv = torch.empty_like(wu), torch.empty_like(wv)
        diss2d_into(wu, wv, nu, nv, grid, par, m, cfg, bc)
        wu, wv, par = nu, nv, hb.flip(par)

    su, sv, par = u.clone(), v.clone(), hb.PRIMAL
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(steps):
        du, dv = torch.empty_like(su), torch.empty_like(sv)
        for ring, a, b, c, d in zip(rings, _views(su, rings, par), _views(sv, rings, par),
                                    _views(du, rings, hb.flip(par)), _views(dv, rings, hb.flip(par))):
            ring.diss2d_step(a, b, c, d, par, m, cfg, bc, stream)
        su, sv, par = du, dv, hb.flip(par)
    torch.cuda.synchronize()
    assert torch.equal(su, wu)
    assert torch.equal(sv, wv)
    # the L2 error reduced per rank (one halo row each) sums to the whole grid's
    ex = hb.StandingWave2D(w, w, w * math.sqrt(2.0), 0.3)
    whole = hb.l2_error_field_2d(hb.Field2D(grid, par, 0.0, su), ex, bc)
    parts = [ring.l2_error(f, par, (m, m), ex, bc) ** 2 for ring, f in zip(rings, _views(su, rings, par))]
    assert math.sqrt(sum(parts)) == pytest.approx(whole, rel=1e-13)


@pytest.mark.parametrize("m,world,par0", [(5, 2, "primal"), (5, 4, "dual"), (3, 4, "primal")])
def test_slab_c3_walls_equal_whole_grid_bitwise(m, world, par0):
    """C3's wall grid: conservative steps in place over `previous`, both
    parities; the end slabs build the Dirichlet / Neumann ghosts; bootstrap;
    the 2D energy's inner products reduced per rank."""
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.stepping import cons2d_into, geom2d, rows2d  # noqa: F401

    n, steps = 32, 5
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0"), hb.BoundarySpec("neumann0", "neumann0"))
    pi, om = math.pi, math.pi * math.sqrt(2.0)
    dt = cfg.dt(grid.hx)
    p1 = hb.flip(par0)
    a = hb.standing_wave_on_grid(grid, par0, 0.0, m, m, pi, pi, om, py=0.5 * pi)
    b = hb.standing_wave_on_grid(grid, p1, -0.5 * dt, m, m, pi, pi, om, py=0.5 * pi)
    rings = [_ring(grid, r, world) for r in range(world)]
    assert sum(r.nrows(hb.PRIMAL) for r in rings) == n + 1

    wa, wb, par = a.clone(), b.clone(), par0
    for _ in range(steps):
        cons2d_into(wa, wb, wb, grid, par, m, cfg, bc)
        wa, wb, par = wb, wa, hb.flip(par)

    sa, sb, par = a.clone(), b.clone(), par0
    for _ in range(steps):
        for ring, c, p in zip(rings, _views(sa, rings, par), _views(sb, rings, hb.flip(par))):
            ring.cons2d_step(c, p, p, par, m, cfg, bc)
        sa, sb, par = sb, sa, hb.flip(par)
    torch.cuda.synchronize()
    assert torch.equal(sa, wa) and torch.equal(sb, wb)

    # bootstrap from the initial level
    g1 = hb.standing_wave_on_grid(grid, par0, 0.0, m, m, pi, pi, om, py=0.5 * pi, tder=1)
    whole = hb.bootstrap_first_half(hb.Field2D(grid, par0, 0.0, a), hb.Field2D(grid, par0, 0.0, g1), cfg, bc)
    out = torch.empty_like(b)
    for ring, x, y, o in zip(rings, _views(a, rings, par0), _views(g1, rings, par0), _views(out, rings, p1)):
        ring.boot2d_step(x, y, o, par0, m, cfg, bc)
    torch.cuda.synchronize()
    assert torch.equal(out, whole.current.values)

    # the 2D energy's per-rank partials sum to the whole-grid energy
    for sem in ("l2", "mixed"):
        want = hb.conservative_energy_2d(hb.Field2D(grid, par, 0.0, sa), hb.Field2D(grid, hb.flip(par), 0.0, sb),
                                         1.0, dt, bc, sem)
        got = 0.0
        for ring in rings:
            got += _energy_partial(ring, sa, sb, par, m, dt, bc, sem)
        assert got == pytest.approx(want, rel=1e-12 if sem == "l2" else 1e-10)


def _energy_partial(ring, a, b, pa, m, dt, bc, sem):
    """SlabRing.conservative_energy's per-rank part with the whole-grid 2 T b
    (the in-process transport cannot hand over a neighbour's temporary)."""
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.slab import _SEMINORMS
    from paper_1802_05246_b200.stepping import cons2d_into  # noqa: F401

    grid = ring.grid
    pb = hb.flip(pa)
    tb2 = torch.zeros_like(a)
    from paper_1802_05246_b200 import _lib as L
    from paper_1802_05246_b200.device import ptr, stream_handle
    from paper_1802_05246_b200.stepping import geom2d, rows2d
    import ctypes as C

    L.check(L.lib().hw_cons2d_step(C.byref(rows2d(b)), ptr(tb2), ptr(tb2), int(m), C.byref(geom2d(grid, pb, bc)),
                                   float(dt), grid.hx, grid.hy, 1.0, stream_handle(a.device)), "T b")
    va, vt = a[ring.row0: ring.row0 + ring.nrows(pa)], tb2[ring.row0: ring.row0 + ring.nrows(pa)]
    vb = b[ring.row0: ring.row0 + ring.nrows(pb)]
    ha, t0a, nta = ring._cells([va, vt], pa)
    hb_, t0b, ntb = ring._cells([vb], pb)
    tot = 0.0
    for dx, dy in _SEMINORMS[sem](m):
        npts = 2 * m + 2 - min(dx, dy)
        tot += ring.backend.inner(ring, va, None, ha[0], None, pa, bc, (m, m), dx, dy, npts, t0a, nta)
        tot += ring.backend.inner(ring, vb, None, hb_[0], None, pb, bc, (m, m), dx, dy, npts, t0b, ntb)
        tot -= ring.backend.inner(ring, va, vt, ha[0], ha[1], pa, bc, (m, m), dx, dy, npts, t0a, nta)
    return 2.0 * tot
