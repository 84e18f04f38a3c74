"""Multi-GPU slab decomposition (paper_1802_05246_b200/slab.py) on the CPU.

world_size-2 and -4 `gloo` ranks run SlabRing's halo exchanges, row split,
interior/edge launch order and all-reduces, with the kernels replaced by an
oracle backend evaluated on the SAME inputs a device launch would see (the
rank's local rows plus the received halo row; wall ghosts built from the
rank's own end row).  The gathered results must equal a single-process
oracle run on the whole grid:

  * periodic dissipative half steps (C2/C5's scheme; the C5 row split with
    m=6 at 4 ranks), several steps of both parities;
  * C3's wall grid (Dirichlet x / Neumann y): conservative full steps from
    both parities and bootstrap — the end slabs build ghosts locally;
  * l2_error_field_2d and the 2D conservative energy, reduced per rank and
    all-reduced.

This pins which row is sent where at each parity (from PRIMAL the
halo is the right neighbour's first row, from DUAL the left neighbour's last
row), the chain ends of wall grids and the extra primal row of the last
rank, without a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import C3_WAVE_BC
from oracle import hermite_oracle as O

LAM = 0.9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bc_tuple(spec):
    return (spec.left, spec.right, spec.left_value, spec.right_value)


class OracleBackend:
    """Stand-in for CabiBackend: the oracle on the rows a launch would read."""

    def reduce_device(self):
        return torch.device("cpu")

    @staticmethod
    def _window(ring, f, halo, parity, t_local, nt, bcx, value_zero=False):
        """Source rows [t0 + off, t0 + off + nt] (global) as the kernel resolves them."""
        off = 0 if parity == O.PRIMAL else -1
        n_src = ring.n_global(parity)
        nloc = ring.nrows(parity)
        rows = []
        for s in range(ring.row0 + t_local + off, ring.row0 + t_local + off + nt + 1):
            li = s - ring.row0
            if 0 <= li < nloc:
                rows.append(f[li].numpy())
            elif li == -1 and halo[0] is not None:
                rows.append(halo[0].numpy())
            elif li == nloc and halo[1] is not None:
                rows.append(halo[1].numpy())
            elif ring.periodic:
                assert ring.world == 1, "a periodic slab must get its halo from the ring"
                rows.append(f[s % n_src].numpy())
            else:  # wall ghost from this rank's own end row (boundary.py:124-130)
                lo = s < 0
                assert (lo and ring.rank == 0) or (not lo and ring.rank == ring.world - 1)
                kind = bcx[0] if lo else bcx[1]
                val = 0.0 if value_zero else (bcx[2] if lo else bcx[3])
                rows.append(O.ghost_2d(f[0 if lo else nloc - 1].numpy(), kind, 0, val))
        return np.stack(rows)

    @staticmethod
    def _corners(win, parity, periodic, bcy, value_zero=False):
        a = O.gather(win, 0, "x", O.PRIMAL, False, None, None)
        vy = (0.0, 0.0) if value_zero else (bcy[2], bcy[3])
        return np.moveaxis(O.gather(a, 2, "y", parity, periodic, bcy[:2], vy), 1, 2)

    def _bcs(self, ring, bc):
        if ring.periodic:
            return O.PERIODIC_BC, O.PERIODIC_BC
        return _bc_tuple(bc.x), _bc_tuple(bc.y)

    def step(self, ring, scheme, srcs, halos, dsts, prev, parity, m, dt, speed, bc, stage_cap, t_local, nt, stream):
        if nt <= 0:
            return
        bx, by = self._bcs(ring, bc)
        g = ring.grid
        vz = [False, scheme in ("diss", "boot")]  # the velocity reflects around 0 (dissipative.py:229)
        d = [self._corners(self._window(ring, f, h, parity, t_local, nt, bx, z), parity, ring.periodic, by, z)
             for f, h, z in zip(srcs, halos, vz)]
        sl = slice(t_local, t_local + nt)
        if scheme == "diss":
            lam = dt * speed / min(g.hx, g.hy)
            uo, vo = O._step_from_corners(d[0], d[1], g.hx, g.hy, m, lam, speed, stage_cap)
            dsts[0][sl] = torch.from_numpy(uo)
            dsts[1][sl] = torch.from_numpy(vo)
        elif scheme == "cons":
            c = O.interp_2d(d[0])
            wt = O.update_tensor_2d(m, 0.5 * speed * dt / g.hx, 0.5 * speed * dt / g.hy)
            new = 2.0 * np.einsum("klab,...ab->...kl", wt, c, optimize=True) - prev[sl].numpy()
            dsts[0][sl] = torch.from_numpy(new)
        else:
            U, _ = O.taylor_2d(O.interp_2d(d[0]), O.interp_2d(d[1]), dt, g.hx, g.hy, speed, 4 * m + 4)
            dsts[0][sl] = torch.from_numpy(np.ascontiguousarray(O.horner(U, 0.5)[..., :m + 1, :m + 1]))

    def _cells(self, ring, f, halo, parity, bc, t_local, nt):
        bx, by = self._bcs(ring, bc)
        return O.interp_2d(self._corners(self._window(ring, f, halo, parity, t_local, nt, bx), parity,
                                         ring.periodic, by))

    def inner(self, ring, f, g, hf, hg, parity, bc, orders, dx, dy, npts, t_local, nt):
        cf = self._cells(ring, f, hf, parity, bc, t_local, nt)
        cg = cf if g is None else self._cells(ring, g, hg, parity, bc, t_local, nt)
        per = O.inner_cells_2d(cf, cg, ring.grid.hx, ring.grid.hy, dx, dy)
        if not ring.periodic and parity == O.DUAL:  # wall-straddling cells count their inner half
            t = np.arange(ring.row0 + t_local, ring.row0 + t_local + nt)
            wx = np.where((t == 0) | (t == ring.n_global(O.PRIMAL) - 1), 0.5, 1.0)
            wy = np.ones(per.shape[1])
            wy[[0, -1]] = 0.5
            per = per * wx[:, None] * wy[None, :]
        return float(np.sum(per))

    def l2(self, ring, f, halo, parity, orders, exact, bc, npts, t_local, nt):
        g = ring.grid
        c = self._cells(ring, f, halo, parity, bc, t_local, nt)
        cx = g.axis(0).nodes(O.flip(parity))[ring.row0 + t_local: ring.row0 + t_local + nt]
        cy = g.axis(1).nodes(O.flip(parity))
        return float(np.sum(O.l2_cells_2d(c, cx, cy, g.hx, g.hy, exact, npts)))


def exact_fn(x, y):
    return np.sin(2.0 * x + 0.3) * np.cos(1.5 * y - 0.2)


def _rand_levels(m, n, periodic, seed, bcs):
    rng = np.random.default_rng(seed)
    nn = lambda p: n if periodic or p == O.DUAL else n + 1  # noqa: E731
    a = rng.standard_normal((nn(O.PRIMAL), nn(O.PRIMAL), m + 1, m + 1))
    b = rng.standard_normal((nn(O.DUAL), nn(O.DUAL), m + 1, m + 1))
    if not periodic:
        a = O.wall_compatible(a, *bcs)
    return a, b


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1802_05246_b200 as hb
        from paper_1802_05246_b200.slab import SlabRing

        kind, m, n, steps = case
        periodic = kind == "diss"
        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, periodic)
        ring = SlabRing(grid, rank, world, backend=OracleBackend())
        cfg = hb.SchemeConfig(m=m, lam=LAM)
        bc = hb.BoundarySpec2D() if periodic else hb.BoundarySpec2D(hb.BoundarySpec(*C3_WAVE_BC[0]),
                                                                   hb.BoundarySpec(*C3_WAVE_BC[1]))
        bcs = None if periodic else C3_WAVE_BC
        out = {}

        def mine(arr, parity):
            return torch.from_numpy(np.array(arr[ring.row0: ring.row0 + ring.nrows(parity)], copy=True))

        def gather(t):
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([t.shape[0]]))
            mx = max(int(s) for s in sizes)
            pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype)
            pad[: t.shape[0]] = t
            parts = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(parts, pad)
            return torch.cat([p[: int(s)] for p, s in zip(parts, sizes)]).numpy()

        if kind == "diss":
            rng = np.random.default_rng(5 + m)
            u = rng.standard_normal((n, n, m + 1, m + 1))
            v = rng.standard_normal((n, n, m, m))
            lu, lv, par = mine(u, O.PRIMAL), mine(v, O.PRIMAL), O.PRIMAL
            for _ in range(steps):
                nu = torch.empty(ring.local_shape(O.flip(par), m, m), dtype=torch.float64)
                nv = torch.empty(ring.local_shape(O.flip(par), m - 1, m - 1), dtype=torch.float64)
                ring.diss2d_step(lu, lv, nu, nv, par, m, cfg, bc)
                lu, lv, par = nu, nv, O.flip(par)
            out["u"], out["v"] = gather(lu), gather(lv)
            out["l2"] = ring.l2_error(lu, par, (m, m), exact_fn, bc)
        else:
            par0 = O.PRIMAL if kind == "cons_primal" else O.DUAL
            a, b = _rand_levels(m, n, periodic, 11 + m, bcs)
            cur, prev = (a, b) if par0 == O.PRIMAL else (b, a)
            lc, lp, par = mine(cur, par0), mine(prev, O.flip(par0)), par0
            dt = cfg.dt(grid.hx)
            out["e0"] = ring.conservative_energy(lc, lp, par, m, 1.0, dt, bc)
            for _ in range(steps):
                ring.cons2d_step(lc, lp, lp, par, m, cfg, bc)  # in place over previous
                lc, lp, par = lp, lc, O.flip(par)
            out["cur"] = gather(lc)
            out["e1"] = ring.conservative_energy(lc, lp, par, m, 1.0, dt, bc)
            out["e1_l2"] = ring.conservative_energy(lc, lp, par, m, 1.0, dt, bc, "l2")
            g1 = np.random.default_rng(3).standard_normal(cur.shape)
            bo = torch.empty(ring.local_shape(O.flip(par0), m, m), dtype=torch.float64)
            ring.boot2d_step(mine(cur, par0), mine(g1, par0), bo, par0, m, cfg, bc)
            out["boot"] = gather(bo)
            out["l2"] = ring.l2_error(mine(cur, par0), par0, (m, m), exact_fn, bc)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = q.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=60)
    for p in procs:
        assert p.exitcode == 0
    return got


def _close(got, want, rtol=1e-13):
    np.testing.assert_allclose(got, want, rtol=0, atol=rtol * np.max(np.abs(want)))


@pytest.mark.parametrize("world,m", [(2, 3), (4, 6)])
def test_slab_dissipative_matches_single_process_oracle(world, m):
    """Periodic dissipative half steps; (4, 6) is C5's scheme and row split."""
    n, steps = 8 * world // 2 if world == 2 else 8, 4
    got = _run(world, ("diss", m, n, steps))
    rng = np.random.default_rng(5 + m)
    u = rng.standard_normal((n, n, m + 1, m + 1))
    v = rng.standard_normal((n, n, m, m))
    h, par = 1.0 / n, O.PRIMAL
    for _ in range(steps):
        u, v = O.half_step_2d(u, v, par, n, n, True, h, h, m, LAM)
        par = O.flip(par)
    tol = {3: 1e-13, 6: 1e-10}[m]  # random high-order data: cond(M_m) amplification
    _close(got["u"], u, tol)
    _close(got["v"], v, tol)
    assert got["l2"] == pytest.approx(O.l2_error_2d(u, par, n, n, True, 0.0, 0.0, h, h, exact_fn), rel=1e-12)


@pytest.mark.parametrize("world,kind", [(2, "cons_primal"), (2, "cons_dual"), (4, "cons_primal")])
def test_slab_c3_walls_match_single_process_oracle(world, kind):
    """C3's wall grid: conservative steps from both parities, bootstrap, the L2
    error and the 2D energy, over ranks whose end slabs build the wall ghosts."""
    m, n, steps = 3, 8, 5
    got = _run(world, (kind, m, n, steps))
    bx, by = C3_WAVE_BC
    a, b = _rand_levels(m, n, False, 11 + m, C3_WAVE_BC)
    par0 = O.PRIMAL if kind == "cons_primal" else O.DUAL
    cur, prev = (a, b) if par0 == O.PRIMAL else (b, a)
    h = 1.0 / n
    dt = LAM * h
    e0 = O.cons_energy_2d(cur, prev, par0, False, h, h, 1.0, dt, bx, by)
    c, p, par = cur, prev, par0
    for _ in range(steps):
        c, p = O.cons_step_2d(c, p, par, False, h, h, m, LAM, 1.0, bx, by), c
        par = O.flip(par)
    _close(got["cur"], c, 1e-12)
    assert got["e0"] == pytest.approx(e0, rel=1e-12)
    assert got["e1"] == pytest.approx(O.cons_energy_2d(c, p, par, False, h, h, 1.0, dt, bx, by), rel=1e-12)
    assert got["e1"] == pytest.approx(e0, rel=1e-11)  # conserved across the slab boundaries too
    assert got["e1_l2"] == pytest.approx(O.cons_energy_2d(c, p, par, False, h, h, 1.0, dt, bx, by, "l2"), rel=1e-12)
    g1 = np.random.default_rng(3).standard_normal(cur.shape)
    _close(got["boot"], O.bootstrap_2d(cur, g1, par0, False, h, h, m, LAM, 1.0, bx, by), 1e-13)
    assert got["l2"] == pytest.approx(O.l2_error_2d(cur, par0, n, n, False, 0.0, 0.0, h, h, exact_fn, None, bx, by),
                                      rel=1e-12)


def test_halo_plan_and_ownership():
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.slab import SlabRing

    g = hb.Grid2D(0.0, 1.0, 0.0, 1.0, 12, 5, True)
    r = SlabRing(g, 1, 3, backend=OracleBackend())
    assert r.halo_plan(hb.PRIMAL) == ("hi", 0, 0, 2)       # send first row left, receive from the right
    assert r.halo_plan(hb.DUAL) == ("lo", 3, 2, 0)         # send last row right, receive from the left
    assert SlabRing(g, 0, 3).halo_plan(hb.DUAL) == ("lo", 3, 1, 2)  # the ring closes through the wrap
    w = hb.Grid2D(0.0, 1.0, 0.0, 1.0, 12, 5, False)
    first, last = SlabRing(w, 0, 3), SlabRing(w, 2, 3)
    assert first.halo_plan(hb.DUAL) == ("lo", 3, 1, None)  # rank 0 builds its wall ghost
    assert last.halo_plan(hb.PRIMAL) == ("hi", 0, 1, None)  # the last rank owns primal row nx
    assert [SlabRing(w, k, 3).nrows(hb.PRIMAL) for k in range(3)] == [4, 4, 5]
    assert [SlabRing(w, k, 3).nrows(hb.DUAL) for k in range(3)] == [4, 4, 4]
    assert SlabRing(g, 0, 1).halo_plan(hb.PRIMAL) == (None, None, None, None)
    with pytest.raises(ValueError):
        SlabRing(hb.Grid2D(0.0, 1.0, 0.0, 1.0, 10, 5, True), 0, 3)
