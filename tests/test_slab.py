"""Multi-GPU slab decomposition (paper_1802_05246_b200/slab.py) on the CPU:
world_size-2 `gloo` ranks run SlabRing's halo exchange and row split with
the kernel replaced by the CPU oracle evaluated on the same source rows
(local rows + the received halo row), and the gathered result must equal a
single-process oracle run on the whole periodic grid.  This pins which row is
sent where at each parity (from PRIMAL the halo is the right
neighbour's first row, from DUAL the left neighbour's last row) and the
interior/edge launch split, without a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hermite_oracle as O

M, NX, NY, STEPS, LAM = 3, 12, 7, 4, 0.9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_kernel(ring, u, v, ud, vd, parity, m, cfg, bc, lo, hi, t_local, nt, stream):
    """Stand-in for the C-ABI launch: the oracle on target rows [t_local, t_local+nt)."""
    off = 0 if parity == O.PRIMAL else -1
    rows_u, rows_v = [], []
    for s_loc in range(t_local + off, t_local + off + nt + 1):
        if 0 <= s_loc < ring.nrows:
            rows_u.append(u[s_loc].numpy())
            rows_v.append(v[s_loc].numpy())
        elif s_loc < 0:
            rows_u.append(lo[0].numpy())
            rows_v.append(lo[1].numpy())
        else:
            rows_u.append(hi[0].numpy())
            rows_v.append(hi[1].numpy())
    wu, wv = np.stack(rows_u), np.stack(rows_v)
    h = ring.grid.hx
    a = O.gather(wu, 0, "x", O.PRIMAL, False, None, None)
    du = np.moveaxis(O.gather(a, 2, "y", parity, True, None, None), 1, 2)
    a = O.gather(wv, 0, "x", O.PRIMAL, False, None, None)
    dv = np.moveaxis(O.gather(a, 2, "y", parity, True, None, None), 1, 2)
    uo, vo = O._step_from_corners(du, dv, h, ring.grid.hy, m, cfg.lam)
    ud[t_local:t_local + nt] = torch.from_numpy(uo)
    vd[t_local:t_local + nt] = torch.from_numpy(vo)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1802_05246_b200 as hb
        from paper_1802_05246_b200.slab import SlabRing

        grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, NX, NY, True)
        ring = SlabRing(grid, rank, world, kernel=_oracle_kernel)
        h = grid.hx
        x = O.nodes(0.0, h, NX, True, O.PRIMAL)
        y = O.nodes(0.0, grid.hy, NY, True, O.PRIMAL)
        u0 = O.planewave_data(x, y, 0.0, M, M, 1, h, grid.hy)
        v0 = O.planewave_data(x, y, 0.0, M - 1, M - 1, 1, h, grid.hy, tder=1)
        sl = slice(ring.row0, ring.row0 + ring.nrows)
        u, v = torch.from_numpy(u0[sl].copy()), torch.from_numpy(v0[sl].copy())
        cfg = hb.SchemeConfig(m=M, lam=LAM)
        par = O.PRIMAL
        for _ in range(STEPS):
            ud, vd = torch.empty_like(u), torch.empty_like(v)
            ring.diss2d_step(u, v, ud, vd, par, M, cfg, hb.BoundarySpec2D())
            u, v, par = ud, vd, O.flip(par)
        gu = [torch.empty_like(u) for _ in range(world)]
        gv = [torch.empty_like(v) for _ in range(world)]
        dist.all_gather(gu, u)
        dist.all_gather(gv, v)
        if rank == 0:
            q.put((torch.cat(gu).numpy(), torch.cat(gv).numpy()))
    finally:
        dist.destroy_process_group()


def test_slab_ring_matches_single_process_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got_u, got_v = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h = 1.0 / NX
    x = O.nodes(0.0, h, NX, True, O.PRIMAL)
    y = O.nodes(0.0, 1.0 / NY, NY, True, O.PRIMAL)
    u = O.planewave_data(x, y, 0.0, M, M, 1, h, 1.0 / NY)
    v = O.planewave_data(x, y, 0.0, M - 1, M - 1, 1, h, 1.0 / NY, tder=1)
    par = O.PRIMAL
    for _ in range(STEPS):
        u, v = O.half_step_2d(u, v, par, NX, NY, True, h, 1.0 / NY, M, LAM)
        par = O.flip(par)
    np.testing.assert_allclose(got_u, u, rtol=0, atol=1e-13 * np.max(np.abs(u)))
    np.testing.assert_allclose(got_v, v, rtol=0, atol=1e-13 * np.max(np.abs(v)))


def test_halo_plan_directions():
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.slab import SlabRing

    g = hb.Grid2D(0.0, 1.0, 0.0, 1.0, 12, 5, True)
    r = SlabRing(g, 1, 3, kernel=lambda *a: None)
    assert r.halo_plan(hb.PRIMAL) == ("hi", 0, 0, 2)       # send first row left, receive from the right
    assert r.halo_plan(hb.DUAL) == ("lo", 3, 2, 0)         # send last row right, receive from the left
    with pytest.raises(ValueError):
        SlabRing(hb.Grid2D(0.0, 1.0, 0.0, 1.0, 10, 5, True), 0, 3)
    with pytest.raises(ValueError):
        SlabRing(hb.Grid2D(0.0, 1.0, 0.0, 1.0, 12, 5, False), 0, 3)
