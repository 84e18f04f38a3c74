"""The multi-GPU slab path end to end in separate processes: two ranks with a
real torch.distributed process group (gloo: host-staged halo rows, since this
pool gives one GPU per job and NCCL refuses two ranks on one device), each
rank launching the C-ABI kernels on its own rows of cuda:0.
The ranks never wait on each other's kernels: every exchange goes through the
host.  Checked against the one-launch whole-grid path computed by rank 0:

  * C5-style periodic dissipative steps (m = 6): gathered slabs bitwise equal;
  * the L2 error through SlabRing.l2_error's all-reduce;
  * C3's wall grid (m = 5, Dirichlet x / Neumann y): conservative steps in
    place over `previous`, bitwise; and SlabRing.conservative_energy, whose
    2 T b temporary crosses the slab boundary (the in-process test of
    tests/test_gpu_slab.py cannot hand it over).
"""

import math
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather(dist, t):
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, t.cpu())
    return parts


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_1802_05246_b200 as hb
    from paper_1802_05246_b200.slab import SlabRing
    from paper_1802_05246_b200.stepping import cons2d_into, diss2d_into

    res = {}
    # ---- C5-style periodic dissipative steps
    m, n, steps = 6, 48, 4
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, True)
    cfg, bc = hb.SchemeConfig(m=m, lam=0.9), hb.BoundarySpec2D()
    w, om = 2.0 * math.pi, 2.0 * math.pi * math.sqrt(2.0)
    ring = SlabRing(grid, rank, world)
    rows = (ring.row0, ring.nrows(hb.PRIMAL))
    u = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, om, rows=rows)
    v = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, om, tder=1, rows=rows)
    par = hb.PRIMAL
    for _ in range(steps):
        du, dv = torch.empty_like(u), torch.empty_like(v)
        ring.diss2d_step(u, v, du, dv, par, m, cfg, bc)
        u, v, par = du, dv, hb.flip(par)
    torch.cuda.synchronize()
    ex = hb.StandingWave2D(w, w, om, 0.3)
    l2 = ring.l2_error(u, par, (m, m), ex, bc)
    gu, gv = _gather(dist, u), _gather(dist, v)
    if rank == 0:
        wu = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m, m, w, w, om)
        wv = hb.standing_wave_on_grid(grid, hb.PRIMAL, 0.1, m - 1, m - 1, w, w, om, tder=1)
        p = hb.PRIMAL
        for _ in range(steps):
            nu, nv = torch.empty_like(wu), torch.empty_like(wv)
            diss2d_into(wu, wv, nu, nv, grid, p, m, cfg, bc)
            wu, wv, p = nu, nv, hb.flip(p)
        res["diss_u"] = bool(torch.equal(torch.cat(gu), wu.cpu()))
        res["diss_v"] = bool(torch.equal(torch.cat(gv), wv.cpu()))
        whole = hb.l2_error_field_2d(hb.Field2D(grid, p, 0.0, wu), ex, bc)
        res["l2"] = (l2, whole)

    # ---- C3's wall grid: conservative steps, energy
    m, n, steps = 5, 40, 5
    grid = hb.Grid2D(0.0, 1.0, 0.0, 1.0, n, n, False)
    cfg = hb.SchemeConfig(m=m, lam=0.9)
    bc = hb.BoundarySpec2D(hb.BoundarySpec("dirichlet0", "dirichlet0"), hb.BoundarySpec("neumann0", "neumann0"))
    pi, om = math.pi, math.pi * math.sqrt(2.0)
    dt = cfg.dt(grid.hx)
    ring = SlabRing(grid, rank, world)
    par0, p1 = hb.PRIMAL, hb.DUAL
    a = hb.standing_wave_on_grid(grid, par0, 0.0, m, m, pi, pi, om, py=0.5 * pi,
                                 rows=(ring.row0, ring.nrows(par0)))
    b = hb.standing_wave_on_grid(grid, p1, -0.5 * dt, m, m, pi, pi, om, py=0.5 * pi,
                                 rows=(ring.row0, ring.nrows(p1)))
    par = par0
    for _ in range(steps):
        ring.cons2d_step(a, b, b, par, m, cfg, bc)
        a, b, par = b, a, hb.flip(par)
    torch.cuda.synchronize()
    energy = ring.conservative_energy(a, b, par, m, 1.0, dt, bc, "l2")
    ga, gb = _gather(dist, a), _gather(dist, b)
    if rank == 0:
        wa = hb.standing_wave_on_grid(grid, par0, 0.0, m, m, pi, pi, om, py=0.5 * pi)
        wb = hb.standing_wave_on_grid(grid, p1, -0.5 * dt, m, m, pi, pi, om, py=0.5 * pi)
        p = par0
        for _ in range(steps):
            cons2d_into(wa, wb, wb, grid, p, m, cfg, bc)
            wa, wb, p = wb, wa, hb.flip(p)
        res["cons_a"] = bool(torch.equal(torch.cat(ga), wa.cpu()))
        res["cons_b"] = bool(torch.equal(torch.cat(gb), wb.cpu()))
        want = hb.conservative_energy_2d(hb.Field2D(grid, p, 0.0, wa), hb.Field2D(grid, hb.flip(p), 0.0, wb),
                                         1.0, dt, bc, "l2")
        res["energy"] = (energy, want)
        torch.save(res, out)
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_slabs_equal_whole_grid(tmp_path):
    import torch
    import torch.multiprocessing as mp

    out = str(tmp_path / "res.pt")
    mp.start_processes(_worker, args=(WORLD, _free_port(), out), nprocs=WORLD, start_method="spawn", join=True)
    res = torch.load(out)
    assert res["diss_u"] and res["diss_v"]
    assert res["cons_a"] and res["cons_b"]
    l2, whole = res["l2"]
    assert l2 == pytest.approx(whole, rel=1e-13)
    e, want = res["energy"]
    assert e == pytest.approx(want, rel=1e-12)
