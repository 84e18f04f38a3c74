"""The multi-GPU slab path with the real kernel, on one GPU (SURVEY §8e:
"the multi-GPU result must equal the single-GPU result bitwise").

A world of W slab ranks is simulated in one process: each rank's SlabRing
launches the C-ABI kernel on its own rows exactly as under torchrun (interior
rows first, then the halo-dependent edge row with the halo passed as the
Rows2D lo/hi pointer); only the transport is replaced — `exchange` hands over
a copy of the neighbour's row instead of an NCCL send/recv.  No rank's kernel
waits on another's.  The gathered slabs must equal the one-launch whole-grid
step bit for bit, over several half steps of both parities.
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


class _LocalRing:
    """SlabRing with an in-process transport (the peers' current fields)."""

    def __new__(cls, grid, rank, world, peers):
        from paper_1802_05246_b200.slab import SlabRing

        class Ring(SlabRing):
            def exchange(self, field, parity, tag=0):
                side, send_row, to, frm = self.halo_plan(parity)
                return side, peers[frm][tag][send_row].clone(), []

        return Ring(grid, rank, world)


@pytest.mark.parametrize("m,world", [(3, 2), (4, 4), (6, 2)])
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

    # whole grid, one launch per half step
    wu, wv, par = u.clone(), v.clone(), hb.PRIMAL
    for _ in range(steps):
        nu, nv = torch.empty_like(wu), torch.empty_like(wv)
        diss2d_into(wu, wv, nu, nv, grid, par, m, cfg, bc)
        wu, wv, par = nu, nv, hb.flip(par)

    # W slab ranks
    rows = nx // world
    peers = [[u[r * rows:(r + 1) * rows].clone(), v[r * rows:(r + 1) * rows].clone()] for r in range(world)]
    rings = [_LocalRing(grid, r, world, peers) for r in range(world)]
    par = hb.PRIMAL
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(steps):
        outs = []
        for r, ring in enumerate(rings):
            su, sv = peers[r]
            du, dv = torch.empty_like(su), torch.empty_like(sv)
            ring.diss2d_step(su, sv, du, dv, par, m, cfg, bc, stream)
            outs.append([du, dv])
        torch.cuda.synchronize()
        for r in range(world):
            peers[r][:] = outs[r]
        par = hb.flip(par)
    gu = torch.cat([p[0] for p in peers])
    gv = torch.cat([p[1] for p in peers])
    assert torch.equal(gu, wu)
    assert torch.equal(gv, wv)
