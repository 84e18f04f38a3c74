"""Slab decomposition of a periodic 2D grid along x with a one-row halo ring.

SURVEY §8e: each target node depends only on its 2x2 flanking source nodes
(boundary.py:119-130), so a half step is a map over target rows plus ONE
exchange: from PRIMAL data, target row t needs source rows t and t+1 (the
halo is the right neighbour's first row); from DUAL data, rows t-1 and t
(the left neighbour's last row).  Rank r owns rows [r*R, (r+1)*R) of both
parities; the ring closes through the periodic wrap.

The exchange is torch.distributed P2P (NCCL on GPUs, gloo in the CPU tests).
The interior rows are launched before waiting on the halo, so the transfer
overlaps the kernel; the one halo-dependent row follows.
"""

from __future__ import annotations

import ctypes as C

from .fields import DUAL, PRIMAL, Grid2D


class SlabRing:
    def __init__(self, grid: Grid2D, rank: int, world: int, kernel=None):
        if not grid.periodic:
            raise ValueError("slab ring decomposition is implemented for periodic grids")
        if grid.nx % world:
            raise ValueError(f"nx={grid.nx} must divide evenly over {world} ranks")
        self.grid = grid
        self.rank = rank
        self.world = world
        self.nrows = grid.nx // world
        self.row0 = rank * self.nrows
        self.kernel = kernel if kernel is not None else _cabi_kernel
        self.kernel_events = None
        self._halo = {}

    # neighbours on the ring
    @property
    def right(self) -> int:
        return (self.rank + 1) % self.world

    @property
    def left(self) -> int:
        return (self.rank - 1) % self.world

    def local_grid(self, parity: str) -> Grid2D:
        """The slab as a grid of its own (x offset row0*hx), for initial data."""
        g = self.grid
        x0 = g.x_left + g.hx * self.row0
        return Grid2D(x0, x0 + g.hx * self.nrows, g.y_left, g.y_right, self.nrows, g.ny, True)

    def halo_plan(self, parity: str):
        """(which halo, row to send, peer to send to, peer to receive from)."""
        if parity == PRIMAL:
            return "hi", 0, self.left, self.right
        return "lo", self.nrows - 1, self.right, self.left

    def exchange(self, field, parity: str, tag: int = 0):
        """Post the halo exchange for `field` (local rows); returns (buffer, works)."""
        import torch
        import torch.distributed as dist

        side, send_row, to, frm = self.halo_plan(parity)
        key = (side, tuple(field.shape[1:]), field.dtype, str(field.device), tag)
        buf = self._halo.get(key)
        if buf is None:
            buf = torch.empty(field.shape[1:], dtype=field.dtype, device=field.device)
            self._halo[key] = buf
        ops = [dist.P2POp(dist.isend, field[send_row].contiguous(), to),
               dist.P2POp(dist.irecv, buf, frm)]
        return side, buf, dist.batch_isend_irecv(ops)

    def diss2d_step(self, u, v, ud, vd, parity, m, cfg, bc, stream=None):
        """One dissipative half step of this rank's slab (u, v local rows)."""
        ev = self.kernel_events
        if self.world == 1:
            if ev is not None:
                ev[0].record()
            self.kernel(self, u, v, ud, vd, parity, m, cfg, bc, None, None, 0, self.nrows, stream)
            if ev is not None:
                ev[1].record()
            return
        side, hu, wu = self.exchange(u, parity, 0)
        _, hv, wv = self.exchange(v, parity, 1)
        # interior rows do not touch the halo: launch them first
        if side == "hi":
            inner = (0, self.nrows - 1)
            edge = (self.nrows - 1, 1)
        else:
            inner = (1, self.nrows - 1)
            edge = (0, 1)
        if ev is not None:
            ev[0].record()
        self.kernel(self, u, v, ud, vd, parity, m, cfg, bc, None, None, inner[0], inner[1], stream)
        for w in wu + wv:
            w.wait()
        lo = (hu, hv) if side == "lo" else (None, None)
        hi = (hu, hv) if side == "hi" else (None, None)
        self.kernel(self, u, v, ud, vd, parity, m, cfg, bc, lo, hi, edge[0], edge[1], stream)
        if ev is not None:
            ev[1].record()


def _cabi_kernel(ring: SlabRing, u, v, ud, vd, parity, m, cfg, bc, lo, hi, t_local, nt, stream):
    """Launch hw_diss2d_half_step on local target rows [t_local, t_local+nt)."""
    from . import _lib as L
    from .device import ptr
    from .stepping import geom2d

    if nt <= 0:
        return
    g = ring.grid
    geo = geom2d(g, parity, bc, ring.row0 + t_local, nt)
    lo = lo or (None, None)
    hi = hi or (None, None)
    ru = L.Rows2D(ptr(u), ptr(lo[0]) if lo[0] is not None else None, ptr(hi[0]) if hi[0] is not None else None,
                  ring.row0, ring.nrows)
    rv = L.Rows2D(ptr(v), ptr(lo[1]) if lo[1] is not None else None, ptr(hi[1]) if hi[1] is not None else None,
                  ring.row0, ring.nrows)
    dt = cfg.dt(min(g.hx, g.hy))
    cap = -1 if cfg.stage_cap is None else int(cfg.stage_cap)
    row_u = int(u[0].numel())
    row_v = int(v[0].numel())
    L.check(L.lib().hw_diss2d_half_step(C.byref(ru), C.byref(rv), ptr(ud) + 8 * row_u * t_local,
                                        ptr(vd) + 8 * row_v * t_local, int(m), C.byref(geo), dt, g.hx, g.hy,
                                        cfg.speed, cap, stream), "half_step_2d (slab)")


__all__ = ["SlabRing", "DUAL", "PRIMAL"]
