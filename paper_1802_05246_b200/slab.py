"""Slab decomposition of a 2D grid along x with one-row halos.

Each target node depends only on its 2x2 flanking source nodes
(boundary.py:119-130), so a half step is a map over target rows plus ONE
exchange: from PRIMAL data target row t needs source rows t and t+1 (the halo
is the right neighbour's first row); from DUAL data rows t-1 and t (the left
neighbour's last row).  Rank r owns rows [r R, (r+1) R) of both parities,
R = nx / world; on a wall grid the primal parity has one row more (nx + 1,
grid.py:48-51), owned by the last rank.  Periodic grids close the ring through
the wrap; on wall grids the end slabs have no neighbour on the wall side and
the kernel builds the wall ghosts locally (boundary.py:124-130), exactly as
on one device.

The exchange is torch.distributed P2P (NCCL on GPUs, gloo in the CPU tests),
posted before the interior rows are launched so the transfer overlaps the
kernel; the one halo-dependent row follows.  Every scheme the drop-in steps
has a slab form — dissipative half steps, conservative full steps (only the
current level needs a halo; `previous` is element-wise, conservative.py:127),
bootstrap — and the diagnostics reduce per rank then all-reduce one or three
doubles: l2_error_field_2d (diagnostics.py:118-135) and the 2D conservative
energy (norms.conservative_energy_2d).

The kernels are reached through a backend object (default: the C ABI of
libhermb200.so); the CPU tests substitute the oracle to pin the row
ownership, halo directions and reductions without a GPU.
"""

from __future__ import annotations

import ctypes as C
import math

from .fields import DUAL, PRIMAL, Grid2D, flip

_SEMINORMS = {"mixed": lambda m: [(m + 1, m + 1)], "l2": lambda m: [(0, 0)], "h1": lambda m: [(1, 0), (0, 1)]}


class SlabRing:
    def __init__(self, grid: Grid2D, rank: int, world: int, backend=None):
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"rank {rank} out of range for world {world}")
        if grid.nx % world:
            raise ValueError(f"nx={grid.nx} must divide evenly over {world} ranks")
        self.grid = grid
        self.rank = rank
        self.world = world
        self.periodic = grid.periodic
        self.R = grid.nx // world
        self.row0 = rank * self.R
        self.backend = backend if backend is not None else CabiBackend()
        self.kernel_events = None
        self._halo = {}

    # ------------------------------------------------------------ ownership
    def nrows(self, parity: str) -> int:
        """Local rows of `parity` (the last rank of a wall grid owns primal row nx)."""
        extra = (not self.periodic) and parity == PRIMAL and self.rank == self.world - 1
        return self.R + (1 if extra else 0)

    def n_global(self, parity: str) -> int:
        return self.grid.axis(0).n_nodes(parity)

    @property
    def right(self):
        if self.rank + 1 < self.world:
            return self.rank + 1
        return 0 if self.periodic else None

    @property
    def left(self):
        if self.rank > 0:
            return self.rank - 1
        return self.world - 1 if self.periodic else None

    def local_shape(self, parity: str, kx: int, ky: int):
        return (self.nrows(parity), self.grid.axis(1).n_nodes(parity), kx + 1, ky + 1)

    def halo_plan(self, parity_src: str):
        """(side, row to send, send-to rank, receive-from rank) of a step from
        `parity_src` data; ranks are None where a wall ends the chain, and a
        single periodic rank wraps inside its own rows (no exchange)."""
        if self.world == 1:
            return None, None, None, None
        if parity_src == PRIMAL:
            # targets t <- sources t, t+1: the right neighbour's first row
            return "hi", 0, self.left, self.right
        return "lo", self.nrows(DUAL) - 1, self.right, self.left

    # ------------------------------------------------------------ transport
    def exchange(self, fields, parity_src: str, tag: int = 0):
        """Post the halo exchange of `fields` (local rows of parity_src).
        Returns (side, [halo buffer or None per field], works)."""
        import torch
        import torch.distributed as dist

        side, send_row, to, frm = self.halo_plan(parity_src)
        if side is None:
            return None, [None] * len(fields), []
        # gloo moves host tensors only: CUDA rows are staged through host memory
        # there (the multi-process GPU test); NCCL sends device rows directly
        staged = dist.get_backend() == "gloo" and any(f.is_cuda for f in fields)
        ops, bufs, landed = [], [], []
        for k, f in enumerate(fields):
            buf = None
            if frm is not None:
                key = (side, tuple(f.shape[1:]), f.dtype, str(f.device), tag + k)
                buf = self._halo.get(key)
                if buf is None:
                    buf = torch.empty(f.shape[1:], dtype=f.dtype, device=f.device)
                    self._halo[key] = buf
                if staged:
                    hbuf = torch.empty(buf.shape, dtype=buf.dtype)
                    landed.append((hbuf, buf))
                    ops.append(dist.P2POp(dist.irecv, hbuf, frm))
                else:
                    ops.append(dist.P2POp(dist.irecv, buf, frm))
            if to is not None:
                row = f[send_row].contiguous()
                ops.append(dist.P2POp(dist.isend, row.cpu() if staged else row, to))
            bufs.append(buf)
        works = dist.batch_isend_irecv(ops) if ops else []
        if staged and works:
            works = [_StagedRecv(works, landed)]
        return side, bufs, works

    def _halos(self, side, bufs):
        return [(b, None) if side == "lo" else (None, b) for b in bufs]

    # ------------------------------------------------------------ steps
    def _step(self, scheme, srcs, dsts, parity, m, dt, speed, bc, prev=None, stage_cap=None, stream=None):
        ev = self.kernel_events
        nt = self.nrows(flip(parity))
        side, bufs, works = self.exchange(srcs, parity)
        none = [(None, None)] * len(srcs)
        if ev is not None:
            ev[0].record()
        if side is None or bufs[0] is None:
            # no neighbour on the halo side (single rank, or a wall ends the chain)
            for w in works:
                w.wait()
            self.backend.step(self, scheme, srcs, none, dsts, prev, parity, m, dt, speed, bc, stage_cap, 0, nt,
                              stream)
        else:
            # interior rows do not touch the halo: launch them first
            inner, edge = ((0, nt - 1), (nt - 1, 1)) if side == "hi" else ((1, nt - 1), (0, 1))
            if inner[1] > 0:
                self.backend.step(self, scheme, srcs, none, dsts, prev, parity, m, dt, speed, bc, stage_cap,
                                  inner[0], inner[1], stream)
            for w in works:
                w.wait()
            self.backend.step(self, scheme, srcs, self._halos(side, bufs), dsts, prev, parity, m, dt, speed, bc,
                              stage_cap, edge[0], edge[1], stream)
        if ev is not None:
            ev[1].record()

    def diss2d_step(self, u, v, ud, vd, parity, m, cfg, bc, stream=None):
        """One dissipative half step of this rank's slab (dissipative.py:215-247)."""
        self._step("diss", [u, v], [ud, vd], parity, m, cfg.dt(min(self.grid.hx, self.grid.hy)), cfg.speed, bc,
                   stage_cap=cfg.stage_cap, stream=stream)

    def cons2d_step(self, cur, prev, out, parity_cur, m, cfg, bc, stream=None):
        """One conservative full step (conservative.py:139-157); out may alias prev."""
        self._step("cons", [cur], [out], parity_cur, m, cfg.dt(min(self.grid.hx, self.grid.hy)), cfg.speed, bc,
                   prev=prev, stream=stream)

    def boot2d_step(self, g0, g1, out, parity, m, cfg, bc, stream=None):
        """bootstrap_first_half (conservative.py:166-195) of this rank's slab."""
        self._step("boot", [g0, g1], [out], parity, m, cfg.dt(min(self.grid.hx, self.grid.hy)), cfg.speed, bc,
                   stream=stream)

    # ------------------------------------------------------------ reductions
    def _allreduce(self, vals):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return list(vals)
        dev = self.backend.reduce_device() if dist.get_backend() != "gloo" else "cpu"
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        return [float(x) for x in t.cpu()]

    def _cells(self, fields, parity):
        """Exchange the halos the cells of `parity`'s corner gather need;
        returns the per-field (lo, hi) halos and this rank's cell rows."""
        side, bufs, works = self.exchange(fields, parity, tag=100)
        for w in works:
            w.wait()
        halos = self._halos(side, bufs) if side is not None else [(None, None)] * len(fields)
        return halos, 0, self.nrows(flip(parity))

    def l2_error(self, f, parity, orders, exact, bc, npts=None):
        """l2_error_field_2d (diagnostics.py:118-135) of the distributed field:
        per-rank Gauss sums over its cells, one all-reduce, sqrt."""
        npts = npts or 2 * max(orders) + 2
        halos, t0, nt = self._cells([f], parity)
        part = self.backend.l2(self, f, halos[0], parity, orders, exact, bc, npts, t0, nt)
        return math.sqrt(self._allreduce([part])[0])

    def conservative_energy(self, cur, prev, parity_cur, m, speed, dt, bc, seminorm="mixed"):
        """norms.conservative_energy_2d of the distributed two-level state:
        2 T b by a slab step, three inner products per rank, one all-reduce."""
        import torch

        pa, pb = parity_cur, flip(parity_cur)
        tb2 = torch.zeros_like(cur)
        self._step("cons", [prev], [tb2], pb, m, dt, speed, bc, prev=tb2)
        ha, ta0, nta = self._cells([cur, tb2], pa)
        hb, tb0, ntb = self._cells([prev], pb)
        parts = [0.0, 0.0, 0.0]
        for dx, dy in _SEMINORMS[seminorm](m):
            npts = 2 * m + 2 - min(dx, dy)
            parts[0] += self.backend.inner(self, cur, None, ha[0], None, pa, bc, (m, m), dx, dy, npts, ta0, nta)
            parts[1] += self.backend.inner(self, prev, None, hb[0], None, pb, bc, (m, m), dx, dy, npts, tb0, ntb)
            parts[2] += self.backend.inner(self, cur, tb2, ha[0], ha[1], pa, bc, (m, m), dx, dy, npts, ta0, nta)
        ia, ib, iab = self._allreduce(parts)
        return 2.0 * (ia + ib - iab)


class _StagedRecv:
    """gloo receives of device halos: wait, then copy the host rows to their
    device buffers (on the current stream, ahead of the edge-row launch)."""

    def __init__(self, works, landed):
        self.works, self.landed = works, landed

    def wait(self):
        for w in self.works:
            w.wait()
        for host, dev in self.landed:
            dev.copy_(host, non_blocking=False)


class CabiBackend:
    """The slab kernels through include/hermb200.h (libhermb200.so)."""

    def reduce_device(self):
        import torch

        return torch.device("cuda", torch.cuda.current_device())

    @staticmethod
    def _rows(ring, t, parity, halo):
        from . import _lib as L
        from .device import ptr

        lo, hi = halo
        return L.Rows2D(ptr(t), ptr(lo) if lo is not None else None, ptr(hi) if hi is not None else None,
                        ring.row0, ring.nrows(parity))

    def step(self, ring, scheme, srcs, halos, dsts, prev, parity, m, dt, speed, bc, stage_cap, t_local, nt,
             stream):
        from . import _lib as L
        from .device import ptr, stream_handle
        from .stepping import geom2d

        if nt <= 0:
            return
        g = ring.grid
        s = stream if stream is not None else stream_handle(srcs[0].device)
        geo = geom2d(g, parity, bc, ring.row0 + t_local, nt)
        rows = [self._rows(ring, f, parity, h) for f, h in zip(srcs, halos)]
        off = [ptr(d) + 8 * int(d[0].numel()) * t_local for d in dsts]
        if scheme == "diss":
            cap = -1 if stage_cap is None else int(stage_cap)
            L.check(L.lib().hw_diss2d_half_step(C.byref(rows[0]), C.byref(rows[1]), off[0], off[1], int(m),
                                                C.byref(geo), dt, g.hx, g.hy, speed, cap, s), "half_step_2d (slab)")
        elif scheme == "cons":
            pv = ptr(prev) + 8 * int(prev[0].numel()) * t_local
            L.check(L.lib().hw_cons2d_step(C.byref(rows[0]), pv, off[0], int(m), C.byref(geo), dt, g.hx, g.hy,
                                           speed, s), "full_step_conservative (slab)")
        else:
            L.check(L.lib().hw_boot2d(C.byref(rows[0]), C.byref(rows[1]), off[0], int(m), C.byref(geo), dt, g.hx,
                                      g.hy, speed, s), "bootstrap_first_half (slab)")

    def inner(self, ring, f, g, hf, hg, parity, bc, orders, dx, dy, npts, t_local, nt):
        from .device import stream_handle
        from .norms import _inner2d

        class _St:
            stream = stream_handle(f.device)

        rf = self._rows(ring, f, parity, hf)
        rg = self._rows(ring, g, parity, hg) if g is not None else None
        return _inner2d(f, g, ring.grid, parity, bc, orders, dx, dy, npts, _St, trow0=ring.row0 + t_local,
                        ntrows=nt, rows_f=rf, rows_g=rg)

    def l2(self, ring, f, halo, parity, orders, exact, bc, npts, t_local, nt):
        from .norms import _l2_sum_2d

        return _l2_sum_2d(f, ring.grid, parity, orders, exact, bc, npts, ring.row0 + t_local, nt,
                          self._rows(ring, f, parity, halo))


__all__ = ["SlabRing", "CabiBackend", "DUAL", "PRIMAL"]
