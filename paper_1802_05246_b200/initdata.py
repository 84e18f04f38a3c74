"""Closed-form initial data generated on the device.

planewave_on_grid mirrors driver.py:241-256 planewave_data evaluated at a
grid's nodes (same scaled blocks); standing_wave_on_grid is the synthetic throughput input of SURVEY §8d
(u = sin(ax x + px) sin(ay y + py) cos(om t)).  Both return float64 CUDA
tensors; pass ``host=True`` for numpy.
"""

from __future__ import annotations

from . import _lib as L
from .device import require_cuda, stream_handle


def _alloc(nx, ny, kx, ky, device):
    t = require_cuda()
    dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
    return t.empty((nx, ny, kx + 1, ky + 1), dtype=t.float64, device=dev)


def _window(grid, parity, rows):
    """(first row, row count) of the node rows [row0, row0 + nrows) (all rows if None);
    the kernel places local row i at x_left + hx (row0 + i + off), bit for bit the
    whole grid's coordinate."""
    nx = grid.axis(0).n_nodes(parity)
    if rows is None:
        return 0, nx
    row0, nrows = rows
    if row0 < 0 or nrows < 0 or row0 + nrows > nx:
        raise ValueError("row window out of range")
    return int(row0), int(nrows)


def planewave_on_grid(grid, parity: str, t: float, kx: int, ky: int, kappa: float, tder: int = 0,
                      host: bool = False, device=None, rows=None):
    """planewave_data at the nodes of `parity` on a Grid2D (x = x_left + h (i + off));
    rows = (row0, nrows) restricts to a slab of node rows."""
    from .fields import DUAL

    off = 0.5 if parity == DUAL else 0.0
    row0, nx = _window(grid, parity, rows)
    ny = grid.axis(1).n_nodes(parity)
    out = _alloc(nx, ny, kx, ky, device)
    L.check(L.lib().hw_init_planewave2d(out.data_ptr(), nx, ny, row0, int(kx), int(ky), float(grid.x_left),
                                        float(grid.y_left), off, float(t), float(kappa), grid.hx, grid.hy,
                                        int(tder), stream_handle(out.device)), "planewave_data")
    return out.cpu().numpy() if host else out


def standing_wave_on_grid(grid, parity: str, t: float, kx: int, ky: int, ax: float, ay: float, om: float,
                          px: float = 0.0, py: float = 0.0, tder: int = 0, host: bool = False, device=None,
                          rows=None):
    """Scaled blocks of sin(ax x + px) sin(ay y + py) cos(om t) (tder = 1: d/dt);
    rows = (row0, nrows) restricts to a slab of node rows."""
    from .fields import DUAL

    off = 0.5 if parity == DUAL else 0.0
    row0, nx = _window(grid, parity, rows)
    ny = grid.axis(1).n_nodes(parity)
    out = _alloc(nx, ny, kx, ky, device)
    L.check(L.lib().hw_init_standing2d(out.data_ptr(), nx, ny, row0, int(kx), int(ky), float(grid.x_left),
                                       float(grid.y_left), off, float(t), float(ax), float(ay), float(px),
                                       float(py), float(om), grid.hx, grid.hy, int(tder),
                                       stream_handle(out.device)), "standing_wave_data")
    return out.cpu().numpy() if host else out
