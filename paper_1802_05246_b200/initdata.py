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


def planewave_on_grid(grid, parity: str, t: float, kx: int, ky: int, kappa: float, tder: int = 0,
                      host: bool = False, device=None):
    """planewave_data at the nodes of `parity` on a Grid2D (x = x_left + h (i + off))."""
    from .fields import DUAL

    off = 0.5 if parity == DUAL else 0.0
    nx, ny = grid.axis(0).n_nodes(parity), grid.axis(1).n_nodes(parity)
    out = _alloc(nx, ny, kx, ky, device)
    L.check(L.lib().hw_init_planewave2d(out.data_ptr(), nx, ny, int(kx), int(ky), float(grid.x_left),
                                        float(grid.y_left), off, float(t), float(kappa), grid.hx, grid.hy,
                                        int(tder), stream_handle(out.device)), "planewave_data")
    return out.cpu().numpy() if host else out


def standing_wave_on_grid(grid, parity: str, t: float, kx: int, ky: int, ax: float, ay: float, om: float,
                          px: float = 0.0, py: float = 0.0, tder: int = 0, host: bool = False, device=None):
    """Scaled blocks of sin(ax x + px) sin(ay y + py) cos(om t) (tder = 1: d/dt)."""
    from .fields import DUAL

    off = 0.5 if parity == DUAL else 0.0
    nx, ny = grid.axis(0).n_nodes(parity), grid.axis(1).n_nodes(parity)
    out = _alloc(nx, ny, kx, ky, device)
    L.check(L.lib().hw_init_standing2d(out.data_ptr(), nx, ny, int(kx), int(ky), float(grid.x_left),
                                       float(grid.y_left), off, float(t), float(ax), float(ay), float(px),
                                       float(py), float(om), grid.hx, grid.hy, int(tder),
                                       stream_handle(out.device)), "standing_wave_data")
    return out.cpu().numpy() if host else out
