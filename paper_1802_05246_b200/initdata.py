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


# ---------------------------------------------------------------- 1D closed-form data (driver.py:195-238)

_KIND_1D = {"gaussian": 0, "gaussian_box": 1, "sine": 2}


def _as_device_nodes(x):
    """Node coordinates -> (device tensor, was-host flag, shape)."""
    import numpy as np

    t = require_cuda()
    if hasattr(x, "device") and getattr(x, "is_cuda", False):
        return x.to(t.float64).contiguous(), False, tuple(x.shape)
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return t.from_numpy(a).to("cuda"), True, a.shape


def _columns(x, kmax: int, kind: str, t: float = 0.0, a: float = -20.0, tder: int = 0):
    xd, host, shp = _as_device_nodes(x)
    out = require_cuda().empty(shp + (int(kmax) + 1,), dtype=xd.dtype, device=xd.device)
    if xd.numel() == 0:
        if not 0 <= kmax <= 12:
            raise ValueError(f"{kind}: derivative count out of range (0..12)")
        return out.cpu().numpy() if host else out
    L.check(L.lib().hw_init_1d(out.data_ptr(), xd.data_ptr(), int(xd.numel()), int(kmax), _KIND_1D[kind], 0.0,
                               0.0, 0.0, 0, float(t), float(a), int(tder), stream_handle(xd.device)), kind)
    return out.cpu().numpy() if host else out


def gaussian_derivs(x, kmax: int, a: float = -20.0):
    """Columns d^k/dx^k exp(a x^2), k = 0..kmax (driver.py:203-219), on the device."""
    return _columns(x, kmax, "gaussian", a=a)


def gaussian_box_u(x, t: float, kmax: int):
    """x-derivative columns of (G(x+t) + G(x-t))/2, G = exp(-20 x^2) (driver.py:222-225)."""
    return _columns(x, kmax, "gaussian_box", t=t)


def gaussian_box_v(x, t: float, kmax: int):
    """x-derivative columns of u_t = (G'(x+t) - G'(x-t))/2 (driver.py:228-231)."""
    return _columns(x, kmax, "gaussian_box", t=t, tder=1)


def sine_derivs(x, kmax: int, t: float):
    """x-derivative columns of sin(x) cos(t) (driver.py:234-238)."""
    return _columns(x, kmax, "sine", t=t)


def scale_cols(vals, h: float):
    """Derivative columns d^l u -> scaled data (h^l / l!) d^l u (driver.py:195-200)."""
    import numpy as np

    t = require_cuda()
    host = not (hasattr(vals, "device") and getattr(vals, "is_cuda", False))
    v = t.from_numpy(np.ascontiguousarray(np.asarray(vals, dtype=np.float64))).to("cuda") if host else \
        vals.to(t.float64).contiguous()
    out = t.empty_like(v)
    cols = int(v.shape[-1])
    L.check(L.lib().hw_scale_cols(v.data_ptr(), out.data_ptr(), int(v.numel() // max(cols, 1)), cols, float(h),
                                  stream_handle(v.device)), "scale_cols")
    return out.cpu().numpy() if host else out


def data_on_grid_1d(grid, parity: str, kind: str, kmax: int, t: float = 0.0, a: float = -20.0, tder: int = 0,
                    host: bool = False, device=None):
    """Scaled blocks (h^k/k!) d^k u at the nodes of `parity` of a Grid1D, in one
    kernel (coordinates x_left + h (i + off) computed on the device):
    kind "gaussian" (exp(a x^2)), "gaussian_box" (tder 0: u, 1: u_t) or "sine"
    (sin(x) cos(t)) — driver.py's initial data, _scale_cols applied."""
    from .fields import DUAL

    n = grid.n_nodes(parity)
    out = require_cuda().empty((n, int(kmax) + 1), dtype=require_cuda().float64,
                               device=device if device is not None else "cuda")
    L.check(L.lib().hw_init_1d(out.data_ptr(), None, int(n), int(kmax), _KIND_1D[kind], float(grid.x_left),
                               float(grid.h), 0.5 if parity == DUAL else 0.0, 1, float(t), float(a), int(tder),
                               stream_handle(out.device)), kind)
    return out.cpu().numpy() if host else out
