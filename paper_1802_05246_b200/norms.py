"""Error norms and rate fitting (drop-in for the L2 parts of hermwave.diagnostics).

The per-cell interpolation, Gauss evaluation and the reduction run on the
device (csrc/diag.cuh).  What stays on the host is geometry only: Gauss rules,
piece clipping and — for a user-supplied Python ``exact`` callable — its
evaluation at the quadrature points, exactly as the reference evaluates it
(diagnostics.py:66-85,118-135).  Built-in closed forms (``PlaneWave2D``,
``StandingWave2D``) are evaluated inside the kernel.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .config import BoundarySpec, BoundarySpec2D, check_periodicity
from .device import Staging, ptr
from .fields import DUAL, PRIMAL, Field1D, Field2D, FieldPair, flip
from .stepping import _PARITY, geom2d, rows2d


def gauss_rule(npts: int):
    """Gauss-Legendre nodes/weights on [-1, 1] (diagnostics.py:33-35)."""
    return np.polynomial.legendre.leggauss(npts)


def default_npts(m: int) -> int:
    """diagnostics.py:38-40."""
    return 2 * m + 2


@dataclass(frozen=True)
class PlaneWave2D:
    """u = sin(w (x + y + sqrt(2) t)), w = 2 pi kappa (driver.py:381,393-394)."""

    kappa: float
    t: float

    def __call__(self, x, y):
        w = 2.0 * np.pi * self.kappa
        return np.sin(w * (x + y + math.sqrt(2.0) * self.t))

    @property
    def device_form(self):
        return 1, (2.0 * np.pi * self.kappa, self.t, 0.0, 0.0)


@dataclass(frozen=True)
class StandingWave2D:
    """u = sin(ax x) sin(ay y) cos(om t) (SURVEY §8d throughput data)."""

    ax: float
    ay: float
    om: float
    t: float

    def __call__(self, x, y):
        return np.sin(self.ax * x) * np.sin(self.ay * y) * math.cos(self.om * self.t)

    @property
    def device_form(self):
        return 2, (self.ax, self.ay, self.om, self.t)


def _l2_sum_2d(f, grid, parity: str, orders, exact, bc: BoundarySpec2D, npts: int, trow0: int = 0,
               ntrows: int = -1, rows=None) -> float:
    """sum over the cells [trow0, trow0 + ntrows) of the field's corner gather of
    (hx hy / 4) sum_pq w_p w_q (I f - exact)^2 (hw_l2err2d; the square of
    diagnostics.py:118-135's result when the window is the whole grid)."""
    mx, my = orders
    g = geom2d(grid, parity, bc, trow0, ntrows)
    xg, wg = gauss_rule(npts)
    params = (C.c_double * 4)(0.0, 0.0, 0.0, 0.0)
    ex_dev = None
    form = getattr(exact, "device_form", None)
    st = Staging(f)
    if form is not None:
        kind, prm = form
        for i, p in enumerate(prm):
            params[i] = float(p)
    else:
        kind = 0
        cx = grid.axis(0).nodes(flip(parity))
        cx = cx[trow0: (len(cx) if ntrows < 0 else trow0 + ntrows)]
        cy = grid.axis(1).nodes(flip(parity))
        x = cx[:, None] + 0.5 * grid.hx * xg[None, :]
        y = cy[:, None] + 0.5 * grid.hy * xg[None, :]
        ex = np.broadcast_to(exact(x[:, None, :, None], y[None, :, None, :]),
                             (len(cx), len(cy), npts, npts))
        ex_dev = st.to_dev(np.ascontiguousarray(ex))
    gx = np.ascontiguousarray(xg, dtype=np.float64)
    gw = np.ascontiguousarray(wg, dtype=np.float64)
    out = C.c_double(0.0)
    r = rows if rows is not None else rows2d(f)
    L.check(L.lib().hw_l2err2d(C.byref(r), int(mx), int(my), C.byref(g), float(grid.x_left),
                               float(grid.y_left), grid.hx, grid.hy, int(npts), gx.ctypes.data_as(C.c_void_p),
                               gw.ctypes.data_as(C.c_void_p), int(kind),
                               ptr(ex_dev) if ex_dev is not None else None, params, C.byref(out), st.stream),
            "l2_error_field_2d")
    return out.value


def l2_error_field_2d(field: Field2D, exact, bc: BoundarySpec2D, npts: int | None = None) -> float:
    """L2 error of the global tensor interpolant (diagnostics.py:118-135).

    Like the reference, cells are the targets of the field's own corner
    gather (no clipping in 2D)."""
    mx, my = field.orders
    npts = npts or default_npts(max(mx, my))
    st = Staging(field.values)
    f = st.to_dev(field.values)
    return math.sqrt(_l2_sum_2d(f, field.grid, field.parity, (mx, my), exact, bc, npts))


def _pieces_1d(field: Field1D):
    """Target centres and breakpoints of the global interpolant (diagnostics.py:47-59)."""
    grid = field.grid
    centers = grid.nodes(flip(field.parity))
    h = grid.h
    bp = np.concatenate([centers - 0.5 * h, centers[-1:] + 0.5 * h])
    return centers, bp, h


def _domain_clip(field):
    if field.grid.periodic:
        return None
    return field.grid.x_left, field.grid.x_right


def _quadrature_1d(field: Field1D, exact, npts: int, clip):
    """Per-piece scaled abscissae, weights and exact values (diagnostics.py:74-85)."""
    centers, bp, h = _pieces_1d(field)
    xg, wg = gauss_rule(npts)
    n = len(centers)
    xi = np.zeros((n, npts))
    w = np.zeros((n, npts))
    ex = np.zeros((n, npts))
    for i in range(n):
        a, b = bp[i], bp[i + 1]
        if clip is not None:
            a, b = max(a, clip[0]), min(b, clip[1])
            if b <= a:
                continue
        x = 0.5 * (a + b) + 0.5 * (b - a) * xg
        xi[i] = (x - centers[i]) / h
        w[i] = 0.5 * (b - a) * wg
        ex[i] = exact(x)
    return xi, w, ex


def _l2_1d(field: Field1D, bc: BoundarySpec, quad, deriv: int, st: Staging) -> float:
    grid = field.grid
    check_periodicity(bc, grid.periodic)
    xi, w, ex = quad
    npts = xi.shape[1]
    f = st.to_dev(field.values)
    dxi, dw, dex = st.to_dev(xi), st.to_dev(w), st.to_dev(ex)
    abc = L.axis_bc(bc)
    out = C.c_double(0.0)
    L.check(L.lib().hw_l2err1d(ptr(f), int(field.order), grid.n_nodes(field.parity), _PARITY[field.parity],
                               C.byref(abc), grid.h, int(deriv), int(npts), ptr(dxi), ptr(dw), ptr(dex),
                               C.byref(out), st.stream), "l2_error")
    return math.sqrt(max(out.value, 0.0))


def l2_error_field(field: Field1D, exact, bc: BoundarySpec, npts: int | None = None) -> float:
    """diagnostics.py:96-100."""
    npts = npts or default_npts(field.order)
    st = Staging(field.values)
    quad = _quadrature_1d(field, exact, npts, _domain_clip(field))
    return _l2_1d(field, bc, quad, 0, st)


def l2_errors_pair(pair: FieldPair, exact_u, exact_dux, exact_v, bc: BoundarySpec,
                   npts: int | None = None):
    """(u, u_x, v) errors of a dissipative state (diagnostics.py:103-115)."""
    m = pair.u.order
    npts = npts or default_npts(m)
    clip = _domain_clip(pair.u)
    st = Staging(pair.u.values, pair.v.values)
    qu = _quadrature_1d(pair.u, exact_u, npts, clip)
    qd = _quadrature_1d(pair.u, exact_dux, npts, clip)
    qv = _quadrature_1d(pair.v, exact_v, npts, clip)
    return (_l2_1d(pair.u, bc, qu, 0, st), _l2_1d(pair.u, bc, qd, 1, st), _l2_1d(pair.v, bc, qv, 0, st))


# ---------------------------------------------------------------- energies (1D)

def _seminorm_sq(field: Field1D, bc: BoundarySpec, order: int, scale: float, st: Staging) -> float:
    """scale * |I field|^2_order on the field's own pieces (diagnostics.py:201-212)."""
    grid = field.grid
    check_periodicity(bc, grid.periodic)
    nd = 2 * field.order + 2 - order  # coefficients of the order-th derivative
    if nd <= 0:
        return 0.0
    xg, wg = gauss_rule(nd)  # seminorm_sq integrates with deg + 1 points
    gx = np.ascontiguousarray(xg, dtype=np.float64)
    gw = np.ascontiguousarray(wg, dtype=np.float64)
    f = st.to_dev(field.values)
    abc = L.axis_bc(bc)
    out = C.c_double(0.0)
    L.check(L.lib().hw_seminorm1d(ptr(f), int(field.order), grid.n_nodes(field.parity), _PARITY[field.parity],
                                  C.byref(abc), grid.h, int(order), float(scale), int(nd),
                                  gx.ctypes.data_as(C.c_void_p), gw.ctypes.data_as(C.c_void_p), C.byref(out),
                                  st.stream), "seminorm_sq")
    return out.value


def dissipative_energy(state: FieldPair, speed: float, bc: BoundarySpec) -> float:
    """c^2 |I_m u|_{m+1}^2 + |I_{m-1} v|_m^2 (diagnostics.py:229-234), on the device."""
    m = state.u.order
    st = Staging(state.u.values, state.v.values)
    return (_seminorm_sq(state.u, bc, m + 1, speed * speed, st) + _seminorm_sq(state.v, bc, m, 1.0, st))


def _seminorm_sq_2d(field: Field2D, dx: int, dy: int, npts: int, st) -> float:
    grid = field.grid
    mx, my = field.orders
    g = geom2d(grid, field.parity, BoundarySpec2D())
    xg, wg = gauss_rule(npts)
    gx = np.ascontiguousarray(xg, dtype=np.float64)
    gw = np.ascontiguousarray(wg, dtype=np.float64)
    f = st.to_dev(field.values)
    out = C.c_double(0.0)
    L.check(L.lib().hw_seminorm2d(C.byref(rows2d(f)), int(mx), int(my), C.byref(g), grid.hx, grid.hy, int(dx),
                                  int(dy), int(npts), gx.ctypes.data_as(C.c_void_p), gw.ctypes.data_as(C.c_void_p),
                                  C.byref(out), st.stream), "dissipative_energy_2d")
    return out.value


def dissipative_energy_2d(state: FieldPair, speed: float) -> float:
    """A defined 2D energy of a dissipative state (the
    reference has none — diagnostics.py:220-234 and the paper's proof are 1D):

        E = c^2 (|d_x^{m+1} I u|^2 + |d_y^{m+1} I u|^2) + |d_x^m I v|^2 + |d_y^m I v|^2,

    I = the tensor Hermite interpolants I_{m,m} u and I_{m-1,m-1} v on every
    cell of the field's periodic grid, |.|^2 the L2 norm over the domain,
    integrated exactly (Gauss, 2m + 2 points per axis).  On y-independent data
    it is L_y times the 1D dissipative_energy (diagnostics.py:229-234) of the
    x-profile — the reduction the tests pin it by."""
    grid = state.u.grid
    if not grid.periodic:
        raise ValueError("the 2D energy is defined on periodic grids")
    m = state.u.orders[0]
    if state.u.orders != (m, m) or state.v.orders != (m - 1, m - 1):
        raise ValueError(f"pair carries orders {state.u.orders} / {state.v.orders}, want (m, m) / (m-1, m-1)")
    npts = 2 * m + 2
    st = Staging(state.u.values, state.v.values)
    eu = _seminorm_sq_2d(state.u, m + 1, 0, npts, st) + _seminorm_sq_2d(state.u, 0, m + 1, npts, st)
    ev = _seminorm_sq_2d(state.v, m, 0, npts, st) + _seminorm_sq_2d(state.v, 0, m, npts, st)
    return speed * speed * eu + ev


def conservative_energy(current: Field1D, previous: Field1D, speed: float, dt: float, bc: BoundarySpec) -> float:
    """E(t_n) = |P+|^2_{m+1} + |P-|^2_{m+1} of a two-level state (diagnostics.py:190-226).

    P± = p^n - S± p^{n-1/2}, S± w(x) = w(x ± c dt/2), integrated exactly on the
    union pieces; periodic grids only, like the reference."""
    grid = current.grid
    check_periodicity(bc, grid.periodic)
    if not (grid.periodic and previous.grid.periodic):
        raise ValueError("conserved variables need a periodic domain")
    if current.parity == previous.parity:
        raise ValueError("the two levels must sit on opposite parities")
    m = current.order
    if previous.order != m:
        raise ValueError(f"levels carry orders {m} and {previous.order}")
    delta = 0.5 * speed * dt
    if abs(delta) >= grid.h:  # poly.py:223-224
        raise ValueError("shift distance must be smaller than the smallest cell")
    xg, wg = gauss_rule(m + 1)
    gx = np.ascontiguousarray(xg, dtype=np.float64)
    gw = np.ascontiguousarray(wg, dtype=np.float64)
    st = Staging(current.values, previous.values)
    c = st.to_dev(current.values)
    p = st.to_dev(previous.values)
    out = C.c_double(0.0)
    L.check(L.lib().hw_cons_energy1d(ptr(c), ptr(p), int(m), grid.n_nodes(current.parity), _PARITY[current.parity],
                                     grid.h, abs(delta), int(m + 1), gx.ctypes.data_as(C.c_void_p),
                                     gw.ctypes.data_as(C.c_void_p), C.byref(out), st.stream), "conservative_energy")
    return out.value


def _inner2d(f, g, grid, parity: str, bc: BoundarySpec2D, orders, dx: int, dy: int, npts: int, st,
             trow0: int = 0, ntrows: int = -1, rows_f=None, rows_g=None) -> float:
    """hw_inner2d: sum_cells w_cell int int (D I f)(D I g) over the field's cells
    (wall cells counted over their physical half; slabs pass row windows)."""
    xg, wg = gauss_rule(npts)
    gx = np.ascontiguousarray(xg, dtype=np.float64)
    gw = np.ascontiguousarray(wg, dtype=np.float64)
    geo = geom2d(grid, parity, bc, trow0, ntrows)
    rf = rows_f if rows_f is not None else rows2d(f)
    rg = None if g is None else (rows_g if rows_g is not None else rows2d(g))
    out = C.c_double(0.0)
    L.check(L.lib().hw_inner2d(C.byref(rf), C.byref(rg) if rg is not None else None, int(orders[0]), int(orders[1]),
                               C.byref(geo), grid.hx, grid.hy, int(dx), int(dy), int(npts),
                               gx.ctypes.data_as(C.c_void_p), gw.ctypes.data_as(C.c_void_p), 1, C.byref(out),
                               st.stream), "conservative_energy_2d")
    return out.value


_SEMINORMS = {"mixed": lambda m: [(m + 1, m + 1)], "l2": lambda m: [(0, 0)], "h1": lambda m: [(1, 0), (0, 1)]}


def conservative_energy_2d(current: Field2D, previous: Field2D, speed: float, dt: float,
                           bc: BoundarySpec2D, seminorm: str = "mixed") -> float:
    """A defined 2D energy of a conservative two-level state (
    the reference's conservative_energy, diagnostics.py:190-226, is 1D and
    periodic only, and the paper proves conservation in 1D only).

    The reference's E = |P+|^2 + |P-|^2 (P± = I a - S± I b, a = current,
    b = previous) equals 2 (|I a|^2 + |I b|^2 - <I a, I (2 T b)>), where
    2 T b is the scheme's own update of b with a zero previous level
    (conservative.py:115-136): Hermite interpolation is an orthogonal
    projection in the (m+1) seminorm, so the shifted pieces can be replaced by
    the update (oracle.cons_energy_1d_adjoint reproduces the reference's values
    to 1e-14, tests/test_energy.py).  In 2D the same form is taken in the mixed
    seminorm |d_x^{m+1} d_y^{m+1} .|, in which the tensor interpolant is an
    orthogonal projection and the wave cosine C(c dt/2) (what the update tensor
    applies within a cell, c dt/2 <= h/2) is self-adjoint, so
    full_step_conservative conserves

        E2 = 2 (|I a|^2 + |I b|^2 - <I a, I (2 T b)>)

    exactly in exact arithmetic.  Wall grids (Dirichlet / Neumann, C3): the
    ghosts are the odd / even reflections (boundary.py:56-98), so the integral
    runs over the physical domain, wall-straddling (ghost-padded) cells
    counting their inner half; conservation then holds for BC-compatible data
    (primal wall nodes carrying the reflection symmetry, which the scheme
    itself produces and exact initial data satisfy; Dirichlet values equal on
    walls that meet at a corner).  Inner products are exact Gauss quadrature
    summed in double-double on the device.

    seminorm: "mixed" (default) is the exactly conserved form above.  Its
    (m+1)-th derivatives of the interpolant are below round-off once h^(m+1)
    falls under eps * cond(M_m) (e.g. C3's m=5 at 2048^2), where it measures
    rounding noise; "l2" and "h1" take the same adjoint form in |.|_0 and
    |grad .|_0: the exact wave conserves them (per Fourier mode E = 2 sin^2(omega
    c dt / 2) (|alpha|^2 + |beta|^2)), the scheme up to its projection error
    (O(h^(2m+2)) for smooth data) — the physical energy check at full size."""
    if not (isinstance(current, Field2D) and isinstance(previous, Field2D)):
        raise ValueError("conservative_energy_2d takes 2D fields")
    if seminorm not in _SEMINORMS:
        raise ValueError(f"unknown seminorm {seminorm!r} (mixed, l2, h1)")
    grid = current.grid
    if previous.grid != grid:
        raise ValueError("the two levels must live on the same grid")
    check_periodicity(bc.x, grid.periodic)
    check_periodicity(bc.y, grid.periodic)
    if current.parity == previous.parity:
        raise ValueError("the two levels must sit on opposite parities")
    m = current.orders[0]
    if current.orders != (m, m) or previous.orders != (m, m):
        raise ValueError(f"levels carry orders {current.orders} and {previous.orders}, want ({m}, {m})")
    if abs(0.5 * speed * dt) > 0.5 * min(grid.hx, grid.hy) * (1.0 + 1e-12):
        raise ValueError("the energy needs c dt / 2 <= h / 2 (lambda <= 1)")
    st = Staging(current.values, previous.values)
    a = st.to_dev(current.values)
    b = st.to_dev(previous.values)
    tb2 = torch_zeros_like(a)
    gb = geom2d(grid, previous.parity, bc)
    L.check(L.lib().hw_cons2d_step(C.byref(rows2d(b)), ptr(tb2), ptr(tb2), int(m), C.byref(gb), float(dt),
                                   grid.hx, grid.hy, float(speed), st.stream), "conservative_energy_2d")
    tot = 0.0
    for dx, dy in _SEMINORMS[seminorm](m):
        npts = 2 * m + 2 - min(dx, dy)  # exact for the degree 2 (2m + 1 - d) integrand
        ia = _inner2d(a, None, grid, current.parity, bc, (m, m), dx, dy, npts, st)
        ib = _inner2d(b, None, grid, previous.parity, bc, (m, m), dx, dy, npts, st)
        iab = _inner2d(a, tb2, grid, current.parity, bc, (m, m), dx, dy, npts, st)
        tot += ia + ib - iab
    return 2.0 * tot


def torch_zeros_like(x):
    import torch

    return torch.zeros_like(x)


@dataclass(frozen=True)
class ErrorReport:
    """Refinement-study results, coarsest first (diagnostics.py:241-270)."""

    ns: np.ndarray
    hs: np.ndarray
    dts: np.ndarray
    err_u: np.ndarray
    err_dux: np.ndarray | None = None
    err_v: np.ndarray | None = None

    def __post_init__(self):
        if np.any(np.diff(self.hs) >= 0):
            raise ValueError("refinement levels must have strictly decreasing h")
        for e in (self.err_u, self.err_dux, self.err_v):
            if e is not None and not np.all(e > 0):
                raise ValueError("error norms must be positive")

    def pair_rates(self) -> np.ndarray:
        e, h = self.err_u, self.hs
        return np.log(e[:-1] / e[1:]) / np.log(h[:-1] / h[1:])

    def rate(self) -> float:
        return fit_rate(self.hs, self.err_u)


def fit_rate(hs, errors) -> float:
    """Least-squares log-log slope over the ceil(L/2) finest levels (diagnostics.py:263-278)."""
    hs = np.asarray(hs, dtype=float)
    errors = np.asarray(errors, dtype=float)
    if len(hs) < 3:
        raise ValueError(f"rate fit needs at least 3 levels, got {len(hs)}")
    k = (len(hs) + 1) // 2
    return float(np.polyfit(np.log(hs[-k:]), np.log(errors[-k:]), 1)[0])


__all__ = ["gauss_rule", "default_npts", "PlaneWave2D", "StandingWave2D", "l2_error_field_2d",
           "l2_error_field", "l2_errors_pair", "dissipative_energy", "conservative_energy", "ErrorReport",
           "fit_rate", "PRIMAL", "DUAL"]
