"""hermwave's lower-level batched building blocks on the device:
the functions the reference re-exports beside the steps, with the same
signatures, shapes and errors — numpy in, numpy out; CUDA tensors in, CUDA
tensors out.  Each is one kernel of csrc/lowlevel.cuh behind the C ABI.

The fused steps (stepping.py) do not go through these; they are for callers
written against the reference's lower-level API:

  apply_interp, apply_interp_2d          interp.py:78-111
  expand_taylor, expand_taylor_2d        dissipative.py:77-106, 184-212
  eval_series                            dissipative.py:116-121
  conservative_update_1d / _2d           conservative.py:115-136
  pascal_table                           conservative.py:43-75 (host table)
  ghost_data, ghost_data_2d              boundary.py:65-98
  pair_sources, corner_sources           boundary.py:135-168
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .config import BoundarySpec, BoundarySpec2D, SchemeConfig, check_periodicity
from .device import Staging, ptr
from .fields import Field1D, Field2D, flip
from .stepping import _PARITY

_KIND = {"dirichlet0": L.HW_DIRICHLET0, "neumann0": L.HW_NEUMANN0}


def _shape(a):
    return tuple(int(s) for s in a.shape)


def _batch(shape, tail: int) -> int:
    return int(np.prod(shape[: len(shape) - tail], dtype=np.int64)) if len(shape) > tail else 1


# ------------------------------------------------------------------ interp.py

def apply_interp(data):
    """(..., 2, mu+1) node data -> (..., 2mu+2) cell coefficients (interp.py:78-90)."""
    shp = _shape(data)
    if len(shp) < 2 or shp[-2] != 2:
        raise ValueError("data must have shape (..., 2, mu+1)")
    mu = shp[-1] - 1
    st = Staging(data)
    d = st.to_dev(data)
    out = st.empty(shp[:-2] + (2 * mu + 2,))
    L.check(L.lib().hw_apply_interp(ptr(d), ptr(out), _batch(shp, 2), int(mu), st.stream), "apply_interp")
    return st.out(out)


def apply_interp_2d(data):
    """(..., 2, 2, mux+1, muy+1) corner data -> (..., 2mux+2, 2muy+2) (interp.py:93-111)."""
    shp = _shape(data)
    if len(shp) < 4 or shp[-4] != 2 or shp[-3] != 2:
        raise ValueError("data must have shape (..., 2, 2, mux+1, muy+1)")
    mux, muy = shp[-2] - 1, shp[-1] - 1
    st = Staging(data)
    d = st.to_dev(data)
    out = st.empty(shp[:-4] + (2 * mux + 2, 2 * muy + 2))
    L.check(L.lib().hw_apply_interp_2d(ptr(d), ptr(out), _batch(shp, 4), int(mux), int(muy), st.stream),
            "apply_interp_2d")
    return st.out(out)


# ------------------------------------------------------------------ dissipative.py

def _fact(n: int) -> float:  # dissipative.py:109-113, the same float product
    out = 1.0
    for k in range(2, n + 1):
        out *= k
    return out


def expand_taylor(cu, cv, dt, h, speed, smax, forcing=None, centers=None, t=0.0):
    """1D recursion on batched cell coefficients (dissipative.py:77-106).

    Returns (CU, CV) with a trailing stage axis of length smax+1.  The
    forcing callable f(l, s, x, t) is evaluated on the host (it is the
    caller's Python code) and its terms are added on the device."""
    su, sv = _shape(cu), _shape(cv)
    lu, lv = su[-1], sv[-1]
    if su[:-1] != sv[:-1] or lv > lu:
        raise ValueError("cu (..., Lu) and cv (..., Lv) need the same batch shape and Lv <= Lu")
    smax = int(smax)
    st = Staging(cu, cv)
    du, dv = st.to_dev(cu), st.to_dev(cv)
    tu, tv = st.empty(su + (smax + 1,)), st.empty(sv + (smax + 1,))
    r = speed * speed * dt / (h * h)
    fterm = None
    if forcing is not None and smax > 0 and lv > 0:
        f = np.zeros(sv[:-1] + (lv, smax))
        for s in range(1, smax + 1):
            for l in range(lv):
                fac = h**l * dt**s / (_fact(l) * _fact(s))
                f[..., l, s - 1] = fac * np.asarray(forcing(l, s - 1, centers, t), dtype=float)
        fterm = st.to_dev(f)
    L.check(L.lib().hw_expand_taylor(ptr(du), ptr(dv), ptr(tu), ptr(tv), _batch(su, 1), int(lu), int(lv),
                                     float(dt), float(r), smax, ptr(fterm) if fterm is not None else None,
                                     st.stream), "expand_taylor")
    return st.out(tu), st.out(tv)


def expand_taylor_2d(c0, d0, dt, hx, hy, speed, smax, d1=None):
    """Tensor-coefficient recursion; tables padded to c0's footprint
    (dissipative.py:184-212).  Returns (C, D) of shape (..., K, K, smax+1)."""
    s0, sd = _shape(c0), _shape(d0)
    k, lv = s0[-1], sd[-1]
    if s0[-2] != k or sd[-2] != lv or lv > k or s0[:-2] != sd[:-2]:
        raise ValueError("c0 (..., K, K) and d0 (..., Lv, Lv) need the same batch shape and Lv <= K")
    if d1 is not None and _shape(d1) != s0[:-2] + (k - 2, k - 2):
        raise ValueError("d1 must have shape (..., K-2, K-2)")
    smax = int(smax)
    st = Staging(c0, d0, d1)
    a, b = st.to_dev(c0), st.to_dev(d0)
    e = st.to_dev(d1) if d1 is not None else None
    ct, dtab = st.empty(s0 + (smax + 1,)), st.empty(s0 + (smax + 1,))
    rx = speed * speed * dt / (hx * hx)
    ry = speed * speed * dt / (hy * hy)
    L.check(L.lib().hw_expand_taylor_2d(ptr(a), ptr(b), ptr(e) if e is not None else None, ptr(ct), ptr(dtab),
                                        _batch(s0, 2), int(k), int(lv), float(dt), float(rx), float(ry), smax,
                                        st.stream), "expand_taylor_2d")
    return st.out(ct), st.out(dtab)


def eval_series(table, theta: float):
    """Horner sum of the trailing stage axis at theta (dissipative.py:116-121)."""
    shp = _shape(table)
    if len(shp) < 1 or shp[-1] < 1:
        raise ValueError("table needs a non-empty trailing stage axis")
    st = Staging(table)
    d = st.to_dev(table)
    out = st.empty(shp[:-1])
    L.check(L.lib().hw_eval_series(ptr(d), ptr(out), _batch(shp, 1), int(shp[-1]), float(theta), st.stream),
            "eval_series")
    return st.out(out)


# ------------------------------------------------------------------ conservative.py

@dataclass(frozen=True)
class PascalTable:
    """conservative.py:43-56: base[i, j] = C(i+j, i) for i+j <= 2m;
    scaled[i, j] = base rho_x^(2i) rho_y^(2j) / (2i+2j)!."""

    m: int
    rho_x: float
    rho_y: float
    base: np.ndarray
    scaled: np.ndarray


def pascal_table(m: int, rho_x: float, rho_y: float) -> PascalTable:
    """The 2D update's Pascal coefficients (conservative.py:59-75): a small
    host table, as in the reference."""
    n = 2 * m + 1
    base = np.zeros((n, n), dtype=np.int64)
    scaled = np.zeros((n, n))
    for i in range(n):
        for j in range(n - i):
            base[i, j] = math.comb(i + j, i)
            scaled[i, j] = base[i, j] * rho_x ** (2 * i) * rho_y ** (2 * j) / math.factorial(2 * i + 2 * j)
    return PascalTable(m, rho_x, rho_y, base, scaled)


def _coeffs(interp):
    return getattr(interp, "coeffs", interp)


def conservative_update_1d(interp, prev, cfg: SchemeConfig, h: float):
    """Node data at t+dt/2 from the target-centred interpolant (..., 2m+2)
    and t-dt/2 (..., m+1) (conservative.py:115-127)."""
    c = _coeffs(interp)
    m = cfg.m
    sc, sp = _shape(c), _shape(prev)
    if sc[-1] != 2 * m + 2 or sp[-1] != m + 1 or sc[:-1] != sp[:-1]:
        raise ValueError(f"interp (..., {2 * m + 2}) and prev (..., {m + 1}) do not match")
    st = Staging(c, prev)
    dc, dp = st.to_dev(c), st.to_dev(prev)
    out = st.empty(sp)
    L.check(L.lib().hw_cons_update_1d(ptr(dc), ptr(dp), ptr(out), _batch(sp, 1), int(m), 0.5 * cfg.lam,
                                      st.stream), "conservative_update_1d")
    return st.out(out)


def conservative_update_2d(interp, prev, cfg: SchemeConfig, hx: float, hy: float):
    """Tensor version on (..., 2m+2, 2m+2) interpolant coefficients
    (conservative.py:130-136)."""
    c = _coeffs(interp)
    m = cfg.m
    sc, sp = _shape(c), _shape(prev)
    k = 2 * m + 2
    if sc[-2:] != (k, k) or sp[-2:] != (m + 1, m + 1) or sc[:-2] != sp[:-2]:
        raise ValueError(f"interp (..., {k}, {k}) and prev (..., {m + 1}, {m + 1}) do not match")
    dt = cfg.dt(min(hx, hy))
    st = Staging(c, prev)
    dc, dp = st.to_dev(c), st.to_dev(prev)
    out = st.empty(sp)
    L.check(L.lib().hw_cons_update_2d(ptr(dc), ptr(dp), ptr(out), _batch(sp, 2), int(m),
                                      0.5 * cfg.speed * dt / hx, 0.5 * cfg.speed * dt / hy, st.stream),
            "conservative_update_2d")
    return st.out(out)


# ------------------------------------------------------------------ boundary.py

def _ghost(interior, kind, axis, value):
    if kind not in _KIND:
        raise ValueError(f"cannot build ghosts for boundary kind {kind!r}")
    shp = _shape(interior)
    st = Staging(interior)
    d = st.to_dev(interior)
    out = st.empty(shp)
    n0, n1 = (shp[-2], shp[-1]) if len(shp) >= 2 and axis is not None else (shp[-1], 1)
    ax = 0 if axis is None else axis
    tail = 2 if axis is not None else 1
    L.check(L.lib().hw_ghost(ptr(d), ptr(out), _batch(shp, tail), int(n0), int(n1), int(ax), _KIND[kind],
                             float(value), st.stream), "ghost_data")
    return st.out(out)


def ghost_data(interior, kind: str, value: float = 0.0):
    """Reflect 1D node data (..., mu+1) across a wall (boundary.py:65-76)."""
    return _ghost(interior, kind, None, value)


def ghost_data_2d(interior, kind: str, normal_axis: int, value: float = 0.0):
    """Reflect 2D node data (..., kx+1, ky+1) in the normal direction (boundary.py:79-98)."""
    if normal_axis not in (0, 1):
        raise ValueError("normal_axis must be 0 or 1")
    return _ghost(interior, kind, normal_axis, value)


def _axis(spec: BoundarySpec, override):
    if override is None:
        return L.axis_bc(spec)
    return L.axis_bc(BoundarySpec(spec.left, spec.right, float(override[0]), float(override[1])))


def pair_sources(field: Field1D, spec: BoundarySpec, dirichlet_values=None):
    """Flanking data (n_targets, 2, mu+1) for every target node of the
    opposite parity, and the target coordinates (boundary.py:135-147)."""
    if spec.periodic != field.grid.periodic:
        raise ValueError("boundary spec and grid disagree about periodicity")
    v = field.values
    n, w = _shape(v)
    st = Staging(v)
    d = st.to_dev(v)
    nt = L.lib().hw_target_count(n, _PARITY[field.parity], int(field.grid.periodic))
    out = st.empty((nt, 2, w))
    bx = _axis(spec, dirichlet_values)
    L.check(L.lib().hw_gather(ptr(d), ptr(out), 1, n, 1, int(w), 1, _PARITY[field.parity], C.byref(bx), None,
                              st.stream), "pair_sources")
    return st.out(out), field.grid.nodes(flip(field.parity))


def corner_sources(field: Field2D, spec: BoundarySpec2D, dirichlet_values=None):
    """Corner data (ntx, nty, 2, 2, kx+1, ky+1) for every 2D target node of
    the opposite parity, and the target coordinates per axis
    (boundary.py:150-168; x gathered first, so corners reflect twice)."""
    for ax_spec in (spec.x, spec.y):
        check_periodicity(ax_spec, field.grid.periodic)
    v = field.values
    nx, ny, w0, w1 = _shape(v)
    st = Staging(v)
    d = st.to_dev(v)
    par = _PARITY[field.parity]
    per = int(field.grid.periodic)
    ntx, nty = L.lib().hw_target_count(nx, par, per), L.lib().hw_target_count(ny, par, per)
    out = st.empty((ntx, nty, 2, 2, w0, w1))
    bx, by = _axis(spec.x, dirichlet_values), _axis(spec.y, dirichlet_values)
    L.check(L.lib().hw_gather(ptr(d), ptr(out), 2, nx, ny, int(w0), int(w1), par, C.byref(bx), C.byref(by),
                              st.stream), "corner_sources")
    tp = flip(field.parity)
    return st.out(out), field.grid.axis(0).nodes(tp), field.grid.axis(1).nodes(tp)


__all__ = ["apply_interp", "apply_interp_2d", "expand_taylor", "expand_taylor_2d", "eval_series", "PascalTable",
           "pascal_table", "conservative_update_1d", "conservative_update_2d", "ghost_data", "ghost_data_2d",
           "pair_sources", "corner_sources"]
