"""The per-class cell maps the 2D kernels apply (csrc/cellmap.cpp), checked on
the CPU through the C ABI (hw_cell_map_2d) against the pinned oracle's
single-cell evaluation of the reference algorithm.  No GPU needed.

The map is built once per (scheme, m, dt, h, c, stages) by evaluating the
reference's interpolation + stage recursion + Horner sum in long double on
unit inputs, then split into the four parity classes; the dense matrix this
test reads back is re-assembled from those classes with the parity signs, so
agreement also proves the class/sign factorisation the kernel relies on.
"""

import ctypes as C

import numpy as np
import pytest

from oracle import hermite_oracle as O
from paper_1802_05246_b200 import _lib as L

DISS, CONS, BOOT = 0, 1, 2
TOL = {1: 1e-14, 2: 1e-14, 3: 1e-13, 4: 1e-13, 5: 1e-12, 6: 1e-11, 7: 1e-10, 8: 1e-9}


def dense_map(scheme, m, dt, hx, hy, speed, stages):
    din, dout = C.c_int(), C.c_int()
    L.check(L.lib().hw_cell_map_dims(scheme, m, C.byref(din), C.byref(dout)), "dims")
    out = np.empty((dout.value, 4 * din.value))
    L.check(L.lib().hw_cell_map_2d(scheme, m, dt, hx, hy, speed, stages, out.ctypes.data_as(C.c_void_p)), "map")
    return out, din.value, dout.value


def corners(rng, w, n=3):
    return rng.standard_normal((n, 2, 2, w, w))


def flat(*fields):
    """(n, 2, 2, w, w) fields -> (n, 4*din) columns corner*din + e."""
    n = fields[0].shape[0]
    per_corner = [np.concatenate([f[:, sx, sy].reshape(n, -1) for f in fields], axis=1)
                  for sx in range(2) for sy in range(2)]
    return np.concatenate(per_corner, axis=1)


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("m", range(1, 9))
@pytest.mark.parametrize("lam,hx,hy,speed,cap", [(0.9, 0.1, 0.1, 1.0, None), (0.7, 0.05, 0.08, 1.3, None),
                                                 (0.9, 0.1, 0.1, 1.0, 5)])
def test_dissipative_map(m, lam, hx, hy, speed, cap):
    rng = np.random.default_rng(100 + m)
    dt = lam * min(hx, hy) / speed
    stages = cap if cap is not None else 4 * m + 4
    W, din, dout = dense_map(DISS, m, dt, hx, hy, speed, stages)
    assert din == (m + 1) ** 2 + m * m and dout == din
    du, dv = corners(rng, m + 1), corners(rng, m)
    got = flat(du, dv) @ W.T
    wu, wv = O._step_from_corners(du, dv, hx, hy, m, lam, speed=speed, stage_cap=cap)
    want = np.concatenate([wu.reshape(len(du), -1), wv.reshape(len(du), -1)], axis=1)
    assert rel(got, want) <= TOL[m]
    # value coefficients are far better conditioned than the top orders
    assert rel(got[:, 0], want[:, 0]) <= max(1e-14, TOL[m] * 1e-2)


@pytest.mark.parametrize("m", range(1, 9))
@pytest.mark.parametrize("lam,hx,hy,speed", [(0.9, 0.1, 0.1, 1.0), (0.6, 0.04, 0.07, 2.0)])
def test_conservative_map(m, lam, hx, hy, speed):
    rng = np.random.default_rng(200 + m)
    dt = lam * min(hx, hy) / speed
    W, din, dout = dense_map(CONS, m, dt, hx, hy, speed, 0)
    assert din == dout == (m + 1) ** 2
    du = corners(rng, m + 1)
    got = flat(du) @ W.T
    c = O.interp_2d(du)
    wt = O.update_tensor_2d(m, 0.5 * speed * dt / hx, 0.5 * speed * dt / hy)
    want = (2.0 * np.einsum("klab,...ab->...kl", wt, c)).reshape(len(du), -1)
    assert rel(got, want) <= TOL[m]


@pytest.mark.parametrize("m", range(1, 9))
def test_bootstrap_map(m):
    rng = np.random.default_rng(300 + m)
    hx, hy, lam, speed = 0.1, 0.12, 0.9, 1.0
    dt = lam * min(hx, hy) / speed
    W, din, dout = dense_map(BOOT, m, dt, hx, hy, speed, 4 * m + 4)
    assert din == 2 * (m + 1) ** 2 and dout == (m + 1) ** 2
    g0, g1 = corners(rng, m + 1), corners(rng, m + 1)
    got = flat(g0, g1) @ W.T
    U, _ = O.taylor_2d(O.interp_2d(g0), O.interp_2d(g1), dt, hx, hy, speed, 4 * m + 4)
    want = O.horner(U, 0.5)[..., :m + 1, :m + 1].reshape(len(g0), -1)
    assert rel(got, want) <= TOL[m]


def test_map_rejects_bad_arguments():
    out = np.empty(16)
    with pytest.raises(ValueError):
        L.check(L.lib().hw_cell_map_2d(7, 2, 0.1, 0.1, 0.1, 1.0, 5, out.ctypes.data_as(C.c_void_p)), "map")
    with pytest.raises(ValueError):
        L.check(L.lib().hw_cell_map_2d(0, 0, 0.1, 0.1, 0.1, 1.0, 5, out.ctypes.data_as(C.c_void_p)), "map")
