"""The C-ABI library loads, exports every symbol include/hermb200.h declares,
and its host-side table code is exact (no GPU needed)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1802_05246_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hermb200.h")).read()
    return sorted(set(re.findall(r"\b(hw_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(L.EXPORTS)


def test_version_and_orders():
    assert L.lib().hw_version() == 4
    assert L.lib().hw_max_order() == 8


@pytest.mark.parametrize("mu", range(13))
def test_interp_matrix_bitwise(golden, mu):
    out = np.empty((2 * mu + 2, 2 * mu + 2))
    L.check(L.lib().hw_interp_matrix(mu, out.ctypes.data_as(C.c_void_p)), "interp")
    np.testing.assert_array_equal(out, golden[f"interp/{mu}"])


def test_interp_matrix_rejects_bad_order():
    out = np.empty(4)
    with pytest.raises(ValueError):
        L.check(L.lib().hw_interp_matrix(13, out.ctypes.data_as(C.c_void_p)), "interp")
    assert "order" in L.lib().hw_last_error().decode()


@pytest.mark.parametrize("n,par,per,want", [(8, 0, 1, 8), (8, 1, 1, 8), (9, 0, 0, 8), (8, 1, 0, 9)])
def test_target_count(n, par, per, want):
    assert L.lib().hw_target_count(n, par, per) == want


def test_bad_geometry_is_an_error_not_a_crash():
    g = L.Geom2D(4, 4, 0, 1, L.AxisBC(1, 1, 0, 0), L.AxisBC(0, 0, 0, 0), 0, -1)
    r = L.Rows2D(1, None, None, 0, 4)
    st = L.lib().hw_diss2d_half_step(C.byref(r), C.byref(r), 1, 1, 4, C.byref(g), 0.1, 0.1, 0.1, 1.0, -1, None)
    assert st == -1
    assert "periodicity" in L.lib().hw_last_error().decode()


@pytest.mark.gpu
def test_row_too_long_for_32_bit_staging_offsets_is_an_error():
    """The 2D kernels stage with 32-bit offsets inside a source row: a row of
    ny * (m+1)^2 >= 2^31 doubles is refused before any launch (fake device
    pointers are never touched)."""
    ny = 90_000_000
    g = L.Geom2D(2, ny, 0, 1, L.AxisBC(0, 0, 0, 0), L.AxisBC(0, 0, 0, 0), 0, -1)
    r = L.Rows2D(1 << 20, None, None, 0, 2)
    st = L.lib().hw_diss2d_half_step(C.byref(r), C.byref(r), 1 << 20, 1 << 20, 4, C.byref(g), 1e-9, 1e-8, 1e-8,
                                     1.0, -1, None)
    assert st == -1
    assert "too long" in L.lib().hw_last_error().decode()
