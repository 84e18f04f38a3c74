"""ctypes binding of the C ABI in include/hermb200.h (libhermb200.so).

The library is built in-tree by ``make`` (or ``__graft_entry__.build()``).
There is no fallback: if the shared object is missing or a CUDA device is
absent, every numerical entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# HERMB200_LIB: an alternative build of the same library (A/B timing of kernel variants, tools/build_variant.sh)
LIB_PATH = os.environ.get("HERMB200_LIB") or os.path.join(_HERE, "libhermb200.so")

HW_PERIODIC, HW_DIRICHLET0, HW_NEUMANN0 = 0, 1, 2
HW_PRIMAL, HW_DUAL = 0, 1

KIND_CODES = {"periodic": HW_PERIODIC, "dirichlet0": HW_DIRICHLET0, "neumann0": HW_NEUMANN0}

# Every symbol include/hermb200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "hw_last_error", "hw_version", "hw_max_order", "hw_interp_matrix", "hw_target_count",
    "hw_diss2d_half_step", "hw_cons2d_step", "hw_boot2d", "hw_diss1d_half_step",
    "hw_cons1d_step", "hw_boot1d", "hw_l2err2d", "hw_l2err1d", "hw_count_nonfinite",
    "hw_init_planewave2d", "hw_init_standing2d", "hw_cell_map_dims", "hw_cell_map_2d",
    "hw_seminorm1d", "hw_cons_energy1d", "hw_seminorm2d", "hw_inner2d", "hw_init_1d", "hw_scale_cols",
    "hw_apply_interp", "hw_apply_interp_2d", "hw_expand_taylor", "hw_expand_taylor_2d", "hw_eval_series",
    "hw_cons_update_1d", "hw_cons_update_2d", "hw_gather", "hw_ghost",
)


class AxisBC(C.Structure):
    _fields_ = [("left_kind", C.c_int32), ("right_kind", C.c_int32),
                ("left_value", C.c_double), ("right_value", C.c_double)]


class Rows2D(C.Structure):
    _fields_ = [("base", C.c_void_p), ("halo_lo", C.c_void_p), ("halo_hi", C.c_void_p),
                ("row0", C.c_int64), ("nrows", C.c_int64)]


class Geom2D(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("parity_src", C.c_int32),
                ("periodic", C.c_int32), ("bcx", AxisBC), ("bcy", AxisBC),
                ("trow0", C.c_int64), ("ntrows", C.c_int64)]


class HermiteLibError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_L = C.c_int64


def _declare(lib):
    sig = {
        "hw_last_error": (C.c_char_p, []),
        "hw_version": (_I, []),
        "hw_max_order": (_I, []),
        "hw_interp_matrix": (_I, [_I, _P]),
        "hw_target_count": (_L, [_L, _I, _I]),
        "hw_cell_map_dims": (_I, [_I, _I, C.POINTER(_I), C.POINTER(_I)]),
        "hw_cell_map_2d": (_I, [_I, _I, _D, _D, _D, _D, _I, _P]),
        "hw_diss2d_half_step": (_I, [C.POINTER(Rows2D), C.POINTER(Rows2D), _P, _P, _I,
                                     C.POINTER(Geom2D), _D, _D, _D, _D, _I, _P]),
        "hw_cons2d_step": (_I, [C.POINTER(Rows2D), _P, _P, _I, C.POINTER(Geom2D),
                                _D, _D, _D, _D, _P]),
        "hw_boot2d": (_I, [C.POINTER(Rows2D), C.POINTER(Rows2D), _P, _I, C.POINTER(Geom2D),
                           _D, _D, _D, _D, _P]),
        "hw_diss1d_half_step": (_I, [_P, _P, _P, _P, _I, _L, _I, C.POINTER(AxisBC),
                                     _D, _D, _D, _I, _P, _P]),
        "hw_cons1d_step": (_I, [_P, _P, _P, _I, _L, _I, C.POINTER(AxisBC), _D, _P]),
        "hw_boot1d": (_I, [_P, _P, _P, _I, _L, _I, C.POINTER(AxisBC), _D, _D, _D, _P]),
        "hw_l2err2d": (_I, [C.POINTER(Rows2D), _I, _I, C.POINTER(Geom2D), _D, _D, _D, _D, _I,
                            _P, _P, _I, _P, _P, C.POINTER(_D), _P]),
        "hw_l2err1d": (_I, [_P, _I, _L, _I, C.POINTER(AxisBC), _D, _I, _I, _P, _P, _P,
                            C.POINTER(_D), _P]),
        "hw_count_nonfinite": (_I, [_P, _L, C.POINTER(_L), _P]),
        "hw_seminorm1d": (_I, [_P, _I, _L, _I, C.POINTER(AxisBC), _D, _I, _D, _I, _P, _P, C.POINTER(_D), _P]),
        "hw_cons_energy1d": (_I, [_P, _P, _I, _L, _I, _D, _D, _I, _P, _P, C.POINTER(_D), _P]),
        "hw_apply_interp": (_I, [_P, _P, _L, _I, _P]),
        "hw_apply_interp_2d": (_I, [_P, _P, _L, _I, _I, _P]),
        "hw_expand_taylor": (_I, [_P, _P, _P, _P, _L, _I, _I, _D, _D, _I, _P, _P]),
        "hw_expand_taylor_2d": (_I, [_P, _P, _P, _P, _P, _L, _I, _I, _D, _D, _D, _I, _P]),
        "hw_eval_series": (_I, [_P, _P, _L, _I, _D, _P]),
        "hw_cons_update_1d": (_I, [_P, _P, _P, _L, _I, _D, _P]),
        "hw_cons_update_2d": (_I, [_P, _P, _P, _L, _I, _D, _D, _P]),
        "hw_gather": (_I, [_P, _P, _I, _L, _L, _I, _I, _I, C.POINTER(AxisBC), C.POINTER(AxisBC), _P]),
        "hw_ghost": (_I, [_P, _P, _L, _I, _I, _I, _I, _D, _P]),
        "hw_seminorm2d": (_I, [C.POINTER(Rows2D), _I, _I, C.POINTER(Geom2D), _D, _D, _I, _I, _I, _P, _P,
                               C.POINTER(_D), _P]),
        "hw_inner2d": (_I, [C.POINTER(Rows2D), C.POINTER(Rows2D), _I, _I, C.POINTER(Geom2D), _D, _D, _I, _I, _I,
                            _P, _P, _I, C.POINTER(_D), _P]),
        "hw_scale_cols": (_I, [_P, _P, _L, _I, _D, _P]),
        "hw_init_1d": (_I, [_P, _P, _L, _I, _I, _D, _D, _D, _I, _D, _D, _I, _P]),
        "hw_init_planewave2d": (_I, [_P, _L, _L, _L, _I, _I, _D, _D, _D, _D, _D, _D, _D, _I, _P]),
        "hw_init_standing2d": (_I, [_P, _L, _L, _L, _I, _I, _D, _D, _D, _D, _D, _D, _D, _D, _D,
                                    _D, _D, _I, _P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """Load libhermb200.so once; raise if it is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise HermiteLibError(
                        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build())")
                handle = C.CDLL(LIB_PATH)
                _declare(handle)
                _lib = handle
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().hw_last_error().decode(errors="replace")
        if status == -1:
            raise ValueError(f"{what}: {msg}")
        raise HermiteLibError(f"{what} failed ({status}): {msg}")


def axis_bc(spec) -> AxisBC:
    return AxisBC(KIND_CODES[spec.left], KIND_CODES[spec.right],
                  float(spec.left_value), float(spec.right_value))
