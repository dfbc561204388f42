"""ctypes binding of the C ABI in include/riesz_mgrit_b200.h.

The shared library is the product: there is no CPU fallback.  Loading it is
cheap and works without a GPU (the CPU test suite checks the exported
symbols); every compute entry point needs a CUDA device and raises
``NativeError`` when the call fails.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

__all__ = ["lib", "NativeError", "Sweep", "check", "EXPORTS"]


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


class Sweep(C.Structure):
    """Mirror of ``rm_sweep`` (include/riesz_mgrit_b200.h)."""

    _fields_ = [
        ("nchains", C.c_int), ("first", C.c_int), ("cstride", C.c_int), ("clen", C.c_int), ("nmax", C.c_int),
        ("explicit_rhs", C.c_int), ("x0_mode", C.c_int), ("out_div", C.c_int),
        ("d_dt", C.c_void_p),
        ("d_src", C.c_void_p), ("src_stride", C.c_int64),
        ("d_x0", C.c_void_p), ("x0_stride", C.c_int64),
        ("d_f", C.c_void_p), ("f_stride", C.c_int64),
        ("d_fscale", C.c_void_p),
        ("d_gadd", C.c_void_p), ("gadd_stride", C.c_int64),
        ("d_sub", C.c_void_p), ("sub_stride", C.c_int64),
        ("d_out", C.c_void_p), ("out_stride", C.c_int64),
        ("d_norms", C.c_void_p),
        ("rel_tol", C.c_double),
        ("max_iter", C.c_int64),
        ("d_counters", C.c_void_p),
        ("group", C.c_int),
        ("precond", C.c_int),
        ("d_guess", C.c_void_p),
        ("guess_stride", C.c_int64),
        ("d_keep", C.c_void_p), ("keep_stride", C.c_int64),
        ("lp_matvec", C.c_int),
        ("d_hg", C.c_void_p), ("hg_stride", C.c_int64),
        ("d_ax", C.c_void_p), ("ax_stride", C.c_int64),
        ("d_gax", C.c_void_p), ("gax_stride", C.c_int64),
        ("d_ain", C.c_void_p), ("ain_stride", C.c_int64),
        ("d_gscale", C.c_void_p),
    ]


_D = C.POINTER(C.c_double)
EXPORTS = {
    "rm_version": (C.c_char_p, []),
    "rm_last_error": (C.c_char_p, []),
    "rm_max_order": (C.c_int, []),
    "rm_grid_create": (C.c_int, [C.c_int, C.c_int, _D, _D, _D, _D, _D, _D, _D, _D, C.c_double, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.POINTER(C.c_void_p)]),
    "rm_grid_destroy": (C.c_int, [C.c_void_p]),
    "rm_apply_batched": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_int64, C.c_void_p]),
    "rm_sweep_run": (C.c_int, [C.c_void_p, C.POINTER(Sweep), C.c_void_p]),
    "rm_grid_set_tau": (C.c_int, [C.c_void_p, _D, _D]),
    "rm_fail_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int64),
                               C.POINTER(C.c_double)]),
    "rm_fail_reset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rm_debug_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong)]),
    "rm_grid_flags": (C.c_int, [C.c_void_p]),
    "rm_correct": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                             C.c_void_p]),
    "rm_diff_sqnorm": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rm_vec_dot": (C.c_int, [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rm_vec_axpby": (C.c_int, [C.c_int64, C.c_double, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rm_pcg64_uniform": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64,
                                   C.c_int64, C.c_void_p, C.c_int64, C.c_void_p]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load (building first if the sources are newer) the shared library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = os.environ.get("RM_LIB")  # e.g. the -DRM_TIMING debug variant
            if not path:
                path = _build.lib_path()
                if not os.path.exists(path) or (_build.is_stale() and os.environ.get("RM_NO_BUILD") != "1"):
                    path = _build.build()
            handle = C.CDLL(path)
            for name, (res, args) in EXPORTS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int, what: str) -> int:
    if status < 0:
        msg = lib().rm_last_error().decode(errors="replace")
        if status == -1:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed ({status}): {msg}")
    return status
