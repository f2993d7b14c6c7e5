"""ctypes binding of the C ABI in ``include/wavekernel_b200.h``.

The shared library ``libwk_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, sm_100a).  There is no fallback: if the
library is missing every GPU entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_double, c_int, c_int32, c_int64,
                    c_void_p, c_char_p)

import numpy as np

LIB_PATH = os.environ.get("WK_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libwk_b200.so")

WK_OK, WK_EINVAL, WK_ECUDA, WK_ESTATE = 0, 1, 2, 3
WK_GEOM_AFFINE, WK_GEOM_CURVED = 0, 1
PARTS = {"cell": 1, "face": 2, "both": 3}
POLICY = {"none": 0, "every_step": 1, "every_second": 2, "every_third": 3}
WK_ADER, WK_ADER_HDG = 0, 1
TABLE = {"gauss_points": 0, "gauss_weights": 1, "gl_points": 2, "gl_weights": 3,
         "gl_to_g": 4, "g_to_gl": 5, "d_gl": 6, "d_co": 7, "resize": 8,
         "a_split": 9, "lift": 10}


class WkDesc(Structure):
    _fields_ = [
        ("dim", c_int32), ("degree", c_int32),
        ("n_elements", c_int64), ("n_ghost_faces", c_int64),
        ("neighbors", POINTER(c_int32)),
        ("inv_rho", POINTER(c_double)), ("c2rho", POINTER(c_double)),
        ("tau", POINTER(c_double)),
        ("stabilization", c_int32), ("geometry_mode", c_int32),
        ("n_classes", c_int64), ("geo_class", POINTER(c_int32)),
        ("affine_G", POINTER(c_double)), ("affine_det", POINTER(c_double)),
        ("affine_normal", POINTER(c_double)), ("affine_fscale", POINTER(c_double)),
        ("n_curved_degrees", c_int32), ("curved_degrees", POINTER(c_int32)),
        ("curved_inv_jac", POINTER(POINTER(c_double))),
        ("curved_jxw", POINTER(POINTER(c_double))),
        ("face_normal", POINTER(POINTER(c_double))),
        ("face_jxw", POINTER(POINTER(c_double))),
    ]


_SIGS = {
    "wk_version": (c_int, []),
    "wk_last_error": (c_char_p, []),
    "wk_ctx_create": (c_int, [POINTER(WkDesc), POINTER(c_void_p)]),
    "wk_ctx_destroy": (c_int, [c_void_p]),
    "wk_apply_K": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "wk_apply_minv_K": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "wk_rhs": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_apply_inverse_mass": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_apply_mass": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_to_gauss_values": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_from_gauss_weighted": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_apply_local_S": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "wk_resize_values": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p]),
    "wk_lsrk_stage": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                              c_double, c_double, c_void_p]),
    "wk_lsrk_stage_ex": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                                 c_double, c_double, c_int, c_void_p]),
    "wk_tck": (c_int, [c_void_p, c_void_p, c_void_p, c_double, c_int, c_int, c_void_p]),
    "wk_ader_step": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p,
                             c_double, c_void_p]),
    "wk_ader_a": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p, c_double,
                          c_void_p]),
    "wk_ader_b": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_curved_metric": (c_int, [c_int, c_int, c_int64, c_void_p, POINTER(c_int32),
                                 POINTER(c_double), POINTER(c_double), POINTER(c_double),
                                 POINTER(c_double), POINTER(c_double),
                                 c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p]),
    "wk_state_norm_sq": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_mode_state": (c_int, [c_int, c_int, c_int64, c_void_p, c_int, c_double, c_double,
                              c_double, c_void_p, c_void_p]),
    "wk_l2_pressure_error": (c_int, [c_int, c_int, c_int64, c_void_p, c_void_p, c_int,
                                     c_double, c_double, c_double, c_int, c_void_p, c_void_p]),
    "wk_ghost_buffer": (c_void_p, [c_void_p]),
    "wk_set_ghost_buffer": (c_int, [c_void_p, c_void_p]),
    "wk_set_halo_exports": (c_int, [c_void_p, c_int64, POINTER(c_int64), POINTER(c_int32)]),
    "wk_pack_halo": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "wk_set_element_range": (c_int, [c_void_p, c_int64, c_int64]),
    "wk_set_tile_order": (c_int, [c_void_p, c_int64, c_int64, c_int64]),
    "wk_lsrk_run_supported": (c_int, [c_void_p]),
    "wk_lsrk_run": (c_int, [c_void_p, c_void_p, c_void_p, c_int, POINTER(c_double),
                            POINTER(c_double), c_double, c_int, c_void_p]),
    "wk_debug_set_neighbor": (c_int, [c_void_p, c_int64, c_int, c_int32]),
    "wk_set_queue_slot": (c_int, [c_void_p, c_int]),
    "wk_basis_table": (c_int, [c_int, c_int, c_int, POINTER(c_double), c_int]),
}

_lib = None


def lib():
    """Load (once) and return the CUDA library; raise loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA library {LIB_PATH} is missing; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == WK_OK:
        return
    msg = lib().wk_last_error().decode(errors="replace")
    if rc == WK_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def dptr(arr):
    """Typed ctypes pointer into a host numpy array (kept alive by caller)."""
    if arr is None:
        return None
    if arr.dtype == np.float64:
        return arr.ctypes.data_as(POINTER(c_double))
    if arr.dtype == np.int32:
        return arr.ctypes.data_as(POINTER(c_int32))
    if arr.dtype == np.int64:
        return arr.ctypes.data_as(POINTER(c_int64))
    raise TypeError(arr.dtype)


def basis_table(kind: str, k: int, k_to: int = 0) -> np.ndarray:
    """1-D tables computed natively (long double) by the library."""
    out = np.empty(2 * 13 * 13 + 32)
    n = lib().wk_basis_table(TABLE[kind], int(k), int(k_to), dptr(out), out.size)
    if n < 0:
        raise ValueError(f"no {kind} table for k={k}")
    res = out[:n].copy()
    sq = {"gl_to_g", "g_to_gl", "d_gl", "d_co", "a_split"}
    if kind in sq:
        return res.reshape(k + 1, k + 1)
    if kind == "resize":
        return res.reshape(k_to + 1, k + 1)
    if kind == "lift":
        return res.reshape(2, k + 1)
    return res
