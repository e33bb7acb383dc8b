"""ctypes binding of libnid.so (the C-ABI declared in include/nid.h).

There is no CPU fallback: if the library or a GPU is missing, every entry
point raises `NidUnavailable` instead of computing anything.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

LIB_PATH = os.environ.get("NID_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnid.so")
MAX_VARS = 16

CONVERGED, AT_INFINITY_CODE, SINGULAR_ENDPOINT_CODE, FAILED_CODE = 0, 1, 2, 3
CLS_AT_INFINITY, CLS_ZERO, CLS_NONZERO = 1, 4, 5

EXPORTS = (
    "nid_last_error", "nid_device_count", "nid_init", "nid_shutdown", "nid_homotopy_create",
    "nid_homotopy_destroy", "nid_eval_batch", "nid_newton_step_batch", "nid_svd_batch",
    "nid_track_batch", "nid_track_batch_strided", "nid_last_counters", "nid_refine_batch", "nid_dd_refine_batch",
    "nid_match_pairs", "nid_track_cells", "nid_track_trace", "nid_init_devices", "nid_use_device",
    "nid_compact_finite", "nid_gather_endpoints", "nid_col_lower",
)


class NidUnavailable(RuntimeError):
    """The CUDA path cannot run here (library not built or no GPU)."""


class NidError(RuntimeError):
    pass


class TrackParamsC(C.Structure):
    _fields_ = [
        ("initial_step", C.c_double), ("min_step", C.c_double), ("max_step", C.c_double),
        ("corrector_tol", C.c_double), ("max_corrector_iters", C.c_int32), ("max_steps", C.c_int32),
        ("infinity_threshold", C.c_double), ("endgame_start", C.c_double),
        ("endgame_contraction", C.c_double), ("snap_remaining", C.c_double),
        ("final_newton_iters", C.c_int32), ("dd_refine_singular", C.c_int32),
        ("soft_infinity", C.c_double), ("precision", C.c_int32), ("_pad", C.c_int32),
    ]


class HomotopyDescC(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("nterms", C.c_int32), ("row_off", C.c_void_p), ("expo", C.c_void_p),
        ("coef_start", C.c_void_p), ("coef_target", C.c_void_p), ("param_slot", C.c_void_p),
        ("nparam", C.c_int32), ("gamma_re", C.c_double), ("gamma_im", C.c_double),
        ("start_kind", C.c_int32), ("start_degrees", C.c_void_p), ("term_texp", C.c_void_p),
    ]


class PathOutC(C.Structure):
    _fields_ = [("x_end", C.c_void_p), ("status", C.c_void_p), ("steps", C.c_void_p),
                ("t_reached", C.c_void_p), ("residual", C.c_void_p), ("condition", C.c_void_p),
                ("regular", C.c_void_p)]


class CountersC(C.Structure):
    _fields_ = [("evals", C.c_longlong), ("jacs", C.c_longlong), ("scales", C.c_longlong),
                ("paths", C.c_longlong), ("dd_polished", C.c_longlong), ("lstsq_fallbacks", C.c_longlong),
                ("kernel_ms_track", C.c_double), ("kernel_ms_endpoint", C.c_double)]


_lock = threading.Lock()
_lib = None
_ready_device = None


def load_library():
    """dlopen libnid.so and declare signatures (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NidUnavailable(f"{LIB_PATH} is not built; run `python -m paper_1804_03807_b200.build`")
        lib = C.CDLL(LIB_PATH)
        p, i, d, ll = C.c_void_p, C.c_int, C.c_double, C.c_longlong
        sig = {
            "nid_last_error": ([], C.c_char_p),
            "nid_device_count": ([p], i),
            "nid_init": ([i], i),
            "nid_shutdown": ([], i),
            "nid_homotopy_create": ([p, p], i),
            "nid_homotopy_destroy": ([p], i),
            "nid_eval_batch": ([p, i, p, p, p, i, p, p, p], i),
            "nid_newton_step_batch": ([i, i, p, p, p], i),
            "nid_svd_batch": ([i, i, i, p, p], i),
            "nid_track_batch": ([p, p, i, p, ll, p, p, i, p, i, p], i),
            "nid_track_batch_strided": ([p, p, i, p, ll, ll, p, p, i, p, i, p], i),
            "nid_track_cells": ([p, p, i, p, p, p, i, p], i),
            "nid_track_trace": ([p, p, i, p, p, i, p, i, p, p], i),
            "nid_init_devices": ([i, p], i),
            "nid_use_device": ([i], i),
            "nid_compact_finite": ([i, ll, p, p, ll, ll, p, p, ll, p, p], i),
            "nid_gather_endpoints": ([i, p, p, p, p, p, p, i, i, p, p, ll, p], i),
            "nid_last_counters": ([p], i),
            "nid_col_lower": ([p, i, p, ll, p, p, ll, p, p, p, p], i),
            "nid_refine_batch": ([p, i, p, d, i, i, d, p, p, p, p, p], i),
            "nid_dd_refine_batch": ([p, i, p, i, p], i),
            "nid_match_pairs": ([i, i, i, p, p, ll, p], i),
            "nid_track_regs": ([i], i),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
        return lib


def lib():
    """The library, with a CUDA device initialised (raises when no GPU)."""
    global _ready_device
    L = load_library()
    if _ready_device is None:
        cnt = C.c_int(0)
        rc = L.nid_device_count(C.byref(cnt))
        if rc != 0 or cnt.value < 1:
            raise NidUnavailable("no CUDA device: the B200 path tracker has no CPU fallback")
        dev = int(os.environ.get("LOCAL_RANK", "0")) % cnt.value
        check(L.nid_init(dev), L)
        _ready_device = dev
    return L


def check(rc: int, L=None):
    if rc != 0:
        L = L or load_library()
        raise NidError(L.nid_last_error().decode(errors="replace"))


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(C.c_void_p)


def last_counters() -> dict:
    c = CountersC()
    check(lib().nid_last_counters(C.byref(c)))
    return {k: getattr(c, k) for k, _ in CountersC._fields_}
