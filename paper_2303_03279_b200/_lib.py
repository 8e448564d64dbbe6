"""ctypes binding of libcsconn.so (include/csconn.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``).  There is
no CPU fallback: importing the product path on a machine without the built
library or without a CUDA device raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

# CSCONN_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("CSCONN_LIB") or Path(__file__).resolve().parent / "libcsconn.so")

CS_OK, CS_EPARAM, CS_EDEGENERATE, CS_ECUDA, CS_ENOMEM = 0, 1, 2, 3, 4
CS_F32, CS_F64 = 0, 1
NUM_METRICS = 8


class CsOutputs(ctypes.Structure):
    _fields_ = [("bins", ctypes.c_void_p * NUM_METRICS),
                ("band", ctypes.c_void_p * NUM_METRICS),
                ("pair_base", ctypes.c_int64),
                ("pair_stride", ctypes.c_int64)]


class CsSums(ctypes.Structure):
    _fields_ = [("csd", ctypes.c_void_p), ("plv", ctypes.c_void_p), ("pli", ctypes.c_void_p),
                ("abs_im", ctypes.c_void_p), ("psd", ctypes.c_void_p),
                ("pair_base", ctypes.c_int64), ("pair_stride", ctypes.c_int64)]


class CsRingHandle(ctypes.Structure):
    _fields_ = [("x64", ctypes.c_ubyte * 64), ("x32", ctypes.c_ubyte * 64), ("n_nodes", ctypes.c_int32),
                ("slot_capacity", ctypes.c_int32), ("n_tapers", ctypes.c_int32), ("n_bins", ctypes.c_int32)]


_lib = None


def lib():
    """Load libcsconn.so once; raise loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build())")
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i32, i64, u32, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint, ctypes.c_double
    L.cs_plan_create.argtypes = [ctypes.POINTER(vp), i32, i32, i32, i32, i32, i32, i32,
                                 ctypes.POINTER(dbl), i32, dbl, u32]
    L.cs_plan_destroy.argtypes = [vp]
    L.cs_spectra.argtypes = [vp, vp, i32, i64, i64, i32, i32, vp]
    L.cs_pair_metrics.argtypes = [vp, vp, i32, u32, i32, i32, i32, i32, ctypes.POINTER(CsOutputs), vp]
    L.cs_pair_metrics_ex.argtypes = [vp, vp, i32, u32, i32, i32, i32, i32, ctypes.POINTER(CsOutputs), u32, vp]
    L.cs_get_spectra.argtypes = [vp, vp, i32, i32, i32, vp, vp]
    L.cs_put_spectra.argtypes = [vp, vp, i32, i32, i32, i32, vp]
    L.cs_net_normalize.argtypes = [vp, vp, i64, vp]
    L.cs_net_threshold.argtypes = [vp, i64, i64, vp, vp]
    L.cs_cor_sums.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    L.cs_xcor_sums.argtypes = [vp, i32, i32, i32, i32, vp, vp, vp, vp]
    L.cs_plan_k1_kind.argtypes = [vp]
    L.cs_pair_sums.argtypes = [vp, vp, i32, i32, i32, ctypes.POINTER(CsSums), vp]
    L.cs_put_taper_spectra.argtypes = [vp, vp, i32, i32, i32, i32, i32, dbl, vp]
    L.cs_num_row_tiles.argtypes = [i32]
    L.cs_row_tile_range.argtypes = [i32, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                    ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.cs_last_fallback_count.argtypes = [vp, vp, ctypes.POINTER(i64)]
    L.cs_last_guard_stats.argtypes = [vp, vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.cs_last_imag_handoff.argtypes = [vp]
    L.cs_last_imag_handoff.restype = ctypes.c_int
    L.cs_fft_call_count.argtypes = [vp]
    L.cs_fft_call_count.restype = i64
    L.cs_reset_fft_call_count.argtypes = [vp]
    L.cs_reset_fft_call_count.restype = None
    L.cs_plan_set_profiling.argtypes = [vp, i32]
    L.cs_profile_read.argtypes = [vp, ctypes.c_char_p, i32]
    L.cs_launch_count.argtypes = [vp]
    L.cs_launch_count.restype = i64
    L.cs_ring_view.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(i64)]
    L.cs_window_create.argtypes = [ctypes.POINTER(vp), vp, u32, i32, i32]
    L.cs_window_destroy.argtypes = [vp]
    L.cs_window_reset.argtypes = [vp, vp]
    L.cs_window_update.argtypes = [vp, vp, i32, i32, vp, i32, ctypes.POINTER(CsOutputs), vp]
    L.cs_apply_inverse.argtypes = [vp, i32, i32, vp, i32, vp, vp]
    L.cs_project_ring.argtypes = [vp, vp, vp, i32, i32, vp]
    L.cs_fir_apply.argtypes = [vp, i32, vp, i32, i32, vp, vp, vp, vp]
    L.cs_spectra_nodes.argtypes = [vp, vp, i32, i64, i64, i32, i32, i32, i32, vp]
    L.cs_ring_export.argtypes = [vp, ctypes.POINTER(CsRingHandle)]
    L.cs_ring_attach.argtypes = [vp, ctypes.POINTER(CsRingHandle), i32, i32, i32]
    L.cs_ring_attach_ptrs.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), i32, i32, i32]
    L.cs_ring_push.argtypes = [vp, i32, i32, i32, i32, vp]
    L.cs_probe_peaks.argtypes = [i32, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]
    L.cs_last_error.restype = ctypes.c_char_p
    L.cs_version.restype = ctypes.c_char_p
    _lib = L
    return L


CS_PLAN_WELCH = 1
CS_PM_REUSE_PREP = 1

EXPORTED = ("cs_plan_create", "cs_plan_destroy", "cs_spectra", "cs_pair_metrics", "cs_pair_metrics_ex", "cs_pair_sums",
            "cs_get_spectra", "cs_put_spectra", "cs_put_taper_spectra", "cs_net_normalize", "cs_net_threshold", "cs_cor_sums", "cs_xcor_sums", "cs_apply_inverse", "cs_project_ring", "cs_fir_apply",
            "cs_window_create", "cs_window_destroy", "cs_window_reset", "cs_window_update", "cs_plan_k1_kind", "cs_num_row_tiles", "cs_row_tile_range", "cs_last_fallback_count", "cs_last_guard_stats", "cs_last_imag_handoff",
            "cs_fft_call_count", "cs_reset_fft_call_count", "cs_plan_set_profiling", "cs_profile_read",
            "cs_launch_count", "cs_ring_view", "cs_spectra_nodes", "cs_ring_export", "cs_ring_attach",
            "cs_ring_attach_ptrs", "cs_ring_push", "cs_probe_peaks", "cs_last_error", "cs_version")


def check(status: int) -> None:
    """Map a csconn status code to the reference's exception classes (core.py:17-22)."""
    if status == CS_OK:
        return
    from .core import DegenerateTrialCountError, ParameterError
    msg = lib().cs_last_error().decode(errors="replace")
    if status == CS_EPARAM:
        raise ParameterError(msg)
    if status == CS_EDEGENERATE:
        raise DegenerateTrialCountError(msg)
    if status == CS_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"csconn CUDA failure: {msg}")
