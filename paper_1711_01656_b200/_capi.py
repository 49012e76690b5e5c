"""ctypes binding of the C-ABI in include/spct_cuda.h (libspct_b200.so, built in-tree).

This module only declares the ABI; paper_1711_01656_b200/api.py is the
Python mirror of the reference interface on top of it.  There is no fallback:
if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SPCT_LIB_PATH: development hook for A/B runs of alternative builds of the same library
LIB_PATH = os.environ.get("SPCT_LIB_PATH") or os.path.join(HERE, "libspct_b200.so")

SPCT_OK, SPCT_ERR_CONTRACT, SPCT_ERR_IO, SPCT_ERR_CUDA, SPCT_ERR_OOM = 0, 2, 3, 4, 5
SRC_BINS_U16, SRC_GRAY_U8, SRC_RGB_U8, SRC_SCALAR_F64 = 0, 1, 2, 3
METRIC_MINKOWSKI, METRIC_INTERSECTION, METRIC_BHATTACHARYYA, METRIC_CHISQ = 0, 1, 2, 3
SPCT_IPC_HANDLE_BYTES = 64
SCHED_SEQUENTIAL, SCHED_STS, SCHED_CW_TIS, SCHED_WF_TIS = 0, 1, 2, 3


class spct_source(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("plane", C.c_void_p * 3),
        ("pitch", C.c_int64),
        ("width", C.c_int),
        ("height", C.c_int),
        ("nbins", C.c_int),
        ("lo", C.c_double),
        ("hi", C.c_double),
    ]


class spct_wih(C.Structure):
    _fields_ = [("data", C.c_void_p), ("bins", C.c_int), ("height", C.c_int), ("width", C.c_int),
                ("row_pitch", C.c_int64), ("plane_pitch", C.c_int64)]


class spct_ih(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("bins", C.c_int),
        ("bin0", C.c_int),
        ("nbins_total", C.c_int),
        ("height", C.c_int),
        ("width", C.c_int),
        ("row_pitch", C.c_int64),
        ("plane_pitch", C.c_int64),
    ]


_i, _i64, _u64, _d, _vp, _sz = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_void_p, C.c_size_t
_src_p, _ih_p = C.POINTER(spct_source), C.POINTER(spct_ih)

# name -> (restype, argtypes); every symbol declared in include/spct_cuda.h
SIGNATURES = {
    "spct_cu_last_error": (C.c_char_p, []),
    "spct_cu_version": (_i, []),
    "spct_cu_device_info": (_i, [C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "spct_cu_to_grayscale": (_i, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "spct_cu_quantize": (_i, [_src_p, _vp, _vp]),
    "spct_cu_binmap_max": (_i, [_vp, _i64, _i, _i, C.POINTER(_i), _vp]),
    "spct_cu_estimate_memory": (_i, [_i, _i, _i, _i, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_i)]),
    "spct_cu_schedule_stats": (_i, [_i, _i, _i, _i, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(_d)]),
    "spct_cu_ih_layout": (_i, [_i, _i, _i, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_u64)]),
    "spct_cu_ih_build_workspace": (_i, [_src_p, _i, _i, C.POINTER(_sz)]),
    "spct_cu_ih_build": (_i, [_src_p, _ih_p, _vp, _sz, _vp]),
    "spct_cu_ih_export_u64": (_i, [_ih_p, _i, _i, _vp, _vp]),
    "spct_cu_region_counts": (_i, [_ih_p, _vp, _i, _vp, _vp]),
    "spct_cu_hist_check": (_i, [_i, _i, _i, C.POINTER(_d), _i, _i, _i, _d]),
    "spct_cu_hist_match": (_i, [_ih_p, _vp, _i, _i, _d, _i, _vp, _vp]),
    "spct_cu_hist_match_exact": (_i, [_ih_p, _vp, _i, _i, _d, _i, _vp, _vp]),
    "spct_cu_hist_partial": (_i, [_ih_p, _vp, _i, _i, _d, _i, _vp, _i, _vp]),
    "spct_cu_hist_finalize": (_i, [_vp, _i, _i, _i, _i, _d, _i, _vp, _vp]),
    "spct_cu_fused_window_ok": (_i, [_i, _i]),
    "spct_cu_ih_build_match": (_i, [_src_p, _ih_p, _vp, _i, _i, _d, _i, _vp, _vp, _sz, _vp]),
    "spct_cu_ih_build_match_map": (_i, [_src_p, _ih_p, _vp, _i, _i, _d, _i, _vp, _vp, _sz, _vp]),
    "spct_cu_ih_build_match_map_multi": (_i, [_i, _src_p, _ih_p, C.POINTER(_vp), _i, _i, _d, _i, C.POINTER(_vp),
                                              C.POINTER(_vp), _sz, _vp]),
    "spct_cu_orientation_workspace": (_i, [_i, _i, C.POINTER(_sz)]),
    "spct_cu_orientation_bins": (_i, [_vp, _i64, _i, _i, _d, _i, _vp, _i64, _vp, _sz, _vp]),
    "spct_cu_ih_dump": (_i, [_ih_p, C.c_char_p, _i, _vp]),
    "spct_cu_ih_load_header": (_i, [C.c_char_p, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "spct_cu_ih_load": (_i, [C.c_char_p, _ih_p, _vp]),
    "spct_cu_fuse_maps": (_i, [C.POINTER(_vp), _i, C.POINTER(_d), _i, _i64, _vp, _vp]),
    "spct_cu_find_peaks_workspace": (_i, [_i, _i, C.POINTER(_sz)]),
    "spct_cu_find_peaks": (_i, [_vp, _i, _i, _vp, _vp, _vp, _i64, C.POINTER(_i64), _vp, _sz, _vp]),
    "spct_cu_score_map": (_i, [_vp, _i, _i, _i, _i, _i, _i, C.POINTER(_i64), _vp, _sz, _vp]),
    "spct_cu_camshift": (_i, [_vp, _i, _i, C.POINTER(_d), _i, _i, _i, _d, _i, C.POINTER(_d), C.POINTER(C.c_int32),
                              C.POINTER(C.c_int32), _vp]),
    "spct_cu_wih_layout": (_i, [_i, _i, _i, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_u64)]),
    "spct_cu_wih_build": (_i, [_vp, _i64, _vp, _i, _i, _i, C.POINTER(spct_wih), _vp]),
    "spct_cu_wih_export_u64": (_i, [C.POINTER(spct_wih), _i, _i, _vp, _vp]),
    "spct_cu_wih_region_counts": (_i, [C.POINTER(spct_wih), _vp, _i, _vp, _vp]),
    "spct_cu_swlh_query": (_i, [C.POINTER(spct_wih), _i, _i, C.POINTER(C.c_int32), _i, _vp, _vp]),
    "spct_cu_swlh_brute": (_i, [_vp, _i64, _i, _i, _i, _i, _i, C.POINTER(C.c_int32), _i, _vp, _vp]),
    "spct_cu_swlh_map": (_i, [C.POINTER(spct_wih), _i, _i, _vp, _vp, _vp]),
    "spct_cu_ih_accumulate": (_i, [_src_p, _ih_p, _i, _vp, _sz, _vp]),
    "spct_cu_ih_slide_workspace": (_i, [_i, _i, _i, C.POINTER(_sz)]),
    "spct_cu_ih_slide": (_i, [_src_p, _src_p, _ih_p, _vp, _sz, _vp]),
    "spct_cu_median_background": (_i, [_ih_p, _i, _i, _i, _vp, _i64, _vp]),
    "spct_cu_median_sort": (_i, [C.POINTER(_vp), _i, _i, _i, _i64, _vp, _i64, _vp]),
    "spct_cu_peer_alloc": (_i, [_sz, C.POINTER(_vp), _vp]),
    "spct_cu_peer_free": (_i, [_vp]),
    "spct_cu_peer_open": (_i, [_vp, C.POINTER(_vp)]),
    "spct_cu_peer_close": (_i, [_vp]),
    "spct_cu_flag_signal": (_i, [_vp, C.c_uint64, _vp]),
    "spct_cu_flag_wait": (_i, [_vp, _i, _i64, C.c_uint64, C.c_uint64, _vp, _vp]),
    "spct_cu_hist_finalize_slots": (_i, [_vp, _i, _i64, _i, _i, _i, _i, _d, _i, _vp, _vp]),
    "spct_cu_hist_finalize_band": (_i, [C.POINTER(_vp), _i, _i, _i, _i, _i, _d, _i, _i, _i, _vp, _vp]),
    "spct_cu_flag_signal_many": (_i, [C.POINTER(_vp), _i, C.c_uint64, _vp]),
    "spct_cu_swlh_map_direct": (_i, [_vp, _i64, _i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "spct_cu_launch_count": (C.c_uint64, []),
    "spct_cu_profile_enable": (None, [_i]),
    "spct_cu_profile_reset": (None, []),
    "spct_cu_profile_read": (_i, [C.c_char_p, C.POINTER(_d), C.POINTER(_i)]),
}


def header_symbols(path: str | None = None) -> list[str]:
    """Every spct_cu_* function declared in include/spct_cuda.h (for the export test)."""
    import re

    path = path or os.path.join(os.path.dirname(HERE), "include", "spct_cuda.h")
    with open(path) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(spct_cu_[a-z0-9_]+)\s*\(", text)))


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
                "there is no CPU fallback for the hot path")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _LIB = L
    return _LIB


class SpctError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class ContractError(SpctError, ValueError):
    """SPCT_ERR_CONTRACT — the reference would throw spct::contract_error."""


def check(status: int):
    if status == SPCT_OK:
        return
    msg = lib().spct_cu_last_error().decode(errors="replace")
    if status == SPCT_ERR_CONTRACT:
        raise ContractError(status, msg)
    raise SpctError(status, msg)
