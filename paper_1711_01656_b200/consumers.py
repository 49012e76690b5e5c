"""Likelihood-map consumers on the device, reference signatures:

    fuse_maps(maps, weights=None)                 likelihood.cpp:257-283
    find_peaks(map) -> (xs, ys, heights)          likelihood.cpp:285-322 (rank = index + 1)
    score_map(map, gt)                            likelihood.cpp:324-330
    camshift_refine(map, cx, cy, w, h, delta, n)  tracker.cpp:77-113

Maps are (height, width) float64 device tensors (e.g. from hist_distance_map or
build_and_match_map); results are bit-identical to the reference.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _capi as A
from ._capi import ContractError, check
from .api import Workspace, _dev, _ptr, _stream

_WS = Workspace()


def _map(m) -> torch.Tensor:
    t = _dev(m, torch.float64)
    if t.dim() != 2:
        raise ContractError(A.SPCT_ERR_CONTRACT, "map must be 2-D (height, width)")
    return t


def fuse_maps(maps, weights=None, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    ms = [_map(m) for m in maps]
    if not ms:
        raise ContractError(A.SPCT_ERR_CONTRACT, "fuse_maps: no maps to fuse")  # likelihood.cpp:258
    if any(m.shape != ms[0].shape for m in ms):
        raise ContractError(A.SPCT_ERR_CONTRACT, "fuse_maps: map dimensions differ")  # :261
    ptrs = (C.c_void_p * len(ms))(*[m.data_ptr() for m in ms])
    w = np.ascontiguousarray([] if weights is None else weights, np.float64)
    if out is None:
        out = torch.empty_like(ms[0])
    check(A.lib().spct_cu_fuse_maps(ptrs, len(ms), w.ctypes.data_as(C.POINTER(C.c_double)), w.size, ms[0].numel(),
                                    _ptr(out), _stream(stream)))
    return out


def _ws(h: int, w: int, dev) -> torch.Tensor:
    n = C.c_size_t()
    check(A.lib().spct_cu_find_peaks_workspace(w, h, C.byref(n)))
    return _WS.get(n.value, dev)


def find_peaks(m, max_out: int | None = None, stream=None):
    """(xs, ys, heights) device tensors of the peaks sorted by height (descending)."""
    t = _map(m)
    h, w = t.shape
    cap = (h * w) // 4 + 2 if max_out is None else max(0, int(max_out))
    xs = torch.empty(cap, dtype=torch.int32, device=t.device)
    ys = torch.empty(cap, dtype=torch.int32, device=t.device)
    hs = torch.empty(cap, dtype=torch.float64, device=t.device)
    cnt = C.c_int64()
    wb = _ws(h, w, t.device)
    check(A.lib().spct_cu_find_peaks(_ptr(t), w, h, _ptr(xs), _ptr(ys), _ptr(hs), cap, C.byref(cnt), _ptr(wb),
                                     wb.numel(), _stream(stream)))
    if max_out is None and cnt.value > cap:  # NaN maps: more peaks than strict maxima allow
        return find_peaks(m, cnt.value, stream)
    k = min(cnt.value, cap)
    return xs[:k], ys[:k], hs[:k]


def score_map(m, gx: int, gy: int, gw: int, gh: int, stream=None) -> int:
    t = _map(m)
    h, w = t.shape
    r = C.c_int64()
    wb = _ws(h, w, t.device)
    check(A.lib().spct_cu_score_map(_ptr(t), w, h, gx, gy, gw, gh, C.byref(r), _ptr(wb), wb.numel(), _stream(stream)))
    return int(r.value)


def camshift_batch(m, starts, win_w: int, win_h: int, delta: float = 0.5, max_iter: int = 20, stream=None):
    """One camshift_refine per (cx, cy) start: (centres (n, 2), iterations (n,), zero_mass (n,))."""
    t = _map(m)
    h, w = t.shape
    st = np.ascontiguousarray(np.asarray(starts, np.float64).reshape(-1, 2))
    n = st.shape[0]
    out = np.empty((n, 2), np.float64)
    it = np.empty(n, np.int32)
    zm = np.empty(n, np.int32)
    dp = C.POINTER(C.c_double)
    ip = C.POINTER(C.c_int32)
    check(A.lib().spct_cu_camshift(_ptr(t), w, h, st.ctypes.data_as(dp), n, win_w, win_h, float(delta), int(max_iter),
                                   out.ctypes.data_as(dp), it.ctypes.data_as(ip), zm.ctypes.data_as(ip),
                                   _stream(stream)))
    return out, it, zm.astype(bool)


def camshift_refine(m, cx: float, cy: float, win_w: int, win_h: int, delta: float = 0.5, max_iter: int = 20):
    """tracker.cpp:77-113 -> (cx, cy, iterations, zero_mass)."""
    c, it, zm = camshift_batch(m, [[cx, cy]], win_w, win_h, delta, max_iter)
    return float(c[0, 0]), float(c[0, 1]), int(it[0]), bool(zm[0])
