"""Spatially weighted local histograms on the device, reference API
(swih.hpp, integral.hpp:102-104):

    kernel_extents(kw, kh)                        swih.cpp:19-27
    build_weighted_tensor(bins, weights, nbins)   integral.cpp:553-559 (uint64, 16.16)
    build_quadrant_set(bins, nbins, kw, kh)       swih.cpp:115-126
    swlh_query_fixed / swlh_query                 swih.cpp:128-164, 182-197
    brute_force_swlh_fixed                        swih.cpp:166-178
    swlh_distance_map(bins, nbins, model, kw, kh) the tracker's channel, track_loop.cpp:264-283

BinMaps are uint16 (numpy or device int16 tensors); frames (uint8) are quantised with
quantize(frame, nbins) first.  Fixed-point results are bit-identical to the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi as A
from ._capi import ContractError, check
from .api import _dev, _ptr, _stream


def kernel_extents(kw: int, kh: int):
    """(sxl, sxr, syt, syb, c), swih.cpp:19-27."""
    if not (kw >= 1 and kh >= 1):
        raise ContractError(A.SPCT_ERR_CONTRACT, "kernel extents must be >= 1")
    sxl, syt = kw // 2, kh // 2
    return sxl, kw - sxl, syt, kh - syt, sxl + syt + 1


class WeightedTensor:
    """Device weighted integral histogram (uint64 cells, unpadded + pitched)."""

    def __init__(self, width: int, height: int, bins: int, device=None):
        rp, pp, nb = C.c_int64(), C.c_int64(), C.c_uint64()
        check(A.lib().spct_cu_wih_layout(width, height, bins, C.byref(rp), C.byref(pp), C.byref(nb)))
        self.width, self.height, self.bins = width, height, bins
        self.storage = torch.empty(nb.value // 8, dtype=torch.int64, device=device or "cuda")
        self.desc = A.spct_wih(self.storage.data_ptr(), bins, height, width, rp.value, pp.value)

    def padded_u64(self, k0: int = 0, k1: int | None = None, stream=None) -> np.ndarray:
        """Reference layout (integral.hpp:78-93): uint64, zero padding row / column."""
        k1 = self.bins if k1 is None else k1
        out = torch.empty((k1 - k0) * (self.height + 1) * (self.width + 1), dtype=torch.int64,
                          device=self.storage.device)
        check(A.lib().spct_cu_wih_export_u64(C.byref(self.desc), k0, k1, _ptr(out), _stream(stream)))
        return out.cpu().numpy().view(np.uint64).reshape(k1 - k0, self.height + 1, self.width + 1)


def _binmap(bm, nbins: int) -> torch.Tensor:
    t = _dev(bm, torch.int16)
    if t.dim() != 2 or t.numel() == 0:
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: empty bin map")
    if nbins < 1:
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: bins must be >= 1")
    h, w = t.shape
    mx = C.c_int()
    check(A.lib().spct_cu_binmap_max(_ptr(t), w, w, h, C.byref(mx), _stream(None)))
    if mx.value >= nbins:  # integral.cpp:337-343
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: bin index out of range")
    return t


def build_weighted_tensor(bm, weights, nbins: int, stream=None) -> WeightedTensor:
    b = _binmap(bm, nbins)
    h, w = b.shape
    wt = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(weights, np.uint64).view(np.int64))
    wt = wt.to(b.device).contiguous()
    if tuple(wt.shape) != (h, w):
        raise ContractError(A.SPCT_ERR_CONTRACT, "build_weighted_tensor: weight size mismatch")  # integral.cpp:557
    t = WeightedTensor(w, h, nbins, device=b.device)
    check(A.lib().spct_cu_wih_build(_ptr(b), w, _ptr(wt), -1, 1, 1, C.byref(t.desc), _stream(stream)))
    return t


@dataclass
class WeightedQuadrantSet:
    kw: int
    kh: int
    sx: int
    sy: int
    pair_sum: int
    tensors: list  # [NW, NE, SW, SE]

    def descs(self):
        return (A.spct_wih * 4)(*[t.desc for t in self.tensors])


def build_quadrant_set(bm, nbins: int, kw: int, kh: int, stream=None) -> WeightedQuadrantSet:
    kernel_extents(kw, kh)
    b = _binmap(bm, nbins)
    h, w = b.shape
    sx, sy = int(kw >= 3), int(kh >= 3)
    ts = []
    for d in range(4):
        t = WeightedTensor(w, h, nbins, device=b.device)
        check(A.lib().spct_cu_wih_build(_ptr(b), w, None, d, kw, kh, C.byref(t.desc), _stream(stream)))
        ts.append(t)
    return WeightedQuadrantSet(kw, kh, sx, sy, 2 + sx * (w - 1) + sy * (h - 1), ts)


def _centres(centres) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(centres, np.int32).reshape(-1, 2))


def swlh_query_fixed(s: WeightedQuadrantSet, centres, kw: int | None = None, kh: int | None = None,
                     stream=None) -> np.ndarray:
    """(n, bins) int64 16.16; kw/kh, when given, must equal the set's kernel (swih.cpp:130)."""
    if (kw is not None and kw != s.kw) or (kh is not None and kh != s.kh):
        raise ContractError(A.SPCT_ERR_CONTRACT, "swlh_query: kernel spec differs from the built set")
    c = _centres(centres)
    bins = s.tensors[0].bins
    out = torch.empty((len(c), bins), dtype=torch.int64, device=s.tensors[0].storage.device)
    check(A.lib().spct_cu_swlh_query(s.descs(), s.kw, s.kh, c.ctypes.data_as(C.POINTER(C.c_int32)), len(c),
                                     _ptr(out), _stream(stream)))
    return out.cpu().numpy()


def swlh_query(s: WeightedQuadrantSet, centres, kw: int | None = None, kh: int | None = None) -> np.ndarray:
    """Unit-mass normalisation (swih.cpp:182-197) in FP64 (the reference: x87 long double)."""
    fx = swlh_query_fixed(s, centres, kw, kh)
    tot = fx.sum(axis=1, keepdims=True).astype(np.float64)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(tot > 0, fx / np.where(tot > 0, tot, 1.0), 0.0)


def brute_force_swlh_fixed(bm, nbins: int, centres, kw: int, kh: int, stream=None) -> np.ndarray:
    b = _binmap(bm, nbins)
    h, w = b.shape
    c = _centres(centres)
    out = torch.empty((len(c), nbins), dtype=torch.int64, device=b.device)
    check(A.lib().spct_cu_swlh_brute(_ptr(b), w, w, h, nbins, kw, kh, c.ctypes.data_as(C.POINTER(C.c_int32)), len(c),
                                     _ptr(out), _stream(stream)))
    return out.cpu().numpy()


def swlh_distance_map(bm, nbins: int, model, kw: int, kh: int, stream=None, method: str = "direct") -> torch.Tensor:
    """The tracker's swlh-distance likelihood map (track_loop.cpp:264-283), (h, w) float64.

    method "direct" (kw <= 128, kh <= 255): one sweep over the BinMap with exact running
    pyramid sums (swlh_fused.cu); "quadrant": the reference's construction, the four
    weighted tensors of build_quadrant_set then a query per centre.  Same bits."""
    if method not in ("direct", "quadrant"):
        raise ContractError(A.SPCT_ERR_CONTRACT, "swlh_map: method must be 'direct' or 'quadrant'")
    if method == "direct" and kw <= 128 and kh <= 255:
        kernel_extents(kw, kh)
        b = _binmap(bm, nbins)
        h, w = b.shape
        md = torch.from_numpy(np.ascontiguousarray(model, np.float64).reshape(-1)).to(b.device)
        if md.numel() != nbins:
            raise ContractError(A.SPCT_ERR_CONTRACT, "swlh_map: model length must equal bins")
        out = torch.empty((h, w), dtype=torch.float64, device=b.device)
        check(A.lib().spct_cu_swlh_map_direct(_ptr(b), w, w, h, nbins, kw, kh, _ptr(md), _ptr(out), _stream(stream)))
        return out
    s = build_quadrant_set(bm, nbins, kw, kh, stream)
    md = torch.from_numpy(np.ascontiguousarray(model, np.float64).reshape(-1)).to(s.tensors[0].storage.device)
    if md.numel() != nbins:
        raise ContractError(A.SPCT_ERR_CONTRACT, "swlh_map: model length must equal bins")
    out = torch.empty((s.tensors[0].height, s.tensors[0].width), dtype=torch.float64, device=md.device)
    check(A.lib().spct_cu_swlh_map(s.descs(), kw, kh, _ptr(md), _ptr(out), _stream(stream)))
    return out
