"""Joint-IH temporal median background on the device, reference API
(motion.hpp:40-68):

    MedianBackgroundIH(frames, bins, m, n)   motion.cpp:35-49 (frames already quantised)
        .slide(next)                         motion.cpp:62-69
        .background()                        motion.cpp:71-99
    median_background_ih(frames, bins, m, n) motion.cpp:101-103
    median_background_sort(frames)           motion.cpp:105-118

The joint integral histogram stays in HBM (uint32); a slide is two accumulate passes of
the build sweep.  Results are bit-identical to the reference.
"""
from __future__ import annotations

import ctypes as C
from collections import deque

import torch

from . import _capi as A
from ._capi import ContractError, check
from .api import IntegralHistogramTensor, Workspace, _dev, _ptr, _source, _stream

_WS = Workspace()


def _frames(frames) -> list:
    fs = [_dev(f, torch.uint8) for f in frames]
    if not fs:
        raise ContractError(A.SPCT_ERR_CONTRACT, "FrameWindow: empty window")  # motion.cpp:13
    if len(fs) % 2 != 1:
        raise ContractError(A.SPCT_ERR_CONTRACT, "FrameWindow: window length must be odd")  # :14
    h, w = fs[0].shape
    if not (w > 0 and h > 0):
        raise ContractError(A.SPCT_ERR_CONTRACT, "FrameWindow: empty frames")
    if any(f.shape != fs[0].shape for f in fs):
        raise ContractError(A.SPCT_ERR_CONTRACT, "FrameWindow: frame dimensions differ")  # :18
    return fs


class MedianBackgroundIH:
    def __init__(self, frames, bins: int, m: int, n: int, stream=None):
        fs = _frames(frames)
        if not (1 <= bins <= 256):
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: bins must be in [1,256]")
        if not (m >= 1 and n >= 1 and m % 2 == 1 and n % 2 == 1):
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: kernel sides must be odd and positive")
        self.height, self.width = fs[0].shape
        if m > self.width or n > self.height:
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: kernel exceeds image")
        if len(fs) * self.width * self.height >= 1 << 32:
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: frames * H * W must be < 2^32")
        self.bins, self.m, self.n, self.stream = bins, m, n, stream
        self.joint = IntegralHistogramTensor(self.width, self.height, bins, device=fs[0].device)
        self.joint.storage.zero_()
        self.frames = deque()
        for f in fs:
            self._add(f, +1)
            self.frames.append(f)

    def _add(self, f: torch.Tensor, sign: int, validate: bool = True) -> None:
        if validate and int(f.max().item()) >= self.bins:  # motion.cpp:23-26
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: frame value exceeds bin count")
        bm = f.to(torch.int16)  # the frame's values are its bins (motion.cpp:53-54)
        src = _source(A.SRC_BINS_U16, [bm], self.width, self.height, self.bins)
        ws = C.c_size_t()
        check(A.lib().spct_cu_ih_build_workspace(C.byref(src), 0, self.bins, C.byref(ws)))
        wb = _WS.get(ws.value, bm.device, self.stream)
        check(A.lib().spct_cu_ih_accumulate(C.byref(src), C.byref(self.joint.desc), sign, _ptr(wb), wb.numel(),
                                            _stream(self.stream)))

    def slide(self, nxt) -> None:
        """motion.cpp:62-69: J += IH(next) - IH(oldest) in one read-modify-write pass of J
        (spct_cu_ih_slide) instead of an add and a subtract pass."""
        f = _dev(nxt, torch.uint8)
        if tuple(f.shape) != (self.height, self.width):
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: slide frame dimensions differ")
        if int(f.max().item()) >= self.bins:  # motion.cpp:23-26
            raise ContractError(A.SPCT_ERR_CONTRACT, "median_background_ih: frame value exceeds bin count")
        # the outgoing frame passed the same check when it entered (motion.cpp:64-65 repeats it)
        old = self.frames.popleft()
        bn, bo = f.to(torch.int16), old.to(torch.int16)  # the frames' values are their bins (motion.cpp:53-54)
        sn = _source(A.SRC_BINS_U16, [bn], self.width, self.height, self.bins)
        so = _source(A.SRC_BINS_U16, [bo], self.width, self.height, self.bins)
        ws = C.c_size_t()
        check(A.lib().spct_cu_ih_slide_workspace(self.width, self.height, self.bins, C.byref(ws)))
        wb = _WS.get(ws.value, bn.device, self.stream)
        check(A.lib().spct_cu_ih_slide(C.byref(sn), C.byref(so), C.byref(self.joint.desc), _ptr(wb), wb.numel(),
                                       _stream(self.stream)))
        self.frames.append(f)

    def background(self) -> torch.Tensor:
        out = torch.empty((self.height, self.width), dtype=torch.uint8, device=self.joint.storage.device)
        check(A.lib().spct_cu_median_background(C.byref(self.joint.desc), len(self.frames), self.m, self.n, _ptr(out),
                                                self.width, _stream(self.stream)))
        return out


def median_background_ih(frames, bins: int, m: int, n: int) -> torch.Tensor:
    return MedianBackgroundIH(frames, bins, m, n).background()


def median_background_sort(frames, stream=None) -> torch.Tensor:
    fs = _frames(frames)
    h, w = fs[0].shape
    out = torch.empty((h, w), dtype=torch.uint8, device=fs[0].device)
    ptrs = (C.c_void_p * len(fs))(*[f.data_ptr() for f in fs])
    check(A.lib().spct_cu_median_sort(ptrs, len(fs), w, h, w, _ptr(out), w, _stream(stream)))
    return out
