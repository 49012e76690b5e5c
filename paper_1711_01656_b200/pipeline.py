"""Double-buffered frame pipeline: host frames in, host likelihood maps out.

The reference overlaps frame decoding with computation on two host threads
(proj/src/pipeline.cpp:45-153, the CPU analogue of the thesis' dual-buffer
Alg. 10).  Here the overlap is between PCIe copies and the
sweep: frame n+1's host->device copy (copy stream 1) and frame n-1's map
device->host copy (copy stream 2) run while the fused sweep processes frame n
on the compute stream.  Device buffers are double-buffered; host buffers must be
pinned for the copies to be asynchronous.  Every frame's copies are real: nothing
is skipped or cached.
"""
from __future__ import annotations

import numpy as np
import torch

from . import api as _api
from ._capi import METRIC_MINKOWSKI


class FramePipeline:
    def __init__(self, width: int, height: int, nbins: int, tmpl, kw: int, kh: int, p: float = 1.0,
                 metric: int = METRIC_MINKOWSKI, store_tensor: bool = True, device=None):
        self.dev = torch.device(device or "cuda")
        self.w, self.h, self.nbins, self.kw, self.kh, self.p, self.metric = width, height, nbins, kw, kh, p, metric
        self.tmpl_dev = _api._tmpl(tmpl, nbins, width, height, kw, kh, p).to(self.dev)
        self.tensor = _api.IntegralHistogramTensor(width, height, nbins, device=self.dev, store=store_tensor)
        self.frames = [torch.empty((height, width), dtype=torch.uint8, device=self.dev) for _ in range(2)]
        self.maps = [torch.empty((height, width), dtype=torch.float64, device=self.dev) for _ in range(2)]
        self.compute = torch.cuda.Stream(self.dev)
        self.h2d = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        self.loaded = [torch.cuda.Event() for _ in range(2)]    # frame i copied in
        self.done = [torch.cuda.Event() for _ in range(2)]      # map i computed
        self.drained = [torch.cuda.Event() for _ in range(2)]   # map i copied out (buffer reusable)
        self.consumed = [torch.cuda.Event() for _ in range(2)]  # frame i read by the sweep (buffer reusable)
        for e in self.drained + self.consumed:
            e.record(self.compute)

    def run(self, host_frames, host_maps) -> None:
        """host_frames: sequence of (h, w) uint8 pinned CPU tensors; host_maps: same length
        of (h, w) float64 pinned CPU tensors, filled in place.  Returns when every map
        has landed on the host."""
        n = len(host_frames)
        for i in range(n):
            b = i & 1
            with torch.cuda.stream(self.h2d):
                self.h2d.wait_event(self.consumed[b])
                self.frames[b].copy_(host_frames[i], non_blocking=True)
                self.loaded[b].record(self.h2d)
            with torch.cuda.stream(self.compute):
                self.compute.wait_event(self.loaded[b])
                self.compute.wait_event(self.drained[b])
                _api.build_and_match_map(self.frames[b], self.nbins, None, self.kw, self.kh, self.p, self.metric,
                                         out=self.tensor, lmap=self.maps[b], tmpl_dev=self.tmpl_dev,
                                         stream=self.compute)
                self.consumed[b].record(self.compute)
                self.done[b].record(self.compute)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.done[b])
                host_maps[i].copy_(self.maps[b], non_blocking=True)
                self.drained[b].record(self.d2h)
        self.d2h.synchronize()

    @staticmethod
    def pinned_frames(frames: list[np.ndarray]) -> list[torch.Tensor]:
        return [torch.from_numpy(np.ascontiguousarray(f, dtype=np.uint8)).pin_memory() for f in frames]

    def pinned_maps(self, n: int) -> list[torch.Tensor]:
        return [torch.empty((self.h, self.w), dtype=torch.float64).pin_memory() for _ in range(n)]
