"""Multi-feature likelihood maps of a tracking batch (BASELINE config 5).

Per frame and per feature channel — intensity (to_grayscale of the RGB frame),
gradient orientation (features.cpp:200-203 + phog.cpp:15-20), and the R, G, B planes —
one fused quantise -> integral histogram -> sliding-window likelihood map
(build_integral_histogram + hist_distance_map, spct_main.cpp:332-333) against that
channel's template histogram.  The reference computes these channels one at a time on
the CPU (track_loop.cpp's channel fan-out); here each channel is one fused sweep on the
device, and frames stream through pinned host buffers.
"""
from __future__ import annotations

import torch

from . import api as _api
from ._capi import METRIC_MINKOWSKI

CHANNELS = ("intensity", "orientation", "red", "green", "blue")


def channel_sources(r, g, b, nbins: int, sigma: float = 1.0, stream=None) -> dict:
    """Device sources of the five channels: the gray frame (to_grayscale, quantised in the
    sweep's load stage: quantize(to_grayscale(rgb)) exactly), the orientation BinMap of
    the gray frame, and the single R, G, B planes."""
    rd, gd, bd = (_api._dev(p, torch.uint8) for p in (r, g, b))
    gray = _api.to_grayscale(rd, gd, bd, stream=stream)
    return {"intensity": gray, "orientation": _api.orientation_bins(gray, nbins, sigma, stream=stream),
            "red": rd, "green": gd, "blue": bd}


def likelihood_channels(r, g, b, nbins: int, templates: dict, kw: int, kh: int, p: float = 1.0,
                        metric: int = METRIC_MINKOWSKI, sigma: float = 1.0, tensors: dict | None = None,
                        maps: dict | None = None, tmpl_dev: dict | None = None, stream=None) -> dict:
    """{channel: (height, width) float64 device map} for one RGB frame.  ``templates`` maps
    each channel to its normalised template histogram (nbins values); ``tensors`` /
    ``maps`` / ``tmpl_dev`` may hold preallocated per-channel outputs for a batch."""
    rd, gd, bd = (_api._dev(x, torch.uint8) for x in (r, g, b))
    dev = rd.device
    h, w = rd.shape
    main = stream if stream is not None else torch.cuda.current_stream(dev)
    ts = {c: tensors[c] if tensors else _api.IntegralHistogramTensor(w, h, nbins, device=dev) for c in CHANNELS}
    ms = {c: maps[c] if maps else torch.empty((h, w), dtype=torch.float64, device=dev) for c in CHANNELS}
    tds = {c: tmpl_dev[c] if tmpl_dev else _api._tmpl(templates[c], nbins, w, h, kw, kh, p).to(dev) for c in CHANNELS}
    gray = _api.to_grayscale(rd, gd, bd, stream=main)
    # the orientation channel (gradient + bins, then its map) branches off on a side stream
    # and overlaps the four plane channels, which share one launch of each carry kernel,
    # of the template prep and of the sweep per source kind (build_and_match_map_multi)
    side = _side_stream(dev)
    fork = torch.cuda.Event()
    fork.record(main)
    side.wait_event(fork)
    gray.record_stream(side)
    with torch.cuda.stream(side):
        ob = _api.orientation_bins(gray, nbins, sigma, stream=side)
        _api.build_and_match_map(ob, nbins, None, kw, kh, p, metric, out=ts["orientation"], lmap=ms["orientation"],
                                 tmpl_dev=tds["orientation"], stream=side, workspace=_api._WS_SIDE)
    planes = {"intensity": gray, "red": rd, "green": gd, "blue": bd}
    pc = [c for c in CHANNELS if c != "orientation"]
    _api.build_and_match_map_multi([planes[c] for c in pc], nbins, [tds[c] for c in pc], kw, kh, p, metric,
                                   outs=[ts[c] for c in pc], lmaps=[ms[c] for c in pc], stream=main)
    join = torch.cuda.Event()
    join.record(side)
    main.wait_event(join)
    return {c: ms[c] for c in CHANNELS}


_SIDE: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _SIDE:
        _SIDE[idx] = torch.cuda.Stream(torch.device("cuda", idx))
    return _SIDE[idx]


class ChannelGraph:
    """One frame's five-channel maps captured as a CUDA graph (the per-frame work is ~30
    small launches; replaying a graph removes their host launch cost).  Frames are copied
    into static device buffers, then the graph replays; `maps` / `tensors` are the static
    outputs, overwritten by every run()."""

    def __init__(self, side_w: int, side_h: int, nbins: int, tmpl_dev: dict, kw: int, kh: int, p: float = 1.0,
                 metric: int = METRIC_MINKOWSKI, sigma: float = 1.0, device=None):
        dev = torch.device(device or "cuda")
        self.rgb = torch.zeros((3, side_h, side_w), dtype=torch.uint8, device=dev)
        self.tensors = {c: _api.IntegralHistogramTensor(side_w, side_h, nbins, device=dev) for c in CHANNELS}
        self.maps = {c: torch.empty((side_h, side_w), dtype=torch.float64, device=dev) for c in CHANNELS}
        args = (nbins, None, kw, kh, p, metric, sigma)

        def body():
            likelihood_channels(self.rgb[0], self.rgb[1], self.rgb[2], *args, tensors=self.tensors, maps=self.maps,
                                tmpl_dev=tmpl_dev)

        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            body()  # warm-up outside the capture: one-time kernel attributes, workspaces
        torch.cuda.current_stream(dev).wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            body()

    def run(self, r, g, b) -> dict:
        self.rgb[0].copy_(r, non_blocking=True)
        self.rgb[1].copy_(g, non_blocking=True)
        self.rgb[2].copy_(b, non_blocking=True)
        self.graph.replay()
        return self.maps
