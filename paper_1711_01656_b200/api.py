"""Python mirror of the reference interface for the hot path, on the C-ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/spct/{imagecore,integral,likelihood}.hpp):

    to_grayscale(r, g, b)                         imagecore.hpp:95
    quantize(img, bins, lo=0.0, hi=256.0)         imagecore.hpp:99-100
    build_integral_histogram(bm, schedule, budget) integral.hpp:98-100
    region_histogram(t, rect) / region_count(...)  integral.hpp:111-114
    schedule_stats / estimate_memory              integral.hpp:122,130
    hist_distance_map(t, tmpl, kw, kh, p=1.0)     likelihood.hpp:59-61

plus the B200 additions (bin slabs, fused build+match, partial maps for the
multi-GPU reduce).  torch provides device memory and streams only; every
computation is a kernel in libspct_b200.so.  Contract violations raise
``ContractError`` (a ValueError) exactly where the reference throws
``spct::contract_error``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi as A
from ._capi import ContractError, check

DEFAULT_BUDGET = 2 << 30  # kDefaultMemoryBudget (integral.hpp:96)

SCHEDULES = {"sequential": 0, "seq": 0, "sts": 1, "scan-transpose-scan": 1, "cw-tis": 2, "crossweave": 2,
             "wf-tis": 3, "wavefront": 3}


@dataclass
class ScanSchedule:
    """integral.hpp:31-35; every kind gives identical bits on the device."""
    kind: int = A.SCHED_SEQUENTIAL
    tile: int = 32
    threads: int = 1


def schedule_from_string(s: str) -> int:
    if s not in SCHEDULES:
        raise ContractError(A.SPCT_ERR_CONTRACT, f"unknown schedule '{s}'")
    return SCHEDULES[s]


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(a, dtype: torch.dtype) -> torch.Tensor:
    """Device tensor for a numpy array / torch tensor (no copy when already on device)."""
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.cuda(non_blocking=True)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    if dtype == torch.uint8:
        arr = arr.astype(np.uint8, copy=False)
        return torch.from_numpy(arr).cuda()
    if dtype == torch.int16:  # uint16 payload
        arr = arr.astype(np.uint16, copy=False)
        return torch.from_numpy(arr.view(np.int16)).cuda()
    if dtype == torch.float64:
        return torch.from_numpy(arr.astype(np.float64, copy=False)).cuda()
    raise TypeError(dtype)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _source(kind: int, planes, width: int, height: int, nbins: int, lo: float = 0.0, hi: float = 256.0,
            pitch: int | None = None) -> A.spct_source:
    s = A.spct_source()
    s.kind = kind
    for i, p in enumerate(planes):
        s.plane[i] = _ptr(p)
    s.pitch = width if pitch is None else pitch
    s.width, s.height, s.nbins = width, height, nbins
    s.lo, s.hi = lo, hi
    return s


# ------------------------------------------------------------------ imagecore

def to_grayscale(r, g, b, stream=None) -> torch.Tensor:
    """imagecore.cpp:17-24 on the device; returns a (h, w) uint8 device tensor."""
    r, g, b = (_dev(x, torch.uint8) for x in (r, g, b))
    out = torch.empty_like(r)
    check(A.lib().spct_cu_to_grayscale(_ptr(r), _ptr(g), _ptr(b), r.numel(), _ptr(out), _stream(stream)))
    return out


def quantize(img, bins: int, lo: float = 0.0, hi: float = 256.0, stream=None) -> torch.Tensor:
    """imagecore.cpp:28-53: uint8 gray (or float64 scalar map) -> uint16 bins (device int16 view)."""
    is_f = (isinstance(img, np.ndarray) and img.dtype != np.uint8) or (
        isinstance(img, torch.Tensor) and img.dtype != torch.uint8)
    x = _dev(img, torch.float64 if is_f else torch.uint8)
    if x.dim() != 2 or x.numel() == 0:
        raise ContractError(A.SPCT_ERR_CONTRACT, "quantize: empty image")
    h, w = x.shape
    out = torch.empty((h, w), dtype=torch.int16, device=x.device)
    src = _source(A.SRC_SCALAR_F64 if is_f else A.SRC_GRAY_U8, [x], w, h, bins, lo, hi)
    check(A.lib().spct_cu_quantize(C.byref(src), _ptr(out), _stream(stream)))
    return out


def orientation_bins(gray, bins: int, sigma: float = 1.0, stream=None) -> torch.Tensor:
    """Gradient-orientation BinMap of a gray uint8 frame (features.cpp:200-203 orientation,
    phog.cpp:15-20 orientation_bin): device int16 tensor carrying uint16 bins, usable as a
    BinMap source of build_integral_histogram / build_and_match (tracking batch, config 5)."""
    g = _dev(gray, torch.uint8)
    if g.dim() != 2 or g.numel() == 0:
        raise ContractError(A.SPCT_ERR_CONTRACT, "gradient_maps: empty image")
    h, w = g.shape
    out = torch.empty((h, w), dtype=torch.int16, device=g.device)
    ws = C.c_size_t()
    check(A.lib().spct_cu_orientation_workspace(w, h, C.byref(ws)))
    wbuf = _WS_ORIENT.get(ws.value, g.device, stream)
    check(A.lib().spct_cu_orientation_bins(_ptr(g), w, w, h, float(sigma), int(bins), _ptr(out), w, _ptr(wbuf),
                                           wbuf.numel(), _stream(stream)))
    return out


def as_numpy_u16(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


# ------------------------------------------------------------------ tensor

class IntegralHistogramTensor:
    """Device-resident integral histogram (integral.hpp:78-93 semantics).

    ``bins`` planes of global bins [bin0, bin0 + bins) out of ``nbins_total``.  Cell
    (k, y, x) in reference (padded) indexing is ``at(k, y, x)``; ``storage`` is the
    uint32 HBM buffer in the unpadded pitched layout of include/spct_cuda.h.
    """

    def __init__(self, width: int, height: int, nbins_total: int, bin0: int = 0, bins: int | None = None,
                 device=None, store: bool = True):
        bins = nbins_total - bin0 if bins is None else bins
        rp, pp, nbytes = C.c_int64(), C.c_int64(), C.c_uint64()
        check(A.lib().spct_cu_ih_layout(width, height, bins, C.byref(rp), C.byref(pp), C.byref(nbytes)))
        self.width, self.height, self.bins, self.bin0, self.nbins_total = width, height, bins, bin0, nbins_total
        self.row_pitch, self.plane_pitch = rp.value, pp.value
        # store=False: a descriptor without cells, for the fused sweeps' map-only form
        self.storage = torch.empty(nbytes.value // 4 if store else 0, dtype=torch.int32, device=device or "cuda")
        self.desc = A.spct_ih(self.storage.data_ptr() if store else None, bins, bin0, nbins_total, height, width,
                              rp.value, pp.value)
        # (spct_source, keep-alive device tensors) of the frame the tensor was built from, if any:
        # window statistics can then be recomputed from 1 B/px instead of re-reading the tensor
        self.source = None

    def planes(self) -> torch.Tensor:
        """(bins, height, row_pitch) int32 view of the unpadded device cells."""
        return self.storage.view(self.bins, self.height, self.row_pitch)

    def padded_u64(self, k0: int = 0, k1: int | None = None, stream=None) -> np.ndarray:
        """Reference layout (integral.hpp:78-93) of planes [k0, k1): uint64, zero padding."""
        k1 = self.bins if k1 is None else k1
        out = torch.empty((k1 - k0) * (self.height + 1) * (self.width + 1), dtype=torch.int64,
                          device=self.storage.device)
        check(A.lib().spct_cu_ih_export_u64(C.byref(self.desc), k0, k1, _ptr(out), _stream(stream)))
        return out.cpu().numpy().view(np.uint64).reshape(k1 - k0, self.height + 1, self.width + 1)

    def at(self, k: int, y: int, x: int) -> int:
        if y == 0 or x == 0:
            return 0
        return int(self.planes()[k, y - 1, x - 1].item()) & 0xFFFFFFFF

    def plane_stride(self) -> int:
        return (self.height + 1) * (self.width + 1)

    def row_stride(self) -> int:
        return self.width + 1


def dump_tensor(t: IntegralHistogramTensor, path: str, elem_bytes: int = 8, stream=None) -> None:
    """integral.cpp:619-633: the IHT1 file of ``t`` (elem_bytes 8 = the reference format;
    4 = half-size extension the reference loader rejects).  Raises IOError-like SpctError
    (status 3) where the reference throws io_error."""
    check(A.lib().spct_cu_ih_dump(C.byref(t.desc), str(path).encode(), int(elem_bytes), _stream(stream)))


def load_tensor(path: str, device=None, stream=None):
    """integral.cpp:635-659: an IHT1 file (elem 8, or 4) into a new device tensor.  A file
    whose cells exceed 2^32 (a dumped weighted tensor) comes back as a swih.WeightedTensor
    with uint64 cells, as the reference's load_tensor keeps them."""
    b, h, w, e = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    check(A.lib().spct_cu_ih_load_header(str(path).encode(), C.byref(b), C.byref(h), C.byref(w), C.byref(e)))
    t = IntegralHistogramTensor(w.value, h.value, b.value, device=device)
    st = A.lib().spct_cu_ih_load(str(path).encode(), C.byref(t.desc), _stream(stream))
    if (st == A.SPCT_ERR_IO and e.value == 8 and
            A.lib().spct_cu_last_error().startswith(b"tensor value exceeds the uint32 device cell")):
        from .swih import WeightedTensor

        pad = np.fromfile(str(path), dtype="<u8", offset=20, count=b.value * (h.value + 1) * (w.value + 1))
        if pad.size != b.value * (h.value + 1) * (w.value + 1):
            raise A.SpctError(A.SPCT_ERR_IO, f"truncated tensor payload: {path}")  # integral.cpp:655
        wt = WeightedTensor(w.value, h.value, b.value, device=t.storage.device)
        cells = pad.reshape(b.value, h.value + 1, w.value + 1)[:, 1:, 1:].view(np.int64)
        view = wt.storage[:b.value * wt.desc.plane_pitch].view(b.value, h.value, wt.desc.row_pitch)
        view[:, :, :w.value].copy_(torch.from_numpy(np.ascontiguousarray(cells)))
        return wt
    check(st)
    return t


def estimate_memory(w: int, h: int, bins: int, elem_bytes: int):
    pad, raw, deg = C.c_uint64(), C.c_uint64(), C.c_int()
    check(A.lib().spct_cu_estimate_memory(w, h, bins, elem_bytes, C.byref(pad), C.byref(raw), C.byref(deg)))
    return pad.value, raw.value, bool(deg.value)


def schedule_stats(w: int, h: int, tile: int, scan_len: int):
    it, tl, ef = C.c_longlong(), C.c_longlong(), C.c_double()
    check(A.lib().spct_cu_schedule_stats(w, h, tile, scan_len, C.byref(it), C.byref(tl), C.byref(ef)))
    return it.value, tl.value, ef.value


def _validate_schedule(schedule: ScanSchedule | None):
    s = schedule or ScanSchedule()
    if not (2 <= s.tile <= 4096):
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: tile must be in [2, 4096]")  # integral.cpp:511
    if not (1 <= s.threads <= 64):
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: threads must be in [1, 64]")  # :512-513


def _check_budget(w, h, bins, budget):
    pad, _, _ = estimate_memory(w, h, bins, 8)  # integral.cpp:330-335 counts 8-byte cells
    if pad > budget:
        raise ContractError(A.SPCT_ERR_CONTRACT,
                            f"tensor of {pad} bytes exceeds the memory budget of {budget}")


class Workspace:
    """Reusable device scratch (carry tables), one buffer per device.  The buffer handed out
    is recorded on the stream that will use it, so the caching allocator keeps a replaced
    (smaller) buffer alive until work already queued on that stream has finished."""

    def __init__(self):
        self.bufs = {}

    def get(self, nbytes: int, device, stream=None) -> torch.Tensor:
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        buf = self.bufs.get(idx)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=torch.device("cuda", idx))
            self.bufs[idx] = buf
        s = stream if stream is not None else torch.cuda.current_stream(idx)
        if s != torch.cuda.default_stream(idx):
            buf.record_stream(s)
        return buf


_WS = Workspace()
_WS_ORIENT = Workspace()
_WS_SIDE = Workspace()  # the orientation branch of a tracking-batch frame (channels.py)


def frame_source(frame, nbins: int, lo: float = 0.0, hi: float = 256.0):
    """(spct_source, keep-alive tensors) for a gray uint8 frame, planar RGB tuple,
    uint16 BinMap or float64 scalar map (numpy or torch)."""
    if isinstance(frame, (tuple, list)):
        planes = [_dev(p, torch.uint8) for p in frame]
        h, w = planes[0].shape
        return _source(A.SRC_RGB_U8, planes, w, h, nbins, lo, hi), planes
    is_t = isinstance(frame, torch.Tensor)
    dt = frame.dtype
    if (is_t and dt == torch.uint8) or (not is_t and dt == np.uint8):
        x = _dev(frame, torch.uint8)
        kind = A.SRC_GRAY_U8
    elif (is_t and dt == torch.int16) or (not is_t and dt == np.uint16):
        x = _dev(frame, torch.int16)
        kind = A.SRC_BINS_U16
    else:
        x = _dev(frame, torch.float64)
        kind = A.SRC_SCALAR_F64
    if x.dim() != 2 or x.numel() == 0:
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: empty bin map")
    h, w = x.shape
    return _source(kind, [x], w, h, nbins, lo, hi), [x]


def build_integral_histogram(bm, nbins: int | None = None, schedule: ScanSchedule | None = None,
                             memory_budget: int = DEFAULT_BUDGET, *, lo: float = 0.0, hi: float = 256.0,
                             bin0: int = 0, bins: int | None = None, validate: bool = True,
                             out: IntegralHistogramTensor | None = None, stream=None) -> IntegralHistogramTensor:
    """integral.cpp:548-551.  ``bm`` is a uint16 BinMap (nbins required), or a frame that
    the fused load stage quantises (gray uint8 / RGB tuple / float64 with lo, hi).
    ``bin0``/``bins`` select a bin slab (multi-GPU sharding)."""
    _validate_schedule(schedule)
    if nbins is None:
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: bins must be >= 1")
    src, keep = frame_source(bm, nbins, lo, hi)
    if nbins < 1:
        raise ContractError(A.SPCT_ERR_CONTRACT, "build: bins must be >= 1")
    if validate and src.kind == A.SRC_BINS_U16:  # integral.cpp:337-343
        mx = C.c_int()
        check(A.lib().spct_cu_binmap_max(_ptr(keep[0]), src.pitch, src.width, src.height, C.byref(mx),
                                         _stream(stream)))
        if mx.value >= nbins:
            raise ContractError(A.SPCT_ERR_CONTRACT, "build: bin index out of range")
    if memory_budget is not None:
        _check_budget(src.width, src.height, nbins, memory_budget)
    t = out or IntegralHistogramTensor(src.width, src.height, nbins, bin0, bins, device=keep[0].device)
    ws = C.c_size_t()
    check(A.lib().spct_cu_ih_build_workspace(C.byref(src), t.bin0, t.bins, C.byref(ws)))
    wbuf = _WS.get(ws.value, keep[0].device, stream)
    check(A.lib().spct_cu_ih_build(C.byref(src), C.byref(t.desc), _ptr(wbuf), wbuf.numel(), _stream(stream)))
    if isinstance(bm, torch.Tensor) and bm.is_cuda:  # caller-owned device memory: keep a private copy
        keep = [k.clone() for k in keep]
        for i, k in enumerate(keep):
            src.plane[i] = _ptr(k)
    t.source = (src, keep)
    return t


def region_histograms(t: IntegralHistogramTensor, rects, stream=None) -> np.ndarray:
    """Batched region_histogram: rects (n, 4) {x, y, w, h} -> (n, bins) uint64."""
    r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1, 4))
    for x, y, w, h in r:
        if not (w >= 0 and h >= 0):
            raise ContractError(A.SPCT_ERR_CONTRACT, "region_histogram: negative extent")
        if not (x >= 0 and y >= 0 and x + w <= t.width and y + h <= t.height):
            raise ContractError(A.SPCT_ERR_CONTRACT, "region_histogram: rect outside image")
    n = r.shape[0]
    if n == 0:
        return np.zeros((0, t.bins), np.uint64)
    dr = torch.from_numpy(r).cuda()
    out = torch.empty(n * t.bins, dtype=torch.int32, device=dr.device)
    check(A.lib().spct_cu_region_counts(C.byref(t.desc), _ptr(dr), n, _ptr(out), _stream(stream)))
    return out.cpu().numpy().view(np.uint32).astype(np.uint64).reshape(n, t.bins)


def region_histogram(t: IntegralHistogramTensor, x: int, y: int, w: int, h: int) -> np.ndarray:
    return region_histograms(t, [[x, y, w, h]])[0]


def region_count(t: IntegralHistogramTensor, k: int, x: int, y: int, w: int, h: int) -> int:
    if not (0 <= k < t.bins):
        raise ContractError(A.SPCT_ERR_CONTRACT, "region_count: bin out of range")
    if not (x >= 0 and y >= 0 and w >= 0 and h >= 0 and x + w <= t.width and y + h <= t.height):
        raise ContractError(A.SPCT_ERR_CONTRACT, "region_count: rect outside image")
    return int(region_histogram(t, x, y, w, h)[k])


# ------------------------------------------------------------------ likelihood

def _tmpl(tmpl, nbins: int, width: int, height: int, kw: int, kh: int, p: float):
    th = np.ascontiguousarray(np.asarray(tmpl, dtype=np.float64).reshape(-1))
    check(A.lib().spct_cu_hist_check(nbins, width, height, th.ctypes.data_as(C.POINTER(C.c_double)), th.size,
                                     kw, kh, p))
    return torch.from_numpy(th).cuda()


def hist_match_map(t: IntegralHistogramTensor, tmpl, kw: int, kh: int, p: float = 1.0,
                   metric: int = A.METRIC_MINKOWSKI, stream=None, exact: bool = False) -> torch.Tensor:
    """likelihood.cpp:193-225 (metric MINKOWSKI) -> (height, width) float64 device map.

    A tensor built by this library remembers its source frame, and the map is then
    recomputed by the fused sweep from 1 B/px (no tensor re-read).  A tensor without a
    source (e.g. loaded from an IHT1 file) is read once: the device recovers and checks
    every pixel's bin, then runs the same sweep (tensor_match.cu); a tensor that is not the
    integral histogram of a bin map gets the reference's arithmetic with actual window
    totals.  Both are bit-identical to the reference for p = 1 with an integral template and
    a power-of-two kw*kh, within the 1e-5 map tolerance otherwise.  ``exact=True`` reads
    the tensor with the reference's operation order (bit-identical for p = 1)."""
    dt = _tmpl(tmpl, t.bins, t.width, t.height, kw, kh, p)
    out = torch.empty((t.height, t.width), dtype=torch.float64, device=dt.device)
    if (not exact and t.source is not None and t.bin0 == 0 and t.bins == t.nbins_total
            and A.lib().spct_cu_fused_window_ok(kw, kh)):
        src, _keep = t.source
        nodata = A.spct_ih(None, t.bins, t.bin0, t.nbins_total, t.height, t.width, t.row_pitch, t.plane_pitch)
        ws = C.c_size_t()
        check(A.lib().spct_cu_ih_build_workspace(C.byref(src), 0, t.bins, C.byref(ws)))
        wbuf = _WS.get(ws.value, dt.device, stream)
        check(A.lib().spct_cu_ih_build_match_map(C.byref(src), C.byref(nodata), _ptr(dt), kw, kh, p, metric,
                                                 _ptr(out), _ptr(wbuf), wbuf.numel(), _stream(stream)))
        return out
    fn = A.lib().spct_cu_hist_match_exact if exact else A.lib().spct_cu_hist_match
    check(fn(C.byref(t.desc), _ptr(dt), kw, kh, p, metric, _ptr(out), _stream(stream)))
    return out


def hist_distance_map(t: IntegralHistogramTensor, tmpl, kw: int, kh: int, p: float = 1.0, stream=None,
                      exact: bool = False):
    return hist_match_map(t, tmpl, kw, kh, p, A.METRIC_MINKOWSKI, stream, exact)


def hist_partial(t: IntegralHistogramTensor, tmpl_dev: torch.Tensor, kw: int, kh: int, p: float = 1.0,
                 metric: int = A.METRIC_MINKOWSKI, out: torch.Tensor | None = None, accumulate: bool = False,
                 stream=None) -> torch.Tensor:
    """Slab partial of the window statistic over the valid grid ((h-kh+1), (w-kw+1))."""
    nu, nv = t.width - kw + 1, t.height - kh + 1
    if out is None:
        out = torch.empty((max(nv, 0), max(nu, 0)), dtype=torch.float64, device=tmpl_dev.device)
    check(A.lib().spct_cu_hist_partial(C.byref(t.desc), _ptr(tmpl_dev), kw, kh, p, metric, _ptr(out),
                                       int(accumulate), _stream(stream)))
    return out


def hist_finalize(partial: torch.Tensor, width: int, height: int, kw: int, kh: int, p: float = 1.0,
                  metric: int = A.METRIC_MINKOWSKI, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    if out is None:
        out = torch.empty((height, width), dtype=torch.float64, device=partial.device)
    check(A.lib().spct_cu_hist_finalize(_ptr(partial), width, height, kw, kh, p, metric, _ptr(out),
                                        _stream(stream)))
    return out


def build_and_match(frame, nbins: int, tmpl, kw: int, kh: int, p: float = 1.0, metric: int = A.METRIC_MINKOWSKI,
                    *, lo: float = 0.0, hi: float = 256.0, bin0: int = 0, bins: int | None = None,
                    out: IntegralHistogramTensor | None = None, partial: torch.Tensor | None = None,
                    tmpl_dev: torch.Tensor | None = None, stream=None):
    """Fused quantise -> build -> partial window statistic for slab [bin0, bin0+bins).
    Returns (tensor, partial).  Summing partials of every slab and calling
    hist_finalize gives hist_distance_map of the full histogram."""
    src, keep = frame_source(frame, nbins, lo, hi)
    if tmpl_dev is None:
        tmpl_dev = _tmpl(tmpl, nbins, src.width, src.height, kw, kh, p)
    t = out or IntegralHistogramTensor(src.width, src.height, nbins, bin0, bins, device=keep[0].device)
    nu, nv = src.width - kw + 1, src.height - kh + 1
    if partial is None:
        partial = torch.empty((nv, nu), dtype=torch.float64, device=keep[0].device)
    ws = C.c_size_t()
    check(A.lib().spct_cu_ih_build_workspace(C.byref(src), t.bin0, t.bins, C.byref(ws)))
    wbuf = _WS.get(ws.value, keep[0].device, stream)
    check(A.lib().spct_cu_ih_build_match(C.byref(src), C.byref(t.desc), _ptr(tmpl_dev), kw, kh, p, metric,
                                         _ptr(partial), _ptr(wbuf), wbuf.numel(), _stream(stream)))
    return t, partial


def build_and_match_map_multi(frames, nbins: int, tmpl_devs, kw: int, kh: int, p: float = 1.0,
                              metric: int = A.METRIC_MINKOWSKI, *, outs, lmaps, stream=None):
    """build_and_match_map for several same-shape sources (the channels of a tracking batch)
    in one call: the carry tables and template preps of all of them in one launch per
    kernel, then one sweep each (spct_cu_ih_build_match_map_multi).  ``tmpl_devs``,
    ``outs`` and ``lmaps`` are per-source device templates, tensors and maps."""
    n = len(frames)
    srcs, keeps, need = (A.spct_source * n)(), [], 0
    for i, f in enumerate(frames):
        src, keep = frame_source(f, nbins)
        srcs[i] = src
        keeps.append(keep)
        ws = C.c_size_t()
        check(A.lib().spct_cu_ih_build_workspace(C.byref(src), outs[i].bin0, outs[i].bins, C.byref(ws)))
        need = max(need, (ws.value + 255) // 256 * 256)
    ihs = (A.spct_ih * n)(*[o.desc for o in outs])
    wbuf = _WS.get(need * n, keeps[0][0].device, stream)
    base = wbuf.data_ptr()
    vp = C.c_void_p * n
    check(A.lib().spct_cu_ih_build_match_map_multi(n, srcs, ihs, vp(*[t.data_ptr() for t in tmpl_devs]), kw, kh, p,
                                                   metric, vp(*[m.data_ptr() for m in lmaps]),
                                                   vp(*[base + i * need for i in range(n)]), need, _stream(stream)))
    return outs, lmaps


def build_and_match_map(frame, nbins: int, tmpl, kw: int, kh: int, p: float = 1.0,
                        metric: int = A.METRIC_MINKOWSKI, *, lo: float = 0.0, hi: float = 256.0,
                        out: IntegralHistogramTensor | None = None, lmap: torch.Tensor | None = None,
                        tmpl_dev: torch.Tensor | None = None, stream=None, workspace: "Workspace | None" = None):
    """Fused quantise -> build -> finished likelihood map (every bin on this device):
    build_integral_histogram + hist_distance_map (spct_main.cpp:332-333) in one pass.
    Returns (tensor, map).  ``out.desc.data = None`` skips storing the tensor.  Calls that
    may run concurrently on different streams need different ``workspace`` caches."""
    src, keep = frame_source(frame, nbins, lo, hi)
    if tmpl_dev is None:
        tmpl_dev = _tmpl(tmpl, nbins, src.width, src.height, kw, kh, p)
    t = out or IntegralHistogramTensor(src.width, src.height, nbins, device=keep[0].device)
    if lmap is None:
        lmap = torch.empty((src.height, src.width), dtype=torch.float64, device=keep[0].device)
    ws = C.c_size_t()
    check(A.lib().spct_cu_ih_build_workspace(C.byref(src), t.bin0, t.bins, C.byref(ws)))
    wbuf = (workspace or _WS).get(ws.value, keep[0].device, stream)
    check(A.lib().spct_cu_ih_build_match_map(C.byref(src), C.byref(t.desc), _ptr(tmpl_dev), kw, kh, p, metric,
                                             _ptr(lmap), _ptr(wbuf), wbuf.numel(), _stream(stream)))
    return t, lmap
