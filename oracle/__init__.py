"""TEST INFRASTRUCTURE ONLY — ctypes/numpy front end of the CPU oracle.

Two back ends, both CPU-only and never imported by the product package
(`paper_1711_01656_b200`):

* ``C``   — oracle/libspct_oracle.so, the plain-C restatement (oracle/spct_oracle.c)
            plus the seeded fixture generators (oracle/fixtures.cpp);
* ``REF`` — oracle/_ref/libspct_ref.so, the unmodified reference library compiled
            from /root/reference/proj/src by oracle/Makefile (absent when the
            reference tree was not available at build time).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference)
may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libspct_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspct_ref.so")

# ScanScheduleKind (reference integral.hpp:21-26)
SEQUENTIAL, STS, CW_TIS, WF_TIS = 0, 1, 2, 3
# metric ids (shared with include/spct_cuda.h)
MINKOWSKI, INTERSECTION, BHATTACHARYYA, CHISQ = 0, 1, 2, 3
DEFAULT_BUDGET = 2 << 30  # kDefaultMemoryBudget, integral.hpp:96

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i, _u32, _u64, _i64, _d, _vp = C.c_int, C.c_uint32, C.c_uint64, C.c_int64, C.c_double, C.c_void_p


class ContractError(ValueError):
    """Oracle-side contract violation (status 2), mirrors spct::contract_error."""


class RefIOError(OSError):
    """Status 3, mirrors spct::io_error."""


def _check(st: int, what: str, lib=None):
    if st == 0:
        return
    msg = what
    if lib is not None and hasattr(lib, "ref_last_error"):
        msg += ": " + lib.ref_last_error().decode()
    if st == 2:
        raise ContractError(msg)
    if st == 3:
        raise RefIOError(msg)
    raise RuntimeError(f"{msg} (status {st})")


def _load_c():
    lib = C.CDLL(ORACLE_SO)
    sig = {
        "or_to_grayscale": (None, [_u8p, _u8p, _u8p, _i64, _u8p]),
        "or_quantize_u8": (_i, [_u8p, _i, _i, _i, _d, _d, _u16p]),
        "or_quantize_f64": (_i, [_f64p, _i, _i, _i, _d, _d, _u16p]),
        "or_estimate_memory": (_i, [_i, _i, _i, _i, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_i)]),
        "or_schedule_stats": (_i, [_i, _i, _i, _i, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(_d)]),
        "or_ih_validate": (_i, [_u16p, _i, _i, _i, _i, _i, _u64]),
        "or_ih_build_u64": (None, [_u16p, _i, _i, _i, _i, _u64p]),
        "or_ih_build_u32": (None, [_u16p, _i, _i, _i, _i, _u32p]),
        "or_region_count": (_i, [_u64p, _i, _i, _i, _i, _i, _i, _i, _i, C.POINTER(_u64)]),
        "or_region_histogram": (_i, [_u64p, _i, _i, _i, _i, _i, _i, _i, _u64p]),
        "or_hist_check": (_i, [_i, _i, _i, _f64p, _i, _i, _i, _d]),
        "or_hist_match_map": (_i, [_u64p, _i, _i, _i, _f64p, _i, _i, _d, _i, _f64p]),
        "or_hist_match_map_direct": (_i, [_u16p, _i, _i, _i, _f64p, _i, _i, _d, _i, _f64p]),
        "or_hist_partial": (_i, [_u16p, _i, _i, _i, _f64p, _i, _i, _d, _i, _i, _f64p]),
        "or_hist_finalize": (_i, [_f64p, _i, _i, _i, _i, _d, _f64p]),
        "or_xorshift_image": (None, [_u32, _i64, _u8p]),
        "or_orientation_bins": (_i, [_u8p, _i, _i, _d, _i, _u16p]),
        "or_fuse_maps": (_i, [C.POINTER(_vp), _i, _vp, _i64, _f64p]),
        "or_weighted_ih_u64": (None, [_u16p, _u64p, _i, _i, _i, _u64p]),
        "or_swlh_fixed_brute": (_i, [_u16p, _i, _i, _i, _i, _i, _i, _i, _i64p]),
        "or_swlh_normalized": (_i, [_u16p, _i, _i, _i, _i, _i, _i, _i, _f64p]),
        "or_swlh_map": (_i, [_u16p, _i, _i, _i, _f64p, _i, _i, _f64p]),
        "or_median_bg_ih": (_i, [_u8p, _i, _i, _i, _i, _i, _i, _i, _u8p]),
        "or_median_bg_sort": (_i, [_u8p, _i, _i, _i, _u8p]),
        "or_find_peaks": (_i, [_f64p, _i, _i, _i32p, _i32p, _f64p, _i, C.POINTER(_i)]),
        "or_score_map": (_i, [_f64p, _i, _i, _i, _i, _i, _i, C.POINTER(_i)]),
        "or_camshift": (_i, [_f64p, _i, _i, _d, _d, _i, _i, _d, _i, C.POINTER(_d), C.POINTER(_d), C.POINTER(_i),
                             C.POINTER(_i)]),
        "fx_noise_image": (None, [_i, _i, _u32, _u8p]),
        "fx_smooth_image": (None, [_i, _i, _u32, _i, _u8p]),
        "fx_noise_color": (None, [_i, _i, _u32, _u8p, _u8p, _u8p]),
        "fx_random_binmap": (None, [_i, _i, _i, _u32, _u16p]),
        "fx_rng_new": (_vp, [_u32]),
        "fx_rng_free": (None, [_vp]),
        "fx_rng_next": (_u32, [_vp]),
        "fx_rng_uniform_int": (_i, [_vp, _i, _i]),
        "fx_rng_binmap": (None, [_vp, _i, _i, _i, _u16p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


def _load_ref():
    if not os.path.exists(REF_SO):
        return None
    lib = C.CDLL(REF_SO)
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_to_grayscale": (_i, [_u8p, _u8p, _u8p, _i, _i, _u8p]),
        "ref_quantize_u8": (_i, [_u8p, _i, _i, _i, _d, _d, _u16p]),
        "ref_quantize_f64": (_i, [_f64p, _i, _i, _i, _d, _d, _u16p]),
        "ref_ih_build": (_i, [_u16p, _i, _i, _i, _i, _i, _i, _u64, C.POINTER(_vp)]),
        "ref_ih_free": (None, [_vp]),
        "ref_ih_data": (C.POINTER(_u64), [_vp]),
        "ref_ih_size": (_u64, [_vp]),
        "ref_region_histogram": (_i, [_vp, _i, _i, _i, _i, _u64p]),
        "ref_region_count": (_i, [_vp, _i, _i, _i, _i, _i, C.POINTER(_u64)]),
        "ref_hist_distance_map": (_i, [_vp, _f64p, _i, _i, _i, _d, _f64p]),
        "ref_schedule_stats": (_i, [_i, _i, _i, _i, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.POINTER(_d)]),
        "ref_estimate_memory": (_i, [_i, _i, _i, _i, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_i)]),
        "ref_schedule_from_string": (_i, [C.c_char_p]),
        "ref_orientation_bins": (_i, [_u8p, _i, _i, _d, _i, _u16p]),
        "ref_dump_tensor": (_i, [_vp, C.c_char_p]),
        "ref_fuse_maps": (_i, [C.POINTER(_vp), _i, _vp, _i, _i, _i, _f64p]),
        "ref_swlh_query_fixed": (_i, [_u16p, _i, _i, _i, _i, _i, _i32p, _i, _i64p]),
        "ref_median_bg_ih": (_i, [_u8p, _i, _i, _i, _i, _i, _i, _i, _u8p]),
        "ref_median_bg_sort": (_i, [_u8p, _i, _i, _i, _u8p]),
        "ref_swlh_query": (_i, [_u16p, _i, _i, _i, _i, _i, _i32p, _i, _f64p]),
        "ref_brute_force_swlh_fixed": (_i, [_u16p, _i, _i, _i, _i, _i, _i, _i, _i64p]),
        "ref_ih_build_weighted": (_i, [_u16p, _u64p, _i, _i, _i, _i, _i, _i, _u64, C.POINTER(_vp)]),
        "ref_find_peaks": (_i, [_f64p, _i, _i, _i32p, _i32p, _f64p, _i32p, _i, C.POINTER(_i)]),
        "ref_score_map": (_i, [_f64p, _i, _i, _i, _i, _i, _i, C.POINTER(_i)]),
        "ref_load_tensor": (_i, [C.c_char_p, C.POINTER(_vp)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


_C = None
_REF = False  # False = not tried yet


def clib():
    global _C
    if _C is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle` (or __graft_entry__.build())")
        _C = _load_c()
    return _C


def reflib():
    """The compiled reference, or None when oracle/_ref was never built."""
    global _REF
    if _REF is False:
        _REF = _load_ref()
    return _REF


def have_ref() -> bool:
    return reflib() is not None


# ----------------------------------------------------------------- fixtures

def xorshift_image(w: int, h: int, seed: int = 1) -> np.ndarray:
    out = np.empty((h, w), np.uint8)
    clib().or_xorshift_image(seed, w * h, out.reshape(-1))
    return out


def noise_image(w: int, h: int, seed: int) -> np.ndarray:
    out = np.empty((h, w), np.uint8)
    clib().fx_noise_image(w, h, seed, out.reshape(-1))
    return out


def smooth_image(w: int, h: int, seed: int, blur_passes: int = 3) -> np.ndarray:
    out = np.empty((h, w), np.uint8)
    clib().fx_smooth_image(w, h, seed, blur_passes, out.reshape(-1))
    return out


def noise_color(w: int, h: int, seed: int):
    r, g, b = (np.empty((h, w), np.uint8) for _ in range(3))
    clib().fx_noise_color(w, h, seed, r.reshape(-1), g.reshape(-1), b.reshape(-1))
    return r, g, b


def random_binmap(w: int, h: int, bins: int, seed: int) -> np.ndarray:
    out = np.empty((h, w), np.uint16)
    clib().fx_random_binmap(w, h, bins, seed, out.reshape(-1))
    return out


class Rng:
    """std::mt19937 threaded through successive draws (acceptance.cpp style)."""

    def __init__(self, seed: int):
        self._h = clib().fx_rng_new(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            clib().fx_rng_free(self._h)
            self._h = None

    def __call__(self) -> int:
        return clib().fx_rng_next(self._h)

    def uniform_int(self, lo: int, hi: int) -> int:
        return clib().fx_rng_uniform_int(self._h, lo, hi)

    def binmap(self, w: int, h: int, bins: int) -> np.ndarray:
        out = np.empty((h, w), np.uint16)
        clib().fx_rng_binmap(self._h, w, h, bins, out.reshape(-1))
        return out


# ----------------------------------------------------------------- C restatement

def to_grayscale(r, g, b) -> np.ndarray:
    r, g, b = (np.ascontiguousarray(a, np.uint8) for a in (r, g, b))
    out = np.empty_like(r)
    clib().or_to_grayscale(r.reshape(-1), g.reshape(-1), b.reshape(-1), r.size, out.reshape(-1))
    return out


def quantize(img, bins: int, lo: float = 0.0, hi: float = 256.0) -> np.ndarray:
    img = np.ascontiguousarray(img)
    h, w = img.shape if img.ndim == 2 else (0, 0)
    out = np.empty((max(h, 0), max(w, 0)), np.uint16)
    if img.dtype == np.uint8:
        st = clib().or_quantize_u8(img.reshape(-1), w, h, bins, lo, hi, out.reshape(-1))
    else:
        img = np.ascontiguousarray(img, np.float64)
        st = clib().or_quantize_f64(img.reshape(-1), w, h, bins, lo, hi, out.reshape(-1))
    _check(st, "quantize")
    return out


def validate_build(bm: np.ndarray, nbins: int, tile: int = 32, threads: int = 1,
                   budget: int = DEFAULT_BUDGET) -> None:
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    _check(clib().or_ih_validate(bm.reshape(-1), w, h, nbins, tile, threads, budget), "build")


def build_ih(bm: np.ndarray, nbins: int, k0: int = 0, k1: int | None = None,
             dtype=np.uint64) -> np.ndarray:
    """Padded reference-layout tensor, shape (k1-k0, h+1, w+1)."""
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    k1 = nbins if k1 is None else k1
    out = np.empty((k1 - k0, h + 1, w + 1), dtype)
    if dtype == np.uint64:
        clib().or_ih_build_u64(bm.reshape(-1), w, h, k0, k1, out.reshape(-1))
    else:
        clib().or_ih_build_u32(bm.reshape(-1), w, h, k0, k1, out.reshape(-1))
    return out


def region_histogram(t: np.ndarray, x: int, y: int, w: int, h: int) -> np.ndarray:
    t = np.ascontiguousarray(t, np.uint64)
    b, hp, wp = t.shape
    out = np.empty(b, np.uint64)
    _check(clib().or_region_histogram(t.reshape(-1), b, wp - 1, hp - 1, x, y, w, h, out), "region_histogram")
    return out


def region_count(t: np.ndarray, k: int, x: int, y: int, w: int, h: int) -> int:
    t = np.ascontiguousarray(t, np.uint64)
    b, hp, wp = t.shape
    v = _u64(0)
    _check(clib().or_region_count(t.reshape(-1), b, wp - 1, hp - 1, k, x, y, w, h, C.byref(v)), "region_count")
    return int(v.value)


def hist_match_map(t: np.ndarray, tmpl, kw: int, kh: int, p: float = 1.0,
                   metric: int = MINKOWSKI) -> np.ndarray:
    t = np.ascontiguousarray(t, np.uint64)
    b, hp, wp = t.shape
    tmpl = np.ascontiguousarray(tmpl, np.float64)
    if tmpl.size != b:
        raise ContractError("hist_distance_map: template bin count mismatch")
    out = np.empty((hp - 1, wp - 1), np.float64)
    _check(clib().or_hist_match_map(t.reshape(-1), b, wp - 1, hp - 1, tmpl, kw, kh, p, metric,
                                    out.reshape(-1)), "hist_distance_map")
    return out


def hist_distance_map(t, tmpl, kw, kh, p=1.0):
    return hist_match_map(t, tmpl, kw, kh, p, MINKOWSKI)


def hist_match_map_direct(bm: np.ndarray, nbins: int, tmpl, kw: int, kh: int, p: float = 1.0,
                          metric: int = MINKOWSKI) -> np.ndarray:
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    tmpl = np.ascontiguousarray(tmpl, np.float64)
    if tmpl.size != nbins:
        raise ContractError("hist_distance_map: template bin count mismatch")
    out = np.empty((h, w), np.float64)
    _check(clib().or_hist_match_map_direct(bm.reshape(-1), nbins, w, h, tmpl, kw, kh, p, metric,
                                           out.reshape(-1)), "hist_distance_map")
    return out


def hist_partial(bm, nbins, tmpl, kw, kh, p, k0, k1) -> np.ndarray:
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    tmpl = np.ascontiguousarray(tmpl, np.float64)
    out = np.empty((h - kh + 1, w - kw + 1), np.float64)
    _check(clib().or_hist_partial(bm.reshape(-1), nbins, w, h, tmpl, kw, kh, p, k0, k1,
                                  out.reshape(-1)), "hist_partial")
    return out


def orientation_bins(gray: np.ndarray, bins: int, sigma: float = 1.0) -> np.ndarray:
    """Gradient-orientation BinMap (features.cpp:78-93 + phog.cpp:15-20), C restatement."""
    gray = np.ascontiguousarray(gray, np.uint8)
    h, w = gray.shape
    out = np.empty((h, w), np.uint16)
    _check(clib().or_orientation_bins(gray.reshape(-1), w, h, sigma, bins, out.reshape(-1)), "orientation_bins")
    return out


def ref_orientation_bins(gray: np.ndarray, bins: int, sigma: float = 1.0) -> np.ndarray:
    """The same through the unmodified reference (gradient_maps) — oracle/_ref."""
    gray = np.ascontiguousarray(gray, np.uint8)
    h, w = gray.shape
    out = np.empty((h, w), np.uint16)
    _check(reflib().ref_orientation_bins(gray.reshape(-1), w, h, sigma, bins, out.reshape(-1)), "orientation_bins",
           reflib())
    return out


def _ptrs(maps):
    arrs = [np.ascontiguousarray(m, np.float64) for m in maps]
    return arrs, (_vp * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])


def fuse_maps(maps, weights=None) -> np.ndarray:
    """likelihood.cpp:257-283 (C restatement)."""
    arrs, ptrs = _ptrs(maps)
    if not arrs:
        raise ContractError("fuse_maps: no maps to fuse")
    if any(a.shape != arrs[0].shape for a in arrs):
        raise ContractError("fuse_maps: map dimensions differ")
    if weights is not None and len(weights) != len(arrs):
        raise ContractError("fuse_maps: weight count mismatch")
    wv = None if weights is None else np.ascontiguousarray(weights, np.float64)
    out = np.empty(arrs[0].shape, np.float64)
    _check(clib().or_fuse_maps(ptrs, len(arrs), None if wv is None else wv.ctypes.data, arrs[0].size,
                               out.reshape(-1)), "fuse_maps")
    return out


def ref_fuse_maps(maps, weights=None) -> np.ndarray:
    arrs, ptrs = _ptrs(maps)
    wv = np.ascontiguousarray([] if weights is None else weights, np.float64)
    h, w = arrs[0].shape if arrs else (0, 0)
    out = np.empty((h, w), np.float64)
    _check(reflib().ref_fuse_maps(ptrs, len(arrs), wv.ctypes.data, wv.size, w, h, out.reshape(-1)), "fuse_maps",
           reflib())
    return out


def find_peaks(m: np.ndarray):
    """likelihood.cpp:285-322: (xs, ys, heights) sorted by height desc (rank = index + 1)."""
    m = np.ascontiguousarray(m, np.float64)
    h, w = m.shape
    xs, ys, hs = np.empty(w * h, np.int32), np.empty(w * h, np.int32), np.empty(w * h, np.float64)
    n = _i()
    _check(clib().or_find_peaks(m.reshape(-1), w, h, xs, ys, hs, w * h, C.byref(n)), "find_peaks")
    return xs[:n.value], ys[:n.value], hs[:n.value]


def ref_find_peaks(m: np.ndarray):
    m = np.ascontiguousarray(m, np.float64)
    h, w = m.shape
    xs, ys, hs, rk = (np.empty(w * h, np.int32), np.empty(w * h, np.int32), np.empty(w * h, np.float64),
                      np.empty(w * h, np.int32))
    n = _i()
    _check(reflib().ref_find_peaks(m.reshape(-1), w, h, xs, ys, hs, rk, w * h, C.byref(n)), "find_peaks", reflib())
    assert np.array_equal(rk[:n.value], np.arange(1, n.value + 1))
    return xs[:n.value], ys[:n.value], hs[:n.value]


def score_map(m: np.ndarray, gx: int, gy: int, gw: int, gh: int) -> int:
    m = np.ascontiguousarray(m, np.float64)
    h, w = m.shape
    r = _i()
    _check(clib().or_score_map(m.reshape(-1), w, h, gx, gy, gw, gh, C.byref(r)), "score_map")
    return r.value


def ref_score_map(m: np.ndarray, gx: int, gy: int, gw: int, gh: int) -> int:
    m = np.ascontiguousarray(m, np.float64)
    h, w = m.shape
    r = _i()
    _check(reflib().ref_score_map(m.reshape(-1), w, h, gx, gy, gw, gh, C.byref(r)), "score_map", reflib())
    return r.value


def camshift(m: np.ndarray, cx: float, cy: float, win_w: int, win_h: int, delta: float = 0.5, max_iter: int = 20):
    """tracker.cpp:77-113: (cx, cy, iterations, zero_mass)."""
    m = np.ascontiguousarray(m, np.float64)
    h, w = m.shape
    ox, oy, it, zm = _d(), _d(), _i(), _i()
    _check(clib().or_camshift(m.reshape(-1), w, h, cx, cy, win_w, win_h, delta, max_iter, C.byref(ox), C.byref(oy),
                              C.byref(it), C.byref(zm)), "camshift_refine")
    return ox.value, oy.value, it.value, bool(zm.value)


def weighted_ih(bm: np.ndarray, weights: np.ndarray, nbins: int) -> np.ndarray:
    """build_weighted_tensor (integral.cpp:553-559), reference layout uint64 (C restatement)."""
    bm = np.ascontiguousarray(bm, np.uint16)
    wt = np.ascontiguousarray(weights, np.uint64)
    h, w = bm.shape
    out = np.empty((nbins, h + 1, w + 1), np.uint64)
    clib().or_weighted_ih_u64(bm.reshape(-1), wt.reshape(-1), w, h, nbins, out.reshape(-1))
    return out


def ref_weighted_ih(bm: np.ndarray, weights: np.ndarray, nbins: int) -> np.ndarray:
    lib = reflib()
    bm = np.ascontiguousarray(bm, np.uint16)
    wt = np.ascontiguousarray(weights, np.uint64)
    h, w = bm.shape
    hdl = _vp()
    _check(lib.ref_ih_build_weighted(bm.reshape(-1), wt.reshape(-1), w, h, nbins, SEQUENTIAL, 32, 1, (1 << 64) - 1,
                                     C.byref(hdl)), "build_weighted_tensor", lib)
    try:
        n = int(lib.ref_ih_size(hdl))
        return np.ctypeslib.as_array(lib.ref_ih_data(hdl), shape=(n,)).reshape(nbins, h + 1, w + 1).copy()
    finally:
        lib.ref_ih_free(hdl)


def swlh_fixed(bm: np.ndarray, nbins: int, cx: int, cy: int, kw: int, kh: int) -> np.ndarray:
    """brute_force_swlh_fixed (swih.cpp:166-178), int64 16.16."""
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    out = np.empty(nbins, np.int64)
    _check(clib().or_swlh_fixed_brute(bm.reshape(-1), w, h, nbins, cx, cy, kw, kh, out), "swlh")
    return out


def swlh(bm: np.ndarray, nbins: int, cx: int, cy: int, kw: int, kh: int) -> np.ndarray:
    """brute_force_swlh (swih.cpp:199-202): normalised with the reference's long double."""
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    out = np.empty(nbins, np.float64)
    _check(clib().or_swlh_normalized(bm.reshape(-1), w, h, nbins, cx, cy, kw, kh, out), "swlh")
    return out


def swlh_map(bm: np.ndarray, nbins: int, model, kw: int, kh: int) -> np.ndarray:
    """The tracker's swlh-distance channel (track_loop.cpp:264-283)."""
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    md = np.ascontiguousarray(model, np.float64)
    out = np.empty((h, w), np.float64)
    _check(clib().or_swlh_map(bm.reshape(-1), w, h, nbins, md, kw, kh, out.reshape(-1)), "swlh_map")
    return out


def ref_swlh_query_fixed(bm, nbins, centres, kw, kh) -> np.ndarray:
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    c = np.ascontiguousarray(np.asarray(centres, np.int32).reshape(-1, 2))
    out = np.empty((len(c), nbins), np.int64)
    _check(reflib().ref_swlh_query_fixed(bm.reshape(-1), w, h, nbins, kw, kh, c.reshape(-1), len(c),
                                         out.reshape(-1)), "swlh_query_fixed", reflib())
    return out


def ref_swlh_query(bm, nbins, centres, kw, kh) -> np.ndarray:
    bm = np.ascontiguousarray(bm, np.uint16)
    h, w = bm.shape
    c = np.ascontiguousarray(np.asarray(centres, np.int32).reshape(-1, 2))
    out = np.empty((len(c), nbins), np.float64)
    _check(reflib().ref_swlh_query(bm.reshape(-1), w, h, nbins, kw, kh, c.reshape(-1), len(c), out.reshape(-1)),
           "swlh_query", reflib())
    return out


def median_bg_ih(frames, nf: int, bins: int, m: int, n: int, ref: bool = False) -> np.ndarray:
    """MedianBackgroundIH on frames[:nf], slid through frames[nf:], background()."""
    fr = np.ascontiguousarray(np.stack(frames), np.uint8)
    h, w = fr.shape[1:]
    out = np.empty((h, w), np.uint8)
    lib = reflib() if ref else clib()
    fn = lib.ref_median_bg_ih if ref else lib.or_median_bg_ih
    _check(fn(fr.reshape(-1), nf, len(fr) - nf, w, h, bins, m, n, out.reshape(-1)), "median_background_ih",
           lib if ref else None)
    return out


def median_bg_sort(frames, ref: bool = False) -> np.ndarray:
    fr = np.ascontiguousarray(np.stack(frames), np.uint8)
    h, w = fr.shape[1:]
    out = np.empty((h, w), np.uint8)
    lib = reflib() if ref else clib()
    fn = lib.ref_median_bg_sort if ref else lib.or_median_bg_sort
    _check(fn(fr.reshape(-1), len(fr), w, h, out.reshape(-1)), "median_background_sort", lib if ref else None)
    return out


def hist_finalize(dsum, w, h, kw, kh, p) -> np.ndarray:
    dsum = np.ascontiguousarray(dsum, np.float64)
    out = np.empty((h, w), np.float64)
    _check(clib().or_hist_finalize(dsum.reshape(-1), w, h, kw, kh, p, out.reshape(-1)), "hist_finalize")
    return out


@dataclass
class ScheduleStats:
    wavefront_iterations: int
    tile_count: int
    scan_efficiency: float


def schedule_stats(w, h, tile, scan_len) -> ScheduleStats:
    it, tl, ef = C.c_longlong(), C.c_longlong(), _d()
    _check(clib().or_schedule_stats(w, h, tile, scan_len, C.byref(it), C.byref(tl), C.byref(ef)), "schedule_stats")
    return ScheduleStats(it.value, tl.value, ef.value)


def estimate_memory(w, h, bins, elem):
    pad, raw, deg = _u64(), _u64(), _i()
    _check(clib().or_estimate_memory(w, h, bins, elem, C.byref(pad), C.byref(raw), C.byref(deg)), "estimate_memory")
    return int(pad.value), int(raw.value), bool(deg.value)


# ----------------------------------------------------------------- compiled reference

class RefTensor:
    """Handle to a reference-built IntegralHistogramTensor (uint64, padded layout)."""

    def __init__(self, bm: np.ndarray, nbins: int, kind: int = SEQUENTIAL, tile: int = 32,
                 threads: int = 1, budget: int = DEFAULT_BUDGET):
        lib = reflib()
        if lib is None:
            raise RuntimeError("oracle/_ref/libspct_ref.so not built")
        self._lib = lib
        bm = np.ascontiguousarray(bm, np.uint16)
        self.h, self.w = bm.shape if bm.ndim == 2 else (0, 0)
        self.bins = nbins
        hdl = _vp()
        _check(lib.ref_ih_build(bm.reshape(-1), self.w, self.h, nbins, kind, tile, threads, budget,
                                C.byref(hdl)), "build_integral_histogram", lib)
        self._h = hdl

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.ref_ih_free(self._h)
            self._h = None

    def dump(self, path: str) -> None:
        """dump_tensor (integral.cpp:619-633) of the reference."""
        _check(self._lib.ref_dump_tensor(self._h, str(path).encode()), "dump_tensor", self._lib)

    @classmethod
    def load(cls, path: str) -> "RefTensor":
        """load_tensor (integral.cpp:635-659) of the reference."""
        lib = reflib()
        hdl = _vp()
        _check(lib.ref_load_tensor(str(path).encode(), C.byref(hdl)), "load_tensor", lib)
        t = cls.__new__(cls)
        t._lib, t._h = lib, hdl
        n = int(lib.ref_ih_size(hdl))
        with open(path, "rb") as f:
            hdr = np.frombuffer(f.read(20)[4:], np.uint32)
        t.bins, t.h, t.w = int(hdr[0]), int(hdr[1]), int(hdr[2])
        assert n == t.bins * (t.h + 1) * (t.w + 1)
        return t

    def array(self) -> np.ndarray:
        n = int(self._lib.ref_ih_size(self._h))
        ptr = self._lib.ref_ih_data(self._h)
        a = np.ctypeslib.as_array(ptr, shape=(n,))
        return a.reshape(self.bins, self.h + 1, self.w + 1).copy()

    def region_histogram(self, x, y, w, h) -> np.ndarray:
        out = np.empty(self.bins, np.uint64)
        _check(self._lib.ref_region_histogram(self._h, x, y, w, h, out), "region_histogram", self._lib)
        return out

    def region_count(self, k, x, y, w, h) -> int:
        v = _u64()
        _check(self._lib.ref_region_count(self._h, k, x, y, w, h, C.byref(v)), "region_count", self._lib)
        return int(v.value)

    def hist_distance_map(self, tmpl, kw, kh, p=1.0) -> np.ndarray:
        tmpl = np.ascontiguousarray(tmpl, np.float64)
        out = np.empty((self.h, self.w), np.float64)
        _check(self._lib.ref_hist_distance_map(self._h, tmpl, tmpl.size, kw, kh, p, out.reshape(-1)),
               "hist_distance_map", self._lib)
        return out


def ref_to_grayscale(r, g, b):
    lib = reflib()
    r, g, b = (np.ascontiguousarray(a, np.uint8) for a in (r, g, b))
    out = np.empty_like(r)
    _check(lib.ref_to_grayscale(r.reshape(-1), g.reshape(-1), b.reshape(-1), r.shape[1], r.shape[0],
                                out.reshape(-1)), "to_grayscale", lib)
    return out


def ref_quantize(img, bins, lo=0.0, hi=256.0):
    lib = reflib()
    img = np.ascontiguousarray(img)
    h, w = img.shape
    out = np.empty((h, w), np.uint16)
    if img.dtype == np.uint8:
        st = lib.ref_quantize_u8(img.reshape(-1), w, h, bins, lo, hi, out.reshape(-1))
    else:
        st = lib.ref_quantize_f64(np.ascontiguousarray(img, np.float64).reshape(-1), w, h, bins, lo, hi,
                                  out.reshape(-1))
    _check(st, "quantize", lib)
    return out


def ref_schedule_stats(w, h, tile, scan_len) -> ScheduleStats:
    lib = reflib()
    it, tl, ef = C.c_longlong(), C.c_longlong(), _d()
    _check(lib.ref_schedule_stats(w, h, tile, scan_len, C.byref(it), C.byref(tl), C.byref(ef)),
           "schedule_stats", lib)
    return ScheduleStats(it.value, tl.value, ef.value)


def ref_estimate_memory(w, h, bins, elem):
    lib = reflib()
    pad, raw, deg = _u64(), _u64(), _i()
    _check(lib.ref_estimate_memory(w, h, bins, elem, C.byref(pad), C.byref(raw), C.byref(deg)),
           "estimate_memory", lib)
    return int(pad.value), int(raw.value), bool(deg.value)
