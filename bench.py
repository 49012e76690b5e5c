#!/usr/bin/env python
"""Benchmark of the B200 integral-histogram + likelihood-map path (BASELINE.json metric).

One step = one frame through the hot path: quantise a 4096x4096 uint8 frame into 128
bins, write the 128-plane uint32 integral histogram to HBM, and produce the 64x64
sliding-window (Minkowski p = 1) likelihood map (float64, W x H).  Throughput is
Gbin*px/s = 128 * 4096^2 / step time, whole job over all ranks.

  python bench.py [--gpus N --steps K --warmup W]     our arm (re-launches itself as N ranks)
  python bench.py --impl reference [...]              the reference CPU path (rank 0 only)

Multi-GPU (N > 1), bin-slab sharding (north star): the headline line is
STRONG scaling of the metric's own configuration — rank r owns bins slab_bounds(128, N, r)
of the same 4096^2 x 128 histogram, sweeps that slab of the tensor and its partial window
sums; the partials are then summed and finalised by the band-owned peer-memory reduce
(--reduce band, default), by the root (--reduce root) or by one NCCL reduce (--reduce
nccl).  Extra lines: `c4` (BASELINE config 4: 8192^2 x 256 bins, strong, every N
including N = 1 with the whole 68.7 GB tensor on one GPU) and, for N > 1, `weak` (128
bins per GPU of a 128 N-bin histogram over the same frame).  N = 1 also reports
build_only, c2 (config 2), tensor_matcher, general-template paths, next_rows (§8(f)),
c5_batch (config 5), dropin_e2e (the C++ drop-in API), parity (this run's GPU tensor and
map against the reference's on the same frame) and cpu_baseline.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
compute stream; a 256 MiB memset flushes L2 between steps outside the events (every
input and output is also larger than L2 except the C2 frame); barrier + synchronize on
both sides; max over ranks.  `e2e` repeats the measurement through the public API with
the frame copied host->device and the map copied device->host inside the timed region.
`roofline` reports the dominant kernel's algorithmic bytes over its event-timed duration
against MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "integral-histogram Gbin·px/s and HBM-roofline fraction, 4096²×128 bins, 1–8 GPU"
UNIT = "Gbin·px/s"
W_IMG = H_IMG = 4096
NBINS = 128
KW = KH = 64
P_ORDER = 1.0
C4_SIDE, C4_BINS = 8192, 256


def make_frame(w: int, h: int, seed: int = 1) -> np.ndarray:
    """Synthetic 8-bit frame: uniform noise (numpy PCG64) — the worst case for run-based schedules."""
    return np.random.default_rng(seed).integers(0, 256, size=(h, w), dtype=np.uint8)


def template_hist(frame: np.ndarray, nbins: int, kw: int, kh: int) -> np.ndarray:
    """Normalised histogram of the centred kw x kh crop (spct_main.cpp:328-331 style)."""
    h, w = frame.shape
    y0, x0 = (h - kh) // 2, (w - kw) // 2
    crop = frame[y0:y0 + kh, x0:x0 + kw].astype(np.int64)
    bins = (crop * nbins) >> 8  # quantize(img, nbins) for the default [0, 256) range
    return np.bincount(bins.reshape(-1), minlength=nbins).astype(np.float64) / crop.size


def general_template(nbins: int, seed: int = 3) -> np.ndarray:
    """A normalised template whose entries are not multiples of 1/(kw kh) (the reference
    accepts any; the integer fast path does not apply)."""
    r = np.random.default_rng(seed).random(nbins) + 0.1
    return r / r.sum()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU baseline (reference / oracle port)

def cpu_sample(rows: int = 192, reps: int = 3, keep_arrays: bool = False) -> dict:
    """The reference CPU path on a bounded sample of the C3 workload, extrapolated to the
    full frame.  Sample: the top `rows` rows of the 4096-wide frame, 128 bins, 64x64 p = 1
    map against the full frame's template.

    * build_integral_histogram: the best of Sequential (1 thread) and CrossWeaveTiled on
      every host thread, memory_budget = UINT64_MAX, after one untimed pre-faulting build,
      best of `reps` each;
    * hist_distance_map: single-threaded as shipped, best of `reps`.
    Full-frame estimate: build x (4096 / rows) + matcher x (4033 / (rows - 63)) — the build
    scales with rows, the matcher with window rows.  Uses oracle/_ref (the unmodified
    reference) when built, else the C port."""
    import oracle  # CPU checker/baseline only — never on the measured GPU path

    full = make_frame(W_IMG, H_IMG)
    frame = full[:rows]
    tmpl = template_hist(full, NBINS, KW, KH)
    threads = min(64, os.cpu_count() or 1)
    kind = "reference" if oracle.have_ref() else "port"
    reps = max(1, reps)
    builds, match_s, lmap, ih = {}, None, None, None
    if kind == "reference":
        qb = oracle.ref_quantize(frame, NBINS)
        budget = (1 << 64) - 1
        oracle.RefTensor(qb, NBINS, oracle.CW_TIS, 32, threads, budget=budget)  # pre-fault warm-up
        t = None
        for name, sk, th in (("sequential", oracle.SEQUENTIAL, 1), ("cw-tis", oracle.CW_TIS, threads)):
            best = None
            for _ in range(reps):
                t = None
                t0 = time.perf_counter()
                t = oracle.RefTensor(qb, NBINS, sk, 32, th, budget=budget)
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            builds[name] = best
        for _ in range(reps):
            t0 = time.perf_counter()
            lmap = t.hist_distance_map(tmpl, KW, KH, P_ORDER)
            dt = time.perf_counter() - t0
            match_s = dt if match_s is None else min(match_s, dt)
        if keep_arrays:
            ih = t.array()
        del t
    else:
        qb = oracle.quantize(frame, NBINS)
        t0 = time.perf_counter()
        ih = oracle.build_ih(qb, NBINS)
        builds["sequential"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        lmap = oracle.hist_distance_map(ih, tmpl, KW, KH, P_ORDER)
        match_s = time.perf_counter() - t0
    best_kind = min(builds, key=builds.get)
    nv_band, nv_full = rows - KH + 1, H_IMG - KH + 1
    full_s = builds[best_kind] * H_IMG / rows + match_s * nv_full / nv_band
    value = NBINS * H_IMG * W_IMG / full_s / 1e9
    out = {"value": value, "unit": UNIT, "cores": threads if kind == "reference" else 1, "kind": kind,
           "cpu_model": cpu_model(),
           "sample": (f"top {rows} rows of the 4096x4096 frame ({nv_band} window rows), 128 bins, 64x64 p=1 map; "
                      f"build best of sequential x1 / cw-tis x{threads} threads (best: {best_kind}, "
                      f"{builds[best_kind] * 1e3:.1f} ms, pre-faulted, best of {reps}); hist_distance_map 1 thread "
                      f"as shipped ({match_s:.2f} s, best of {reps}); full frame estimated as build x {H_IMG}/{rows} "
                      f"+ matcher x {nv_full}/{nv_band} = {full_s:.1f} s"),
           "seconds_full_frame_estimate": full_s,
           "build_ms": {k: round(v * 1e3, 2) for k, v in builds.items()}, "match_s": match_s}
    if keep_arrays:
        out["_map"], out["_ih"] = lmap, ih
    return out


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    secs, last = [], None
    for i in range(warm + steps):
        last = cpu_sample(args.ref_rows, 1)
        if i >= warm:
            secs.append(last["seconds_full_frame_estimate"])
    sec = sum(secs) / len(secs)
    value = NBINS * H_IMG * W_IMG / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
        "config": {"workload": "C3: 4096x4096 uint8 frame -> 128-bin integral histogram + 64x64 p=1 likelihood map",
                   "bins_total": NBINS, "window": [KW, KH], "p": P_ORDER,
                   "estimate": ("each step times a band of the same frame (build on every host thread, matcher "
                                "single-threaded as shipped) and scales it to the full frame: build by rows, "
                                "matcher by window rows")},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": last["kind"],
                         "cpu_model": last["cpu_model"], "sample": last["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm: helpers

def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def box_peaks(dev) -> dict:
    """Copy and write-only bandwidth of this device, measured live ("also
    record a measured device write/copy peak on the box").  2 GiB buffers (> L2), torch's
    own copy_/fill_ kernels, CUDA events over 10 back-to-back launches each.  Outside
    every timed region."""
    import torch

    n = 1 << 31
    a = torch.empty(n // 4, dtype=torch.int32, device=dev)
    b = torch.empty_like(a)
    a.fill_(1)
    b.copy_(a)
    torch.cuda.synchronize(dev)

    def t(fn, reps=10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    copy_ms = t(lambda: b.copy_(a))
    write_ms = t(lambda: a.fill_(3))
    del a, b
    torch.cuda.empty_cache()
    return {"copy_gbs": round(2 * n / (copy_ms * 1e-3) / 1e9, 1), "write_gbs": round(n / (write_ms * 1e-3) / 1e9, 1),
            "method": "torch copy_ (read + write bytes) and fill_ of 2 GiB int32, CUDA events, outside the timed region"}


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    v = d.get(kernel)
    return None if v is None else float(v.get("dram_bytes_per_launch"))


class Timer:
    """CUDA-event timing of `fn` on the compute stream, K steps, L2 flushed between steps
    (outside the events), barrier + synchronize on both sides, max over ranks."""

    def __init__(self, world, dev, stream, shared):
        import torch

        self.world, self.dev, self.stream, self.shared = world, dev, stream, shared
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier(self):
        import torch
        import torch.distributed as dist

        torch.cuda.synchronize()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def __call__(self, fn, k: int, warmup: int = 0, flush: bool = True) -> float:
        import torch

        from paper_1711_01656_b200.sharding import max_over_ranks

        for _ in range(warmup):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        self.barrier()
        for a, b in ev:
            if flush:
                self.flush.zero_()
            a.record(self.stream)
            fn()
            b.record(self.stream)
        self.barrier()
        ms = sum(a.elapsed_time(b) for a, b in ev)
        return max_over_ranks(ms, None if self.shared else self.dev) / k


def kernel_ms(profiling, names) -> dict:
    out = {}
    for name in names:
        kt, kn = profiling.kernel_time(name)
        if kn:
            out[name] = (kt, kn)
    return out


def roofline_of(kms: float, alg: int, pk: dict) -> dict:
    achieved = alg / (kms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": round(achieved / pk["hbm_gbs"], 4), "alg_bytes": alg, "kernel_ms": round(kms, 4)}


def run_c5(P, dev, stream, frames: int = 100, side: int = 2048, nbins: int = 32, kw: int = 64, kh: int = 64):
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(5)
    rgb = torch.randint(0, 256, (frames, 3, side, side), dtype=torch.uint8, device=dev, generator=g)
    # templates: each channel's histogram of the centred kw x kh crop of frame 0
    srcs = P.channel_sources(rgb[0, 0], rgb[0, 1], rgb[0, 2], nbins)
    y0, x0 = (side - kh) // 2, (side - kw) // 2
    tdev = {}
    for c, s in srcs.items():
        qb = s if c == "orientation" else P.quantize(s, nbins)
        crop = qb[y0:y0 + kh, x0:x0 + kw].to(torch.int64).reshape(-1) & 0xFFFF
        tdev[c] = (torch.bincount(crop, minlength=nbins).to(torch.float64) / crop.numel()).contiguous()
    from paper_1711_01656_b200.channels import ChannelGraph

    graph = ChannelGraph(side, side, nbins, tdev, kw, kh, 1.0, device=dev)

    def frame(i):
        graph.run(rgb[i, 0], rgb[i, 1], rgb[i, 2])
    for i in range(3):
        frame(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(frames):
        frame(i)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    binpx = frames * len(P.CHANNELS) * nbins * side * side
    return {"frames": frames, "channels": list(P.CHANNELS), "bins": nbins, "side": side, "window": [kw, kh],
            "ms_per_frame": round(ms / frames, 4), "value": round(binpx / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "data": "synthetic uint8 RGB (torch RNG on the device), frames resident; every channel's IH written",
            "launch": "one CUDA graph per frame (channels.ChannelGraph): frame copied into static buffers, replayed",
            "l2": f"frames and tensors ({frames * 3 * side * side / 2**20:.0f} MiB of frames) exceed L2"}


def run_c2(P, dev, timer, pk):
    """BASELINE config 2: 1024^2 RGB frame (planar, uniform noise) -> gray -> 32 bins -> IH
    + 64x64 intersection-equivalent (p = 1) map against the crop at (480, 480).  Latency
    bound (report only): 200 steps per event pair, no flush (the 3 MB frame and 134 MB
    tensor are re-written every step)."""
    import torch

    rng = np.random.default_rng(2)
    r, g, b = (rng.integers(0, 256, (1024, 1024), dtype=np.uint8) for _ in range(3))
    gray = ((r.astype(np.int32) + g + b + 1) // 3).astype(np.int64)  # to_grayscale (imagecore.cpp:20-21)
    crop = (gray[480:544, 480:544] * 32) >> 8
    tmpl = np.bincount(crop.reshape(-1), minlength=32).astype(np.float64) / crop.size
    planes = [torch.from_numpy(x).to(dev) for x in (r, g, b)]
    tdev = torch.from_numpy(tmpl).to(dev)
    t = P.IntegralHistogramTensor(1024, 1024, 32, device=dev)
    lmap = torch.empty((1024, 1024), dtype=torch.float64, device=dev)

    def step():
        P.build_and_match_map(tuple(planes), 32, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=tdev)
    reps = 200
    ms = timer(lambda: [step() for _ in range(reps)], 3, warmup=2, flush=False) / reps
    peak_at = float(lmap[480 + 31, 480 + 31].item())
    alg = 32 * 1024 * 1024 * 4 + 3 * 1024 * 1024 + 1024 * 1024 * 8
    return {"workload": "C2: 1024x1024 planar RGB -> gray -> 32 bins, IH + 64x64 p=1 map (crop template at 480,480)",
            "ms_per_step": round(ms, 5), "value": round(32 * 1024 * 1024 / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
            "frac_of_peak_step": round(alg / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], 4), "alg_bytes": alg,
            "template_window_score": peak_at, "note": "latency-bound at this size (BASELINE.md §3: report only)"}


def run_next_rows(P, dev, pk_gbs: float) -> dict:
    """SURVEY §8(f) rows on resident inputs, device-timed (CUDA events, synchronised): the
    SWIH tracker channel, the map consumers at the C3 map size and the joint-IH temporal
    median.  Each entry: ms per call, algorithmic bytes, GB/s and fraction of the HBM peak
    (bytes that must move: outputs written + inputs read once)."""
    import torch

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def line(cfg, ms, alg):
        gbs = alg / (ms * 1e-3) / 1e9 if alg else None
        return {"config": cfg, "ms": round(ms, 4), "alg_bytes": alg,
                "gbs": round(gbs, 1) if gbs else None, "frac": round(gbs / pk_gbs, 4) if gbs else None}

    out = {}
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    n, nb, k = 1024, 32, 31
    bm = torch.randint(0, nb, (n, n), dtype=torch.int16, device=dev, generator=g)
    model = np.full(nb, 1.0 / nb)
    ms_b = timed(lambda: P.swih.build_quadrant_set(bm, nb, k, k))
    out["swih_quadrant_set"] = line(f"{n}x{n} BinMap, {nb} bins, {k}x{k} kernel: four uint64 16.16 tensors", ms_b,
                                    4 * nb * n * n * 8 + n * n * 2)
    ms_m = timed(lambda: P.swih.swlh_distance_map(bm, nb, model, k, k))
    out["swih_distance_map"] = line("swlh-distance map (float64) in one sweep over the BinMap (no tensors; "
                                    "W / mass from a table of every window sum; compute-bound by the FP64 "
                                    "per-bin terms |q - model| summed in bin order)", ms_m, n * n * 2 + n * n * 8)
    ms_q = timed(lambda: P.swih.swlh_distance_map(bm, nb, model, k, k, method="quadrant"))
    out["swih_distance_map_quadrant"] = line("the same map through the quadrant tensors (reference construction)",
                                             ms_q, 4 * nb * n * n * 8 + n * n * 2 + n * n * 8)
    m4 = [torch.rand((H_IMG, W_IMG), dtype=torch.float64, device=dev, generator=g) for _ in range(5)]
    fused = torch.empty_like(m4[0])
    ms_f = timed(lambda: P.fuse_maps(m4, [1, 2, 3, 4, 5], out=fused))
    out["fuse_maps"] = line("5 maps 4096x4096 float64, weighted", ms_f, 6 * H_IMG * W_IMG * 8)
    ms_p = timed(lambda: P.find_peaks(fused))
    out["find_peaks"] = line("4096x4096: 3x3 mean, strict local maxima, stable sort by height", ms_p,
                             H_IMG * W_IMG * 8)
    ms_s = timed(lambda: P.score_map(fused, 1000, 1000, 64, 64))
    out["score_map"] = line("4096x4096, 64x64 ground-truth rect", ms_s, H_IMG * W_IMG * 8)
    starts = [[64 + 61 * i, 64 + 57 * i] for i in range(64)]
    ms_c = timed(lambda: P.camshift_batch(fused, starts, 64, 64))
    out["camshift_batch"] = line("64 starts, 64x64 windows, 4096x4096 map", ms_c, None)
    fr = [torch.randint(0, 16, (n, n), dtype=torch.uint8, device=dev, generator=g) for _ in range(8)]
    mb = P.motion.MedianBackgroundIH(fr[:5], 16, 7, 7)
    it = iter(range(10 ** 9))
    ms_sl = timed(lambda: mb.slide(fr[5 + next(it) % 3]))
    out["median_slide"] = line(f"{n}x{n}, 16 bins, 5 frames: joint tensor += IH(new) - IH(old), one read-modify-"
                               "write pass (algorithmic bytes: the joint tensor read + written once, two frames)", ms_sl,
                               2 * 16 * n * n * 4 + 2 * n * n)
    ms_bg = timed(lambda: mb.background())
    out["median_background"] = line("7x7 windows, per-pixel CDF walk over 16 bins", ms_bg, 16 * n * n * 4 + n * n)
    return out


def run_dropin(timeout: int = 600) -> dict:
    """The C++ drop-in API (include/spct/spct.hpp, reference signatures, host buffers in and
    results returned by value) timed by tests/cpp/dropin_bench at C3."""
    exe = os.path.join(ROOT, "build", "dropin_bench")
    if not os.path.exists(exe):
        return {"unavailable": "build/dropin_bench not built (make dropin_bench)"}
    try:
        r = subprocess.run([exe, str(W_IMG), str(NBINS), "5", "--json"], capture_output=True, text=True,
                           timeout=timeout)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except (subprocess.SubprocessError, ValueError, IndexError) as e:
        err = (locals().get("r").stderr if locals().get("r") is not None else "")[-300:]
        return {"unavailable": f"{str(e)[:100]}; rc={getattr(locals().get('r'), 'returncode', None)}; {err}"}
    d["unit"] = UNIT
    d["note"] = ("value: Gbin*px/s of build_integral_histogram(BinMap) + hist_distance_map(t, ...) per frame with "
                 "host buffers (the reference's call sequence, spct_main.cpp:332-333); value_fused: the one-call "
                 "likelihood_from_frame(GrayImage, ...); map results returned by value as std::vector<double>")
    return d


# ---------------------------------------------------------------- our arm

def relaunch(args) -> None:
    """`--gpus N` without a torchrun environment: start N ranks of this script."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device")
    # SPCT_BENCH_SHARED_GPU=1: every rank on cuda:0 with a gloo group (functional check of
    # the N > 1 path on a one-GPU box; its numbers are not scaling numbers)
    shared = os.environ.get("SPCT_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1711_01656_b200 as P
    from paper_1711_01656_b200 import profiling
    from paper_1711_01656_b200.sharding import ShardedMapStep

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    timer = Timer(world, dev, stream, shared)
    pk = peaks()
    frame_h = make_frame(W_IMG, H_IMG)
    tmpl = template_hist(frame_h, NBINS, KW, KH)
    frame = torch.from_numpy(frame_h).to(dev)

    # ---- headline: C3, 128 bins split over the ranks (strong scaling)
    main = ShardedMapStep(W_IMG, H_IMG, NBINS, tmpl, KW, KH, P_ORDER, reduce=args.reduce, device=dev)
    for _ in range(args.warmup):
        main.step(frame)
    timer.barrier()
    profiling.reset()
    profiling.enable(True)
    l0 = profiling.launch_count()
    with ClockSampler(local) as clk:
        ms = timer(lambda: main.step(frame), args.steps)
    launches = profiling.launch_count() - l0
    profiling.enable(False)
    kernels = kernel_ms(profiling, ("ih_sweep", "ih_sweep_match", "match_partial", "narrow_sweep_match"))
    profiling.reset()

    def strong_roofline(name, kt, kn, steps, side, nbins_total, nbins_rank, finished_map):
        """Dominant kernel of a bin-sharded step: IH write + frame read + map write
        (finished W x H map at N = 1, the rank's partial (H-kh+1) x (W-kw+1) otherwise)."""
        kms_step = kt / steps
        binpx = nbins_rank * side * side
        alg = binpx * 4 + side * side + (side * side * 8 if finished_map else (side - KW + 1) * (side - KH + 1) * 8)
        r = roofline_of(kms_step, alg, pk)
        r.update({"kernel": name, "launches_per_step": kn // steps, "kernel_ms_per_step": round(kms_step, 4)})
        return r

    roof = None
    if kernels:
        name, (kt, kn) = max(kernels.items(), key=lambda kv: kv[1][0])
        roof = strong_roofline(name, kt, kn, args.steps, W_IMG, NBINS, main.bin1 - main.bin0, world == 1)
        roof.update({"traffic": ncu_traffic(name) if world == 1 else None, "step_share": round(kt / args.steps / ms, 3),
                     "peak_source": pk["source"], "kernels_ms": {k: round(v[0] / args.steps, 4)
                                                                 for k, v in kernels.items()}})

    extras = {}
    # ---- weak scaling (N > 1): 128 bins per rank of a 128 N-bin histogram, same frame
    if world > 1 and not args.no_weak:
        tw = template_hist(frame_h, NBINS * world, KW, KH)
        weak = ShardedMapStep(W_IMG, H_IMG, NBINS * world, tw, KW, KH, P_ORDER, bins_per_rank=NBINS,
                              reduce=args.reduce, device=dev)
        ms_w = timer(lambda: weak.step(frame), args.steps, warmup=args.warmup)
        extras["weak"] = {"workload": f"C3 frame, {NBINS} bins per GPU of a {NBINS * world}-bin histogram "
                                      "(weak scaling: fixed work per GPU)",
                          "ms_per_step": round(ms_w, 4), "scaling": "weak",
                          "value": round(NBINS * world * W_IMG * H_IMG / (ms_w * 1e-3) / 1e9, 2), "unit": UNIT,
                          "reduce": weak.note}
        if weak.error():
            raise SystemExit("bench.py: a peer-reduce wait timed out (weak)")
        weak.close()
        del weak

    # ---- N > 1: the north star's collective (one NCCL reduce of the partial maps + finalise
    # on the root) beside the default peer-memory band reduce, same configuration
    if world > 1 and args.reduce != "nccl":
        try:
            alt = ShardedMapStep(W_IMG, H_IMG, NBINS, tmpl, KW, KH, P_ORDER, reduce="nccl", device=dev)
            ms_n = timer(lambda: alt.step(frame), args.steps, warmup=args.warmup)
            extras["reduce_nccl"] = {"workload": "the headline step with one dist.reduce (NCCL) of the partial maps "
                                                 "and hist_finalize on rank 0", "ms_per_step": round(ms_n, 4),
                                     "value": round(NBINS * W_IMG * H_IMG / (ms_n * 1e-3) / 1e9, 2), "unit": UNIT,
                                     "reduce": alt.note, "backend": dist.get_backend()}
            alt.close()
            del alt
        except Exception as e:  # e.g. the shared-GPU functional mode runs gloo
            extras["reduce_nccl"] = {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}

    # ---- single-GPU extras
    if world == 1:
        t = main.tensor

        def build_step():
            P.build_integral_histogram(frame, NBINS, memory_budget=None, out=t, validate=False)
        profiling.reset()
        profiling.enable(True)
        ms_b = timer(build_step, args.steps, warmup=args.warmup)
        profiling.enable(False)
        kb = kernel_ms(profiling, ("ih_sweep",))
        profiling.reset()
        alg_b = NBINS * W_IMG * H_IMG * 4 + W_IMG * H_IMG
        extras["build_only"] = {"workload": "C3 plain build_integral_histogram (BASELINE config 3)",
                                "ms_per_step": round(ms_b, 4),
                                "value": round(NBINS * W_IMG * H_IMG / (ms_b * 1e-3) / 1e9, 2), "unit": UNIT,
                                "roofline": roofline_of(kb["ih_sweep"][0] / kb["ih_sweep"][1], alg_b, pk)
                                if "ih_sweep" in kb else None}
        # main.tensor again holds the headline frame's IH (the same frame): parity below reads it
        if not args.no_c2:
            extras["c2"] = run_c2(P, dev, timer, pk)
        if not args.no_paths:
            extras.update(run_paths(P, dev, timer, pk, frame, tmpl, t, args))
        if not args.no_next:
            extras["next_rows"] = run_next_rows(P, dev, pk["hbm_gbs"])
        if not args.no_c5:
            extras["c5_batch"] = run_c5(P, dev, stream)

    # ---- BASELINE config 4: 8192^2 x 256 bins, strong scaling (N = 1: the whole 68.7 GB tensor)
    if not args.no_c4:
        need = C4_BINS // world * C4_SIDE * C4_SIDE * 4 + 4 * C4_SIDE * C4_SIDE * 8
        free = torch.cuda.mem_get_info(dev)[0]
        if need < free * 0.95:
            f4h = make_frame(C4_SIDE, C4_SIDE, seed=4)
            t4 = template_hist(f4h, C4_BINS, KW, KH)
            f4 = torch.from_numpy(f4h).to(dev)
            c4 = ShardedMapStep(C4_SIDE, C4_SIDE, C4_BINS, t4, KW, KH, P_ORDER, reduce=args.reduce, device=dev)
            for _ in range(args.warmup):
                c4.step(f4)
            profiling.reset()
            profiling.enable(True)
            ms4 = timer(lambda: c4.step(f4), args.steps)
            profiling.enable(False)
            k4 = kernel_ms(profiling, ("ih_sweep_match", "narrow_sweep_match"))
            profiling.reset()
            line4 = {"workload": f"C4: {C4_SIDE}x{C4_SIDE} uint8 frame -> {C4_BINS}-bin uint32 integral histogram "
                                 f"(bin slab {c4.bin1 - c4.bin0} bins on this rank) + 64x64 p=1 likelihood map",
                     "ms_per_step": round(ms4, 4), "scaling": "strong",
                     "value": round(C4_BINS * C4_SIDE * C4_SIDE / (ms4 * 1e-3) / 1e9, 2), "unit": UNIT,
                     "tensor_bytes_per_gpu": (c4.bin1 - c4.bin0) * C4_SIDE * C4_SIDE * 4, "reduce": c4.note}
            if k4:
                name, (kt, kn) = max(k4.items(), key=lambda kv: kv[1][0])
                line4["roofline"] = strong_roofline(name, kt, kn, args.steps, C4_SIDE, C4_BINS, c4.bin1 - c4.bin0,
                                                    False)  # > 128 bins per GPU: groups of partial sums
            if c4.error():
                raise SystemExit("bench.py: a peer-reduce wait timed out (c4)")
            if world == 1:  # property checks (the full cell-by-cell parity is in the -m gpu tests)
                cx, cy = (C4_SIDE - KW) // 2 + (KW - 1) // 2, (C4_SIDE - KH) // 2 + (KH - 1) // 2
                line4["template_window_score"] = float(c4.map[cy, cx].item())
            elif rank == 0:
                cx, cy = (C4_SIDE - KW) // 2 + (KW - 1) // 2, (C4_SIDE - KH) // 2 + (KH - 1) // 2
                line4["template_window_score"] = float(c4.map[cy, cx].item())
            extras["c4"] = line4
            c4.close()
            del c4, f4
            torch.cuda.empty_cache()
        else:
            extras["c4"] = {"skipped": f"needs {need / 1e9:.1f} GB, {free / 1e9:.1f} GB free"}

    # ---- end to end through the public API: pinned host frame in, host map out, every step
    if world == 1:
        # K distinct pinned host frames in, K host maps out; copies of frame n+1 / map n-1
        # overlap the sweep of frame n (double-buffered, 3 streams)
        from paper_1711_01656_b200.pipeline import FramePipeline

        pipe = FramePipeline(W_IMG, H_IMG, NBINS, tmpl, KW, KH, P_ORDER, device=dev)
        hframes = FramePipeline.pinned_frames([make_frame(W_IMG, H_IMG, seed=100 + i) for i in range(args.steps)])
        hmaps = pipe.pinned_maps(2)
        ring = [hmaps[i & 1] for i in range(args.steps)]
        pipe.run(hframes[:max(1, args.warmup)], ring[:max(1, args.warmup)])
        timer.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(pipe.h2d)
        pipe.run(hframes, ring)
        ev1.record(pipe.d2h)
        timer.barrier()
        ms_e2e = ev0.elapsed_time(ev1) / args.steps
        e2e_mode = "pipelined (FramePipeline: H2D / sweep / D2H on three streams, double-buffered)"
        del pipe
    else:
        host_frame = torch.from_numpy(frame_h).pin_memory()
        host_map = torch.empty((H_IMG, W_IMG), dtype=torch.float64).pin_memory()
        dframe = torch.empty_like(frame)

        def e2e_step():
            dframe.copy_(host_frame, non_blocking=True)
            main.step(dframe)
            if rank == 0:
                host_map.copy_(main.map, non_blocking=True)
        ms_e2e = timer(e2e_step, args.steps, warmup=max(1, args.warmup))
        e2e_mode = "serial (every rank copies the frame in, rank 0 copies the map out)"

    # ---- parity against the reference on this very frame, cpu baseline, C++ drop-in (rank 0, N = 1)
    parity, cpu = None, None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(args.ref_rows, 3, keep_arrays=not args.no_parity)
            if not args.no_parity:
                parity = check_parity(cpu.pop("_map"), cpu.pop("_ih"), main, args.ref_rows)
        except Exception as e:  # the baseline is reported, never required for the GPU number
            cpu = {"value": None, "error": str(e)[:200]}
        for k in ("_map", "_ih", "seconds_full_frame_estimate", "match_s"):
            (cpu or {}).pop(k, None)
    if world == 1 and not args.no_dropin:
        extras["dropin_e2e"] = run_dropin()

    if main.error():
        raise SystemExit("bench.py: a peer-reduce wait timed out")
    main.close()
    bx = None
    if rank == 0 and roof is not None:
        try:
            bx = box_peaks(dev)
            bx["frac_vs_copy"] = round(roof["achieved"] / bx["copy_gbs"], 4)
            bx["frac_vs_write"] = round(roof["achieved"] / bx["write_gbs"], 4)
            roof["box_measured"] = bx
        except RuntimeError as e:  # e.g. no room for the 4 GiB of probe buffers
            roof["box_measured"] = {"unavailable": str(e).splitlines()[0]}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    total_binpx = NBINS * W_IMG * H_IMG
    line = {
        "metric": METRIC, "value": round(total_binpx / (ms * 1e-3) / 1e9, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
        "config": {"workload": ("C3: 4096x4096 uint8 frame -> quantise -> 128-bin uint32 integral histogram "
                                "+ 64x64 p=1 likelihood map (float64)"),
                   "bins_total": NBINS, "bins_per_gpu": main.bin1 - main.bin0, "window": [KW, KH], "p": P_ORDER,
                   "parallelism": f"bin-slab x{world}" + ("" if world == 1 else f" + {main.note} reduce of partial maps"),
                   **({"shared_gpu": True} if shared else {}),
                   "l2": "256 MiB memset between timed steps (outside the events); step writes 8.6 GB in total"},
        "roofline": roof,
        "e2e": {"value": round(total_binpx / (ms_e2e * 1e-3) / 1e9, 2), "unit": UNIT,
                "h2d_bytes_per_step": W_IMG * H_IMG * world, "d2h_bytes_per_step": W_IMG * H_IMG * 8,
                "ms_per_step": round(ms_e2e, 4), "mode": e2e_mode},
        "gpu_launches": int(launches),
        "parity": parity,
        **extras,
        "clocks": clk.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_paths(P, dev, timer, pk, frame, tmpl, t, args) -> dict:
    """The other C3 matcher paths on the same frame (one line each): the tensor-reading
    matcher (hist_distance_map of a tensor with no known source frame, e.g. an IHT1 file),
    and the fused sweep with a general (non-integral) template at p = 1, p = 2 and the
    Bhattacharyya metric."""
    import torch

    from paper_1711_01656_b200 import profiling

    out = {}
    lmap = torch.empty((H_IMG, W_IMG), dtype=torch.float64, device=dev)
    src = t.source
    t.source = None  # as a loaded tensor: the map must come from the tensor itself
    tdev = torch.from_numpy(tmpl).to(dev)
    profiling.reset()
    profiling.enable(True)
    ms_t = timer(lambda: P.hist_match_map(t, tmpl, KW, KH, P_ORDER), args.steps, warmup=2)
    profiling.enable(False)
    kt = kernel_ms(profiling, ("ih_recover_bins", "sweep_match_nostore", "match_partial"))
    profiling.reset()
    # algorithmic bytes of the step: the tensor read once + the finished map written
    alg_t = NBINS * W_IMG * H_IMG * 4 + W_IMG * H_IMG * 8
    line = {"workload": "C3 tensor -> 64x64 p=1 map (hist_distance_map of a tensor without a source frame)",
            "ms_per_step": round(ms_t, 4), "value": round(NBINS * W_IMG * H_IMG / (ms_t * 1e-3) / 1e9, 2),
            "unit": UNIT, "roofline": roofline_of(ms_t, alg_t, pk),
            "kernels_ms": {k: round(v[0] / v[1], 4) for k, v in kt.items()}}
    line["roofline"]["kernel"] = "whole step (bin recovery + fused no-store sweep)"
    if "ih_recover_bins" in kt:
        ks, kn = kt["ih_recover_bins"]
        line["recover_roofline"] = roofline_of(ks / kn, NBINS * W_IMG * H_IMG * 4 + W_IMG * H_IMG * 2, pk)
    out["tensor_matcher"] = line
    t.source = src
    gt = general_template(NBINS)
    gdev = torch.from_numpy(gt).to(dev)
    alg_f = NBINS * W_IMG * H_IMG * 4 + W_IMG * H_IMG + W_IMG * H_IMG * 8
    for key, p, metric in (("general_template_p1", 1.0, 0), ("general_template_intersection", 1.0, 1),
                           ("general_template_p2", 2.0, 0), ("general_template_bhattacharyya", 1.0, 2),
                           ("general_template_chisq", 1.0, 3)):
        profiling.reset()
        profiling.enable(True)
        ms_g = timer(lambda: P.build_and_match_map(frame, NBINS, None, KW, KH, p, metric, out=t, lmap=lmap,
                                                   tmpl_dev=gdev), args.steps, warmup=2)
        profiling.enable(False)
        kg = kernel_ms(profiling, ("ih_sweep_match",))
        profiling.reset()
        out[key] = {"workload": f"C3 fused IH + 64x64 map, normalised random template, p={p}, "
                                f"metric={['minkowski', 'intersection', 'bhattacharyya', 'chi-square'][metric]}",
                    "ms_per_step": round(ms_g, 4), "value": round(NBINS * W_IMG * H_IMG / (ms_g * 1e-3) / 1e9, 2),
                    "unit": UNIT,
                    "roofline": roofline_of(kg["ih_sweep_match"][0] / kg["ih_sweep_match"][1], alg_f, pk)
                    if "ih_sweep_match" in kg else None}
    # leave the headline frame's tensor in t for the parity check
    P.build_and_match_map(frame, NBINS, None, KW, KH, P_ORDER, out=t, lmap=lmap, tmpl_dev=tdev)
    torch.cuda.synchronize()
    return out


def check_parity(ref_map: np.ndarray, ref_ih: np.ndarray, main, rows: int) -> dict:
    """This run's GPU results against the reference's on the same frame (the band the CPU
    baseline computed): every IH cell of rows [0, rows) and every map cell whose window lies
    in the band (map rows [0, (kh-1)/2 + rows - kh + 1))."""
    import torch

    torch.cuda.synchronize()
    out = {"reference": "oracle/_ref (unmodified reference, compiled from its sources)"
           if ref_ih is not None and ref_ih.dtype == np.uint64 else "oracle port"}
    t = main.tensor
    planes = t.planes()
    ih_bad = 0
    if ref_ih is not None:
        for k in range(t.bins):
            dev_k = planes[k, :rows, :W_IMG].cpu().numpy().view(np.uint32)
            ih_bad += int(np.count_nonzero(dev_k.astype(np.uint64) != ref_ih[k, 1:rows + 1, 1:W_IMG + 1]))
        out["ih_cells"] = int(t.bins * rows * W_IMG)
        out["ih_mismatches"] = ih_bad
    mrows = (KH - 1) // 2 + rows - KH + 1
    g = main.map[:mrows].cpu().numpy()
    r = ref_map[:mrows]
    err = np.abs(g - r)
    rel = err / np.maximum(np.abs(r), 1e-12)
    out.update({"map_cells": int(g.size), "map_bit_exact_cells": int(np.count_nonzero(g == r)),
                "map_max_abs_err": float(err.max()), "map_max_rel_err": float(rel.max()),
                "map_tolerance": "1e-5 relative (north star); p = 1 with a crop template is bit-exact",
                "ok": bool(ih_bad == 0 and rel.max() <= 1e-5)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None, help="ranks (default: WORLD_SIZE, else 1)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-rows", type=int, default=192,
                    help="rows of the frame in the bounded CPU sample (window rows = rows - 63)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the config-5 tracking-batch measurement")
    ap.add_argument("--no-next", action="store_true", help="skip the SURVEY 8(f) rows (SWIH, consumers, median)")
    ap.add_argument("--no-paths", action="store_true", help="skip the tensor-matcher / general-template lines")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--reduce", choices=["band", "root", "nccl"], default="band",
                    help="N > 1: band-owned reduce over peer memory (default), partials pushed into the "
                         "root's slots, or one NCCL reduce")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus is None:
        args.gpus = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch(args)
    run_ours(args)


if __name__ == "__main__":
    main()
