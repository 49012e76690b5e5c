#!/usr/bin/env python
"""Benchmark of the B200 integral-histogram + likelihood-map path (BASELINE.json metric).

One step = one frame through the hot path: quantise a 4096x4096 uint8 frame into
b bins, write the b-plane uint32 integral histogram to HBM, and produce the 64x64
sliding-window (Minkowski p = 1 / intersection) likelihood map (float64, W x H).
Throughput is Gbin*px/s = b * H * W / step time, whole job over all ranks.

  python bench.py [--gpus N --steps K --warmup W]          our arm (torchrun for N > 1)
  python bench.py --impl reference [...]                   the reference CPU path

Multi-GPU (N > 1): bin-slab sharding.  Rank r owns bins [128 r, 128 r + 128) of a
b = 128 N histogram over the same frame (weak scaling: fixed work per GPU); each rank's
sweep writes its slab of the integral histogram and its partial window sums; then
(--reduce band, default) every rank pulls one band of rows from all partials over peer
memory, sums and finalises them into rank 0's map; --reduce root pushes every partial
into a slot on rank 0, which finalises; --reduce nccl runs one NCCL reduce instead.

Extra lines of the JSON: build_only (plain build), c5_batch (config 5 tracking batch)
and next_rows (SWIH, map consumers, temporal median).

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
compute stream; a 256 MiB memset flushes L2 between steps outside the events;
barrier + synchronize on both sides; max over ranks.  `e2e` repeats the measurement
through the public API with the frame copied host->device and the map copied
device->host inside the timed region.  `roofline` reports the dominant kernel's
algorithmic bytes over its event-timed duration against MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import os
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
BINS_PER_GPU = 128
KW = KH = 64
P_ORDER = 1.0


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

def cpu_sample(rows: int = 128, reps: int = 1) -> dict:
    """The reference CPU path on a bounded sample of the same workload: the top `rows`
    rows of the 4096-wide frame, 128 bins, 64x64 p = 1 map.  build_integral_histogram
    with CrossWeaveTiled on every host thread + hist_distance_map (single-threaded as
    shipped).  Uses oracle/_ref (the unmodified reference) when built, else the C port."""
    import oracle  # CPU checker/baseline only — never on the measured GPU path

    frame = make_frame(W_IMG, H_IMG)[:rows]
    nb = BINS_PER_GPU
    tmpl = template_hist(make_frame(W_IMG, H_IMG), nb, KW, KH)
    threads = min(64, os.cpu_count() or 1)
    best = None
    kind = "reference" if oracle.have_ref() else "port"
    for _ in range(max(1, reps)):
        t0 = time.perf_counter()
        if kind == "reference":
            qb = oracle.ref_quantize(frame, nb)
            t = oracle.RefTensor(qb, nb, oracle.CW_TIS, 32, threads, budget=(1 << 64) - 1)
            t.hist_distance_map(tmpl, KW, KH, P_ORDER)
            del t
        else:
            qb = oracle.quantize(frame, nb)
            ih = oracle.build_ih(qb, nb)
            oracle.hist_distance_map(ih, tmpl, KW, KH, P_ORDER)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    value = nb * rows * W_IMG / best / 1e9
    return {"value": value, "unit": UNIT, "cores": threads if kind == "reference" else 1, "kind": kind,
            "sample": (f"top {rows} rows of the 4096x4096 frame ({rows - KH + 1} window rows), {nb} bins, "
                       f"64x64 p=1 map; IH build cw-tis x{threads} threads, hist_distance_map 1 thread "
                       f"(as shipped); best of {max(1, reps)}; {best:.2f} s"),
            "seconds": best}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    rows = args.ref_rows
    steps, warm = args.steps, args.warmup
    times = []
    for i in range(warm + steps):
        r = cpu_sample(rows, 1)
        if i >= warm:
            times.append(r["seconds"])
    sec = sum(times) / len(times)
    value = BINS_PER_GPU * rows * W_IMG / sec / 1e9
    kind = "reference" if oracle.have_ref() else "port"
    threads = min(64, os.cpu_count() or 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64/f64", "data": "synthetic",
        "config": {"workload": f"C3 sample: {rows}x4096 band of the 4096x4096 frame, 128 bins, 64x64 p=1 map",
                   "bins_total": BINS_PER_GPU, "window": [KW, KH], "p": P_ORDER},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm

def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


def box_peaks(dev) -> dict:
    """Copy and write-only bandwidth of this device, measured live ("also
    record a measured device write/copy peak on the box").  2 GiB buffers (> L2), torch's
    own copy_/fill_ kernels, CUDA events over 10 back-to-back launches each.  Outside
    every timed region; the sweep is write-dominated (8.6 GB written, 17 MB read), so the
    write peak is its tightest like-for-like denominator."""
    import torch

    n = 1 << 31  # bytes per buffer; int32 elements (torch's byte-wise fill runs at half speed)
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


def run_c5(P, dev, stream, args, frames: int = 100, side: int = 2048, nbins: int = 32, kw: int = 64, kh: int = 64):
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(5)
    rgb = torch.randint(0, 256, (frames, 3, side, side), dtype=torch.uint8, device=dev, generator=g)
    # templates: each channel's histogram of the centred kw x kh crop of frame 0
    srcs = P.channel_sources(rgb[0, 0], rgb[0, 1], rgb[0, 2], nbins)
    y0, x0 = (side - kh) // 2, (side - kw) // 2
    tdev = {}
    for c, s in srcs.items():
        if c == "orientation":
            qb = s
        else:
            qb = P.quantize(s, nbins)
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
    # 1. SWIH (swih.cpp:115-164, track_loop.cpp:264-283): 1024^2 BinMap, 32 bins, 31 x 31 kernel
    n, nb, k = 1024, 32, 31
    bm = torch.randint(0, nb, (n, n), dtype=torch.int16, device=dev, generator=g)
    model = np.full(nb, 1.0 / nb)
    ms_b = timed(lambda: P.swih.build_quadrant_set(bm, nb, k, k))
    out["swih_quadrant_set"] = line(f"{n}x{n} BinMap, {nb} bins, {k}x{k} kernel: four uint64 16.16 tensors", ms_b,
                                    4 * nb * n * n * 8 + n * n * 2)
    ms_m = timed(lambda: P.swih.swlh_distance_map(bm, nb, model, k, k))
    out["swih_distance_map"] = line("swlh-distance map (float64) in one sweep over the BinMap (no tensors; "
                                    "bound by the FP64 division per window and bin)", ms_m, n * n * 2 + n * n * 8)
    ms_q = timed(lambda: P.swih.swlh_distance_map(bm, nb, model, k, k, method="quadrant"))
    out["swih_distance_map_quadrant"] = line("the same map through the quadrant tensors (reference construction)",
                                             ms_q, 4 * nb * n * n * 8 + n * n * 2 + n * n * 8)
    # 2. map consumers (likelihood.cpp:257-330, tracker.cpp:77-113) at the C3 map size
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
    # 3. joint-IH temporal median (motion.cpp:35-99): 1024^2, 16 bins, 5-frame window, 7x7
    fr = [torch.randint(0, 16, (n, n), dtype=torch.uint8, device=dev, generator=g) for _ in range(8)]
    mb = P.motion.MedianBackgroundIH(fr[:5], 16, 7, 7)
    it = iter(range(10 ** 9))
    ms_sl = timed(lambda: mb.slide(fr[5 + next(it) % 3]))
    out["median_slide"] = line(f"{n}x{n}, 16 bins, 5 frames: joint tensor += IH(new), -= IH(old)", ms_sl,
                               2 * 2 * 16 * n * n * 4 + 2 * n * n)
    ms_bg = timed(lambda: mb.background())
    out["median_background"] = line("7x7 windows, per-pixel CDF walk over 16 bins", ms_bg, 16 * n * n * 4 + n * n)
    return out


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    from paper_1711_01656_b200.sharding import max_over_ranks, reduce_partials, slab_bounds

    nbins = BINS_PER_GPU * world
    bin0, bin1 = slab_bounds(nbins, world, rank)
    frame_h = make_frame(W_IMG, H_IMG)
    tmpl = template_hist(frame_h, nbins, KW, KH)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    frame = torch.from_numpy(frame_h).to(dev)
    tm = torch.from_numpy(tmpl).to(dev)
    t = P.IntegralHistogramTensor(W_IMG, H_IMG, nbins, bin0, BINS_PER_GPU, device=dev)
    nu, nv = W_IMG - KW + 1, H_IMG - KH + 1
    part = torch.empty((nv, nu), dtype=torch.float64, device=dev)
    lmap = torch.empty((H_IMG, W_IMG), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    peer, reduce_note = None, args.reduce
    if world > 1 and args.reduce in ("band", "root"):
        from paper_1711_01656_b200.sharding import PeerBandReduce, PeerSlabReduce

        try:  # fails on every rank or on none (the reducers agree on the outcome)
            peer = PeerBandReduce(W_IMG, H_IMG, KW, KH, device=dev) if args.reduce == "band" else \
                PeerSlabReduce(nu, nv, device=dev)
        except RuntimeError as e:  # no IPC / peer access between these GPUs: the NCCL reduce instead
            reduce_note = "nccl (peer setup failed: %s)" % str(e)[:120]
        if peer is not None and args.reduce == "band" and rank == 0:
            lmap = peer.map  # the final map lives in the shared buffer the band owners write

    def step(src):
        if world == 1:
            # every bin on this GPU: the sweep writes the finished map itself
            P.build_and_match_map(src, nbins, None, KW, KH, P_ORDER, out=t, lmap=lmap, tmpl_dev=tm)
            return
        if peer is not None and args.reduce == "band":
            # partials stay in each rank's HBM; every rank pulls its band of rows from all
            # partials over NVLink, sums and finalises them into rank 0's map
            peer.begin()
            P.build_and_match(src, nbins, None, KW, KH, P_ORDER, bin0=bin0, bins=bin1 - bin0, out=t,
                              partial=peer.slot(), tmpl_dev=tm)
            peer.publish()
            peer.finalize(P_ORDER)
            return
        if peer is not None:
            # the sweep writes its slab's partial map into its slot on rank 0 over NVLink;
            # rank 0 waits for every rank's flag, sums the slots while finalising
            peer.begin()
            P.build_and_match(src, nbins, None, KW, KH, P_ORDER, bin0=bin0, bins=bin1 - bin0, out=t,
                              partial=peer.slot(), tmpl_dev=tm)
            peer.publish()
            if rank == 0:
                peer.finalize(lmap, W_IMG, H_IMG, KW, KH, P_ORDER)
            return
        P.build_and_match(src, nbins, None, KW, KH, P_ORDER, bin0=bin0, bins=bin1 - bin0, out=t, partial=part,
                          tmpl_dev=tm)
        reduce_partials(part, dst=0)
        if rank == 0:
            P.hist_finalize(part, W_IMG, H_IMG, KW, KH, P_ORDER, out=lmap)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier()
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            fn()
            b.record(stream)
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in ev)
        return max_over_ranks(ms, None if shared else dev) / k

    for _ in range(args.warmup):
        step(frame)
    barrier()

    profiling.reset()
    profiling.enable(True)
    l0 = profiling.launch_count()
    with ClockSampler(local) as clk:
        ms = timed(lambda: step(frame), args.steps)
    launches = profiling.launch_count() - l0
    profiling.enable(False)
    kernels = {}
    for name in ("ih_sweep", "ih_sweep_match", "match_partial"):
        kt, kn = profiling.kernel_time(name)
        if kn:
            kernels[name] = (kt / kn, kn)
    profiling.reset()

    # plain build (BASELINE config "4096x4096 WAMI frame, 128-bin integral histogram on 1 B200"):
    # the drop-in build_integral_histogram path alone, same frame, same timing protocol
    build_only = None
    if world == 1:
        def build_step():
            P.build_integral_histogram(frame, nbins, memory_budget=None, out=t, validate=False)
        for _ in range(args.warmup):
            build_step()
        profiling.reset()
        profiling.enable(True)
        ms_b = timed(build_step, args.steps)
        profiling.enable(False)
        kt, kn = profiling.kernel_time("ih_sweep")
        profiling.reset()
        alg_b = BINS_PER_GPU * W_IMG * H_IMG * 4 + W_IMG * H_IMG
        build_only = {"ms_per_step": round(ms_b, 4), "value": round(nbins * W_IMG * H_IMG / (ms_b * 1e-3) / 1e9, 2),
                      "unit": UNIT, "kernel": "ih_sweep",
                      "kernel_ms": round(kt / kn, 4) if kn else None,
                      "frac": round(alg_b / (kt / kn * 1e-3) / 1e9 / peaks()["hbm_gbs"], 4) if kn else None,
                      "alg_bytes": alg_b}

    # tracking batch (BASELINE config 5): 100 synthetic 2048x2048 RGB frames x 32 bins, five
    # feature channels (intensity, gradient orientation, R, G, B) -> five likelihood maps per
    # frame, each channel one fused quantise -> integral histogram -> map sweep; frames resident
    nxt = None
    if world == 1 and not args.no_next:
        nxt = run_next_rows(P, dev, peaks()["hbm_gbs"])

    c5 = None
    if world == 1 and not args.no_c5:
        c5 = run_c5(P, dev, stream, args)

    # end to end through the public API: pinned host frame in, host map out, every step
    host_frame = torch.from_numpy(frame_h).pin_memory()
    host_map = torch.empty((H_IMG, W_IMG), dtype=torch.float64).pin_memory()
    dframe = torch.empty_like(frame)

    def e2e_step():
        dframe.copy_(host_frame, non_blocking=True)
        step(dframe)
        if rank == 0:
            host_map.copy_(lmap, non_blocking=True)

    e2e_mode = "serial"
    if world == 1:
        # public pipeline API: K distinct pinned host frames in, K host maps out; copies of
        # frame n+1 / map n-1 overlap the sweep of frame n (double-buffered, 3 streams)
        from paper_1711_01656_b200.pipeline import FramePipeline

        pipe = FramePipeline(W_IMG, H_IMG, nbins, tmpl, KW, KH, P_ORDER, device=dev)
        hframes = FramePipeline.pinned_frames([make_frame(W_IMG, H_IMG, seed=100 + i) for i in range(args.steps)])
        hmaps = pipe.pinned_maps(2)
        ring = [hmaps[i & 1] for i in range(args.steps)]
        pipe.run(hframes[:max(1, args.warmup)], ring[:max(1, args.warmup)])
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(pipe.h2d)
        pipe.run(hframes, ring)
        ev1.record(pipe.d2h)
        barrier()
        ms_e2e = ev0.elapsed_time(ev1) / args.steps
        e2e_mode = "pipelined (FramePipeline: H2D / sweep / D2H on three streams, double-buffered)"
    else:
        for _ in range(max(1, args.warmup)):
            e2e_step()
        ms_e2e = timed(e2e_step, args.steps)

    if peer is not None:
        if peer.error():
            raise SystemExit("bench.py: a peer-reduce wait timed out")
        peer.close()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    total_binpx = nbins * W_IMG * H_IMG
    value = total_binpx / (ms * 1e-3) / 1e9
    pk = peaks()
    # dominant kernel: the largest share of the step
    dom = max(kernels.items(), key=lambda kv: kv[1][0]) if kernels else None
    roof = None
    if dom is not None:
        name, (kms, kn) = dom
        binpx = BINS_PER_GPU * W_IMG * H_IMG
        if name == "match_partial":
            alg = binpx * 4 + nu * nv * 8  # standalone matcher: IH read once + partial write
        elif name == "ih_sweep_match":
            # IH write + frame read + map write (N = 1: finished W x H map; N > 1: partial nu x nv)
            alg = binpx * 4 + W_IMG * H_IMG + (W_IMG * H_IMG * 8 if world == 1 else nu * nv * 8)
        else:
            alg = binpx * 4 + W_IMG * H_IMG  # IH write + frame read
        achieved = alg / (kms * 1e-3) / 1e9
        tr = ncu_traffic(name)
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": tr, "kernel": name,
                "kernel_ms": round(kms, 4), "step_share": round(kms / ms, 3), "alg_bytes": alg,
                "peak_source": pk["source"],
                "kernels_ms": {k: round(v[0], 4) for k, v in kernels.items()}}
        try:
            bx = box_peaks(dev)
            bx["frac_vs_copy"] = round(achieved / bx["copy_gbs"], 4)
            bx["frac_vs_write"] = round(achieved / bx["write_gbs"], 4)
            roof["box_measured"] = bx
        except RuntimeError as e:  # e.g. no room for the 4 GiB of probe buffers
            roof["box_measured"] = {"unavailable": str(e).splitlines()[0]}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
        "config": {"workload": ("C3: 4096x4096 uint8 frame -> quantise -> %d-bin uint32 integral histogram "
                                "+ 64x64 p=1 likelihood map (float64)" % nbins),
                   "bins_total": nbins, "bins_per_gpu": BINS_PER_GPU, "window": [KW, KH], "p": P_ORDER,
                   "parallelism": f"bin-slab x{world}" + (
                       "" if world == 1 else (
                           " + band-owned reduce over peer memory (each rank pulls and finalises a band of rows)"
                           if peer is not None and args.reduce == "band" else
                           " + partial maps written to rank 0 over peer memory" if peer is not None
                           else " + NCCL reduce of partial maps")),
                   **({"reduce": reduce_note} if world > 1 else {}),
                   **({"shared_gpu": True} if shared else {}),
                   "l2": "256 MiB memset between timed steps (outside the events); step writes 8.6 GB/GPU"},
        "roofline": roof,
        "e2e": {"value": round(total_binpx / (ms_e2e * 1e-3) / 1e9, 2), "unit": UNIT,
                "h2d_bytes_per_step": W_IMG * H_IMG * world, "d2h_bytes_per_step": W_IMG * H_IMG * 8,
                "ms_per_step": round(ms_e2e, 4), "mode": e2e_mode},
        "gpu_launches": int(launches),
        "build_only": build_only,
        "c5_batch": c5,
        "next_rows": nxt,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_sample(args.ref_rows, 1)
            line["cpu_baseline"].pop("seconds", None)
        except Exception as e:  # the baseline is reported, never required for the GPU number
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-rows", type=int, default=192,
                    help="rows of the frame in the bounded CPU sample (window rows = rows - 63)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the config-5 tracking-batch measurement")
    ap.add_argument("--no-next", action="store_true", help="skip the SURVEY 8(f) rows (SWIH, consumers, median)")
    ap.add_argument("--reduce", choices=["band", "root", "nccl"], default="band",
                    help="N > 1: band-owned reduce over peer memory (default), partials pushed into the "
                         "root's slots, or one NCCL reduce")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
