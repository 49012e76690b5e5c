"""GPU parity: the CUDA path against the CPU oracle and the reference's golden vectors.

Bars (BASELINE.json north star):
  * integral histograms: bit-exact, uint32 device cells == uint64 oracle cells, padding included;
  * likelihood maps: Minkowski p = 1 over a full-bin tensor is bit-exact (same operation
    order as likelihood.cpp:211-221); other p / metrics / slab sums within
    |g - r| <= 1e-5 * |r| + 1e-12 (RTOL/ATOL below).
Sizes are the reference's own awkward sizes (test_integral.cpp:74) plus strip / band
boundaries of the device sweep; full-size configs are covered by size-independent
properties in test_gpu_properties.py.
"""
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-5, 1e-12


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1711_01656_b200 as P

    return P


@pytest.fixture
def band_rows(monkeypatch):
    def set_rows(n):
        monkeypatch.setenv("SPCT_BAND_ROWS", str(n))
    return set_rows


def close(g, r):
    return np.all(np.abs(g - r) <= RTOL * np.abs(r) + ATOL)


def test_golden_reference_tensors(P, golden):
    vec = golden[1]
    for key in [k for k in vec if k.endswith("_tensor")]:
        bm = vec[key.replace("_tensor", "_bins")]
        t = P.build_integral_histogram(bm, 16)
        assert np.array_equal(t.padded_u64(), vec[key]), key


def test_known_answers(P, golden):
    kn = golden[0]
    k = kn["ih_2x2"]
    t = P.build_integral_histogram(np.array(k["binmap"], np.uint16), k["bins"])
    for kk, y, x, v in k["expect_at"]:
        assert t.at(kk, y, x) == v
    a = t.padded_u64()
    assert not a[:, 0, :].any() and not a[:, :, 0].any()
    k = kn["ih_1x1"]
    t = P.build_integral_histogram(np.array(k["binmap"], np.uint16), k["bins"])
    assert np.argwhere(t.padded_u64()).tolist() == [e[:3] for e in k["nonzero"]]
    q = kn["quantize_32"]
    img = np.array([q["pixels"]], np.uint8)
    assert P.api.as_numpy_u16(P.quantize(img, 32)).tolist() == [q["expect"]]
    c = kn["quantize_clamp"]
    out = P.api.as_numpy_u16(P.quantize(img, c["bins"], c["lo"], c["hi"]))
    assert out[0, 0] == c["expect_first"] and out[0, -1] == c["expect_last"]
    for bins, lo, hi in kn["quantize_contract"]["bad"]:
        with pytest.raises(P.ContractError):
            P.quantize(img, bins, lo, hi)
    g = kn["grayscale"]
    rgb = np.array(g["rgb"], np.uint8)
    gray = P.to_grayscale(rgb[None, :, 0], rgb[None, :, 1], rgb[None, :, 2]).cpu().numpy()
    assert gray.tolist() == [g["expect"]]
    f = kn["hist_fixture_0p7"]
    t = P.build_integral_histogram(np.array(f["image"], np.uint8), f["bins"])
    m = P.hist_distance_map(t, f["template"], f["kw"], f["kh"], f["p"]).cpu().numpy()
    assert abs(m[f["at"][1], f["at"][0]] - f["expect"]) <= f["eps"]


SIZES = [(1, 1), (5, 3), (33, 31), (64, 64), (70, 129), (256, 40), (127, 5), (128, 9), (129, 300), (383, 77),
         (513, 260)]


@pytest.mark.parametrize("w,h", SIZES)
@pytest.mark.parametrize("bins", [1, 3, 16, 37])
def test_ih_bit_exact_binmap(P, w, h, bins):
    bm = oracle.random_binmap(w, h, bins, 1000 + w * 7 + h + bins)
    t = P.build_integral_histogram(bm, bins)
    assert np.array_equal(t.padded_u64(), oracle.build_ih(bm, bins))


@pytest.mark.parametrize("rows", [1, 2, 7, 64])
def test_ih_band_carries(P, band_rows, rows):
    band_rows(rows)
    for (w, h, bins) in [(70, 129, 16), (300, 150, 9), (257, 64, 33)]:
        bm = oracle.random_binmap(w, h, bins, rows * 31 + w)
        t = P.build_integral_histogram(bm, bins)
        assert np.array_equal(t.padded_u64(), oracle.build_ih(bm, bins)), (rows, w, h, bins)


@pytest.mark.parametrize("bins", [2, 4, 5, 8, 9, 16, 17, 32, 64, 100, 128, 200, 256])
def test_ih_bin_counts(P, bins):
    img = oracle.smooth_image(300, 97, bins)
    bm = oracle.quantize(img, bins)
    t = P.build_integral_histogram(bm, bins)
    assert np.array_equal(t.padded_u64(), oracle.build_ih(bm, bins))


def test_ih_sources_fused_quantize(P):
    """gray u8 (fast and general lo/hi), planar RGB and float64 sources quantise in the load stage."""
    g = oracle.noise_image(301, 133, 5)
    for bins, lo, hi in [(16, 0.0, 256.0), (32, 0.0, 256.0), (7, 30.0, 200.0), (300, 0.0, 256.0), (5, -3.5, 97.25)]:
        t = P.build_integral_histogram(g, bins, lo=lo, hi=hi)
        want = oracle.build_ih(oracle.quantize(g, bins, lo, hi), bins)
        assert np.array_equal(t.padded_u64(), want), (bins, lo, hi)
    r, gg, b = oracle.noise_color(150, 77, 1)
    t = P.build_integral_histogram((r, gg, b), 32)
    want = oracle.build_ih(oracle.quantize(oracle.to_grayscale(r, gg, b), 32), 32)
    assert np.array_equal(t.padded_u64(), want)
    rng = np.random.default_rng(3)
    s = rng.normal(0.0, 50.0, (61, 140))
    s[0, :4] = [np.inf, -np.inf, 1e300, -1e300]  # out-of-int-range floor -> bin 0 like x86
    t = P.build_integral_histogram(s, 12, lo=-100.0, hi=100.0)
    want = oracle.build_ih(oracle.quantize(s, 12, -100.0, 100.0), 12)
    assert np.array_equal(t.padded_u64(), want)


def test_quantize_kernel_matches_reference(P, golden):
    vec = golden[1]
    gray = P.to_grayscale(vec["color_r"], vec["color_g"], vec["color_b"]).cpu().numpy()
    assert np.array_equal(gray, vec["color_gray"])
    assert np.array_equal(P.api.as_numpy_u16(P.quantize(gray, 32)), vec["color_q32"])
    assert np.array_equal(P.api.as_numpy_u16(P.quantize(gray, 7, 30.0, 200.0)), vec["color_q7_lohi"])
    v = np.arange(256, dtype=np.uint8)[None]
    for bins in [1, 3, 128, 255, 256, 1000, 65536]:
        assert np.array_equal(P.api.as_numpy_u16(P.quantize(v, bins)), oracle.quantize(v, bins))


@pytest.mark.parametrize("k0,k1", [(0, 5), (5, 16), (3, 4), (16, 37), (0, 37)])
def test_ih_bin_slab(P, k0, k1):
    bm = oracle.random_binmap(211, 97, 37, k0 * 100 + k1)
    t = P.build_integral_histogram(bm, 37, bin0=k0, bins=k1 - k0)
    assert np.array_equal(t.padded_u64(), oracle.build_ih(bm, 37, k0, k1))


def test_region_queries(P, golden):
    vec = golden[1]
    t = P.build_integral_histogram(vec["region_bins"], 32)
    got = P.region_histograms(t, vec["region_rects"])
    assert np.array_equal(got, vec["region_hists"])
    # exhaustive rects on 6x6 two-bin maps (test_integral.cpp:91-105)
    rng = oracle.Rng(4242)
    for trial in range(20):
        bm = rng.binmap(6, 6, 2)
        t = P.build_integral_histogram(bm, 2)
        rects = [[x1, y1, x2 - x1, y2 - y1] for y1 in range(7) for y2 in range(y1, 7) for x1 in range(7)
                 for x2 in range(x1, 7)]
        got = P.region_histograms(t, rects)
        ot = oracle.build_ih(bm, 2)
        want = np.stack([oracle.region_histogram(ot, *r) for r in rects])
        assert np.array_equal(got, want)
    t = P.build_integral_histogram(oracle.random_binmap(8, 8, 4, 5), 4)
    assert not P.region_histogram(t, 3, 3, 0, 0).any()
    with pytest.raises(P.ContractError):
        P.region_histogram(t, 5, 5, 4, 4)
    with pytest.raises(P.ContractError):
        P.region_histogram(t, -1, 0, 2, 2)
    with pytest.raises(P.ContractError):
        P.region_count(t, 9, 0, 0, 1, 1)


def test_build_contract_errors(P):
    bm = oracle.random_binmap(16, 16, 4, 3)
    bad = bm.copy()
    bad[0, 7] = 4
    with pytest.raises(P.ContractError):
        P.build_integral_histogram(bad, 4)
    with pytest.raises(P.ContractError):
        P.build_integral_histogram(bm, 4, memory_budget=64)
    with pytest.raises(P.ContractError):
        P.build_integral_histogram(np.zeros((0, 0), np.uint16), 4)
    with pytest.raises(P.ContractError):
        P.build_integral_histogram(bm, 4, P.ScanSchedule(3, 32, 0))


def test_maps_golden_reference(P, golden):
    vec = golden[1]
    t = P.build_integral_histogram(vec["lmap_noise_img"], 8)
    tm = np.full(8, 1 / 8)
    assert np.array_equal(P.hist_distance_map(t, tm, 7, 5, 1.0, exact=True).cpu().numpy(), vec["lmap_noise_p1"])
    assert close(P.hist_distance_map(t, tm, 7, 5, 1.0).cpu().numpy(), vec["lmap_noise_p1"])
    assert close(P.hist_distance_map(t, tm, 7, 5, 2.0).cpu().numpy(), vec["lmap_noise_p2"])
    assert close(P.hist_distance_map(t, tm, 7, 5, 2.0, exact=True).cpu().numpy(), vec["lmap_noise_p2"])
    t = P.build_integral_histogram(vec["lmap_smooth_img"], 16)
    th = vec["lmap_smooth_tmpl"]
    assert np.array_equal(P.hist_distance_map(t, th, 20, 16, 1.0, exact=True).cpu().numpy(), vec["lmap_smooth_p1"])
    assert close(P.hist_distance_map(t, th, 20, 16, 1.0).cpu().numpy(), vec["lmap_smooth_p1"])
    assert close(P.hist_distance_map(t, th, 20, 16, 3.0).cpu().numpy(), vec["lmap_smooth_p3"])


@pytest.mark.parametrize("w,h,bins,kw,kh", [(96, 80, 16, 20, 16), (130, 67, 9, 13, 11), (257, 140, 32, 64, 64),
                                            (50, 40, 5, 50, 40), (61, 33, 24, 1, 1), (200, 100, 128, 31, 17)])
def test_maps_vs_oracle(P, w, h, bins, kw, kh):
    img = oracle.smooth_image(w, h, w + h)
    qb = oracle.quantize(img, bins)
    y0, x0 = (h - kh) // 3, (w - kw) // 2
    crop = qb[y0:y0 + kh, x0:x0 + kw]
    th = np.bincount(crop.reshape(-1), minlength=bins).astype(np.float64) / crop.size
    t = P.build_integral_histogram(img, bins)
    want = oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0)
    got = P.hist_distance_map(t, th, kw, kh, 1.0, exact=True).cpu().numpy()
    assert np.array_equal(got, want)  # tensor path: the reference's rounding sequence
    assert close(P.hist_distance_map(t, th, kw, kh, 1.0).cpu().numpy(), want)  # source path
    assert got[y0 + (kh - 1) // 2, x0 + (kw - 1) // 2] == 1.0  # the template's own window
    for p in (1.5, 2.0, 3.0):
        assert close(P.hist_distance_map(t, th, kw, kh, p, exact=True).cpu().numpy(),
                     oracle.hist_match_map_direct(qb, bins, th, kw, kh, p))
        assert close(P.hist_distance_map(t, th, kw, kh, p).cpu().numpy(),
                     oracle.hist_match_map_direct(qb, bins, th, kw, kh, p))
    for metric in (1, 2, 3):  # extensions: parity against the self-written oracle definitions
        assert close(P.hist_match_map(t, th, kw, kh, 1.0, metric).cpu().numpy(),
                     oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0, metric))


def test_map_contracts(P):
    t = P.build_integral_histogram(oracle.random_binmap(30, 22, 8, 1), 8)
    good = np.full(8, 1 / 8)
    for args in [(good, 7, 5, 0.5), (good, 31, 5, 1.0), (np.full(9, 1 / 9), 7, 5, 1.0), (good * 2, 7, 5, 1.0)]:
        with pytest.raises(P.ContractError):
            P.hist_distance_map(t, *args)


@pytest.mark.parametrize("p,metric", [(1.0, 0), (2.0, 0), (1.0, 1), (1.0, 2), (1.0, 3)])
def test_slab_partials_recompose(P, p, metric):
    """Bin-slab sharding (what each GPU computes before the NCCL reduce)."""
    img = oracle.smooth_image(190, 120, 77)
    bins, kw, kh = 40, 24, 18
    qb = oracle.quantize(img, bins)
    crop = qb[40:58, 60:84]
    th = np.bincount(crop.reshape(-1), minlength=bins).astype(np.float64) / crop.size
    tm = torch.from_numpy(th).cuda()
    acc = None
    for k0, k1 in [(0, 13), (13, 27), (27, 40)]:
        t = P.build_integral_histogram(img, bins, bin0=k0, bins=k1 - k0)
        part = P.hist_partial(t, tm, kw, kh, p, metric)
        acc = part if acc is None else acc + part
    got = P.hist_finalize(acc, 190, 120, kw, kh, p, metric).cpu().numpy()
    assert close(got, oracle.hist_match_map_direct(qb, bins, th, kw, kh, p, metric))


@pytest.mark.parametrize("slabs", [1, 2, 5])
def test_fused_build_match(P, slabs):
    img = oracle.smooth_image(333, 211, 9)
    bins, kw, kh = 48, 64, 64
    qb = oracle.quantize(img, bins)
    crop = qb[100:164, 150:214]
    th = np.bincount(crop.reshape(-1), minlength=bins).astype(np.float64) / crop.size
    edges = np.linspace(0, bins, slabs + 1).astype(int)
    acc = None
    for k0, k1 in zip(edges[:-1], edges[1:]):
        t, part = P.build_and_match(img, bins, th, kw, kh, 1.0, bin0=int(k0), bins=int(k1 - k0))
        assert np.array_equal(t.padded_u64(), oracle.build_ih(qb, bins, int(k0), int(k1)))
        acc = part.clone() if acc is None else acc + part
    got = P.hist_finalize(acc, 333, 211, kw, kh, 1.0).cpu().numpy()
    want = oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0)
    assert close(got, want)


def _crop_template(qb, bins, x0, y0, kw, kh):
    crop = qb[y0:y0 + kh, x0:x0 + kw]
    return np.bincount(crop.reshape(-1), minlength=bins).astype(np.float64) / crop.size


FUSED_CASES = [  # w, h, bins, kw, kh
    (333, 211, 48, 64, 64), (130, 67, 9, 13, 11), (257, 140, 130, 64, 64), (300, 200, 128, 128, 100),
    (97, 301, 20, 1, 1), (128, 128, 16, 127, 5), (45, 33, 7, 45, 33), (700, 90, 256, 31, 17), (520, 260, 33, 65, 3),
    # kw * kh > 24576: the unsigned 16-bit window-count path (kw = 128 and a general kw)
    (260, 300, 24, 128, 255), (310, 280, 40, 100, 250)]


@pytest.mark.parametrize("w,h,bins,kw,kh", FUSED_CASES)
@pytest.mark.parametrize("store", [True, False])
def test_fused_integral_template(P, w, h, bins, kw, kh, store):
    """Template = histogram of a kw x kh crop (integral s_k): the exact integer path."""
    img = oracle.smooth_image(w, h, w * 3 + h)
    qb = oracle.quantize(img, bins)
    th = _crop_template(qb, bins, (w - kw) // 3, (h - kh) // 2, kw, kh)
    want = oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0)
    if store:
        t, part = P.build_and_match(img, bins, th, kw, kh, 1.0)
        assert np.array_equal(t.padded_u64(), oracle.build_ih(qb, bins))
    else:
        t = P.IntegralHistogramTensor(w, h, bins)
        t.desc.data = None
        _, part = P.build_and_match(img, bins, th, kw, kh, 1.0, out=t)
    got = P.hist_finalize(part, w, h, kw, kh, 1.0).cpu().numpy()
    assert close(got, want)
    inter = oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0, oracle.INTERSECTION)
    _, part = P.build_and_match(img, bins, th, kw, kh, 1.0, 1)
    assert close(P.hist_finalize(part, w, h, kw, kh, 1.0, 1).cpu().numpy(), inter)


@pytest.mark.parametrize("w,h,bins,kw,kh", FUSED_CASES + [(300, 290, 100, 64, 50), (260, 140, 64, 128, 128)])
@pytest.mark.parametrize("store", [True, False])
def test_fused_map_direct(P, w, h, bins, kw, kh, store):
    """spct_cu_ih_build_match_map: finished map (incl. spread_valid borders) in the sweep."""
    img = oracle.smooth_image(w, h, w + 5 * h)
    qb = oracle.quantize(img, bins)
    th = _crop_template(qb, bins, (w - kw) // 2, (h - kh) // 3, kw, kh)
    t = P.IntegralHistogramTensor(w, h, bins)
    if not store:
        t.desc.data = None
    _, lmap = P.build_and_match_map(img, bins, th, kw, kh, 1.0, out=t)
    assert close(lmap.cpu().numpy(), oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0))
    if store:
        assert np.array_equal(t.padded_u64(), oracle.build_ih(qb, bins))
    rng = np.random.default_rng(w)
    tg = rng.random(bins)
    tg /= tg.sum()
    for p, metric in [(1.0, 0), (2.0, 0), (1.0, 1), (1.0, 3)]:
        _, lmap = P.build_and_match_map(img, bins, tg, kw, kh, p, metric, out=t)
        assert close(lmap.cpu().numpy(), oracle.hist_match_map_direct(qb, bins, tg, kw, kh, p, metric)), (p, metric)


def test_frame_pipeline_matches_single_frames(P):
    from paper_1711_01656_b200.pipeline import FramePipeline

    w, h, bins, kw, kh = 300, 220, 64, 64, 48
    frames = [oracle.smooth_image(w, h, 500 + i) for i in range(5)]
    qb0 = oracle.quantize(frames[0], bins)
    th = _crop_template(qb0, bins, 100, 80, kw, kh)
    pipe = FramePipeline(w, h, bins, th, kw, kh, 1.0)
    hf = FramePipeline.pinned_frames(frames)
    hm = pipe.pinned_maps(len(frames))
    pipe.run(hf, hm)
    for f, m in zip(frames, hm):
        qb = oracle.quantize(f, bins)
        assert close(m.numpy(), oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0))
    # the tensor of the last frame stays resident
    assert np.array_equal(pipe.tensor.padded_u64(), oracle.build_ih(oracle.quantize(frames[-1], bins), bins))


def test_fused_map_rejects_slabs(P):
    img = oracle.smooth_image(100, 80, 1)
    t = P.IntegralHistogramTensor(100, 80, 32, bin0=16, bins=16)
    with pytest.raises(P.ContractError):
        P.build_and_match_map(img, 32, np.full(32, 1 / 32), 16, 16, 1.0, out=t)


def _blocky_image(w, h, seed):
    """Uniform blocks (one bin over whole windows) beside a noisy patch: window counts of
    kw * kh in one bin against template counts below 16 (negative min thresholds in the
    integer path)."""
    rng = np.random.default_rng(seed)
    img = np.zeros((h, w), np.uint8)
    img[:, w // 2:] = 255
    img[h // 3:2 * h // 3, :] = 130
    y0, x0 = h // 4, w // 4
    img[y0:y0 + 90, x0:x0 + 90] = rng.integers(20, 120, (90, 90), dtype=np.uint8)  # no block bin
    return img


@pytest.mark.parametrize("bins,kw,kh", [(16, 64, 64), (128, 64, 64), (40, 33, 21), (200, 128, 100)])
@pytest.mark.parametrize("general", [False, True])
def test_fused_uniform_regions(P, bins, kw, kh, general):
    """Windows entirely inside one bin next to templates with few (< 16) pixels of that bin."""
    w, h = 420, 330
    img = _blocky_image(w, h, bins)
    qb = oracle.quantize(img, bins)
    y0, x0 = h // 4, w // 4
    th = _crop_template(qb, bins, x0 + 90 - kw + 3, y0 + 90 - kh + 2, kw, kh)  # crop: 3 x 2 pixels of a block
    if general:
        th = th * 0.97 + 0.03 / bins
    for metric in (0, 1):
        want = oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0, metric)
        for store in (True, False):
            t = P.IntegralHistogramTensor(w, h, bins)
            if not store:
                t.desc.data = None
            _, lmap = P.build_and_match_map(img, bins, th, kw, kh, 1.0, metric, out=t)
            got = lmap.cpu().numpy()
            assert close(got, want), (metric, store, np.abs(got - want).max())


@pytest.mark.parametrize("bins,kw,kh", [(128, 64, 64), (48, 33, 17), (200, 40, 40)])
@pytest.mark.parametrize("p,metric", [(1.0, 0), (2.0, 0), (1.0, 1), (1.0, 2), (1.0, 3)])
def test_fused_near_zero_likelihoods(P, bins, kw, kh, p, metric):
    """Templates whose mass sits on bins most windows lack (likelihoods down to ~1e-6): the
    fractional (p = 1 / intersection) and integer / FP32 (p = 2, Bhattacharyya, chi-square)
    paths keep the relative tolerance where the map is near 0."""
    w, h = 380, 260
    img = oracle.smooth_image(w, h, bins + kw)
    qb = oracle.quantize(img, bins)
    cnt = np.bincount(qb.reshape(-1), minlength=bins).astype(np.float64)
    rng = np.random.default_rng(bins * kh)
    th = rng.random(bins) * 1e-6
    rare = np.argsort(cnt)[: max(2, bins // 8)]  # the least frequent bins carry the mass
    th[rare] += rng.random(rare.size)
    th /= th.sum()
    for store in (True, False):
        t = P.IntegralHistogramTensor(w, h, bins)
        if not store:
            t.desc.data = None
        _, lmap = P.build_and_match_map(img, bins, th, kw, kh, p, metric, out=t)
        want = oracle.hist_match_map_direct(qb, bins, th, kw, kh, p, metric)
        got = lmap.cpu().numpy()
        assert close(got, want), (store, np.abs(got - want).max(), want.min())


@pytest.mark.parametrize("w,h,bins,kw,kh", FUSED_CASES[:6])
@pytest.mark.parametrize("p,metric", [(1.0, 0), (2.0, 0), (1.7, 0), (1.0, 1), (1.0, 2), (1.0, 3)])
def test_fused_general_template(P, w, h, bins, kw, kh, p, metric):
    """Non-integral template (random weights): the FP64 per-bin path."""
    img = oracle.noise_image(w, h, w + 7 * h)
    qb = oracle.quantize(img, bins)
    rng = np.random.default_rng(w * h)
    th = rng.random(bins)
    th /= th.sum()
    t, part = P.build_and_match(img, bins, th, kw, kh, p, metric)
    got = P.hist_finalize(part, w, h, kw, kh, p, metric).cpu().numpy()
    assert close(got, oracle.hist_match_map_direct(qb, bins, th, kw, kh, p, metric))


@pytest.mark.parametrize("rows", [1, 5, 64, 100])
@pytest.mark.parametrize("bins", [40, 24])
def test_fused_bands(P, band_rows, rows, bins):
    """Forced band heights: band tops start from the window-start carry tables (bins <= 64,
    narrow CTAs) with the window start in the band above, further up, or above row 0."""
    band_rows(rows)
    w, h, kw, kh = 290, 173, 64, 37
    img = oracle.smooth_image(w, h, rows)
    qb = oracle.quantize(img, bins)
    th = _crop_template(qb, bins, 100, 60, kw, kh)
    t, part = P.build_and_match(img, bins, th, kw, kh, 1.0)
    assert np.array_equal(t.padded_u64(), oracle.build_ih(qb, bins))
    assert close(P.hist_finalize(part, w, h, kw, kh, 1.0).cpu().numpy(),
                 oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0))


def test_fused_sources_and_slabs(P):
    r, g, b = oracle.noise_color(403, 150, 2)
    gray = oracle.to_grayscale(r, g, b)
    bins, kw, kh = 200, 64, 64
    qb = oracle.quantize(gray, bins)
    th = _crop_template(qb, bins, 200, 40, kw, kh)
    acc = None
    for k0, k1 in [(0, 77), (77, 200)]:
        t, part = P.build_and_match((r, g, b), bins, th, kw, kh, 1.0, bin0=k0, bins=k1 - k0)
        assert np.array_equal(t.padded_u64(), oracle.build_ih(qb, bins, k0, k1))
        acc = part.clone() if acc is None else acc + part
    assert close(P.hist_finalize(acc, 403, 150, kw, kh, 1.0).cpu().numpy(),
                 oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0))


def test_fused_large_window_falls_back(P):
    w, h, bins, kw, kh = 300, 280, 12, 200, 150
    img = oracle.smooth_image(w, h, 4)
    qb = oracle.quantize(img, bins)
    th = _crop_template(qb, bins, 50, 60, kw, kh)
    t, part = P.build_and_match(img, bins, th, kw, kh, 1.0)
    assert np.array_equal(P.hist_finalize(part, w, h, kw, kh, 1.0).cpu().numpy(),
                          oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0))


@pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")
def test_against_live_reference(P):
    img = oracle.noise_image(57, 43, 3)
    qb = oracle.ref_quantize(img, 9)
    rt = oracle.RefTensor(qb, 9, oracle.WF_TIS, 32, 4)
    t = P.build_integral_histogram(img, 9)
    assert np.array_equal(t.padded_u64(), rt.array())
    crop = qb[10:21, 5:18]
    th = np.bincount(crop.reshape(-1), minlength=9).astype(np.float64) / crop.size
    assert np.array_equal(P.hist_distance_map(t, th, 13, 11, 1.0, exact=True).cpu().numpy(),
                          rt.hist_distance_map(th, 13, 11, 1.0))


# ------------------------------------------------------------------ tracking batch (config 5)

@pytest.mark.parametrize("w,h,sigma,bins", [(1, 1, 1.0, 8), (64, 48, 1.0, 32), (300, 211, 1.0, 32), (131, 97, 1.5, 16),
                                            (257, 140, 0.0, 9)])
def test_orientation_bins_exact(P, w, h, sigma, bins):
    """Device orientation BinMap == the oracle restatement (== the reference, test_oracle.py)."""
    for img in (oracle.smooth_image(w, h, w + 2 * h), oracle.noise_image(w, h, 3 * w + h)):
        got = P.api.as_numpy_u16(P.orientation_bins(img, bins, sigma))
        assert np.array_equal(got, oracle.orientation_bins(img, bins, sigma))


@pytest.mark.parametrize("bins", [32, 8, 12, 256, 300])
def test_orientation_bins_on_bin_boundaries(P, bins):
    """Ramps whose gradient ratio dy/dx sits exactly on (or next to) a bin boundary
    (q = 0, +-1, +-2, +-1/2, ...): the boundary search hands those pixels to the reference
    formula; bins > 256 take the formula everywhere.  Plus tiles with flat and dx == 0
    regions, a 1-pixel-wide and a 1-pixel-tall frame."""
    h, w = 70, 150
    y, x = np.mgrid[0:h, 0:w]
    imgs = [(x + y) % 256, (x - y) % 256, (2 * x + y) % 256, (x + 2 * y) % 256, (3 * y) % 256, np.full((h, w), 77),
            (x // 16 * 9 + y // 8 * 9) % 256]
    for img in imgs:
        img = np.ascontiguousarray(img, np.uint8)
        for sigma in (1.0, 0.0):
            got = P.api.as_numpy_u16(P.orientation_bins(img, bins, sigma))
            assert np.array_equal(got, oracle.orientation_bins(img, bins, sigma)), (bins, sigma)
    for img in (oracle.noise_image(1, 97, 5), oracle.noise_image(131, 1, 6)):
        got = P.api.as_numpy_u16(P.orientation_bins(img, bins, 1.0))
        assert np.array_equal(got, oracle.orientation_bins(img, bins, 1.0))


@pytest.mark.parametrize("frames", [2])
def test_tracking_batch_channels(P, frames):
    """Config 5 in miniature: per frame, intensity / orientation / R / G / B likelihood maps
    (fused build + match per channel) against the oracle on each channel's BinMap."""
    w, h, nbins, kw, kh = 280, 190, 32, 32, 24
    x0, y0 = 120, 70
    for f in range(frames):
        r, g, b = oracle.noise_color(w, h, 500 + f) if f % 2 else (oracle.smooth_image(w, h, 600 + f),
                                                                  oracle.smooth_image(w, h, 700 + f),
                                                                  oracle.smooth_image(w, h, 800 + f))
        gray = oracle.to_grayscale(r, g, b)
        chan_bins = {"intensity": oracle.quantize(gray, nbins), "orientation": oracle.orientation_bins(gray, nbins, 1.0),
                     "red": oracle.quantize(r, nbins), "green": oracle.quantize(g, nbins),
                     "blue": oracle.quantize(b, nbins)}
        templates = {c: _crop_template(qb, nbins, x0, y0, kw, kh) for c, qb in chan_bins.items()}
        maps = P.likelihood_channels(r, g, b, nbins, templates, kw, kh, 1.0)
        assert set(maps) == set(P.CHANNELS)
        for c, qb in chan_bins.items():
            want = oracle.hist_match_map_direct(qb, nbins, templates[c], kw, kh, 1.0)
            got = maps[c].cpu().numpy()
            assert close(got, want), c
            assert got[y0 + (kh - 1) // 2, x0 + (kw - 1) // 2] == 1.0, c  # the template's own window


# ------------------------------------------------------------------ IHT1 wire format

@pytest.mark.parametrize("w,h,bins", [(1, 1, 8), (70, 129, 16), (257, 140, 37)])
def test_iht1_dump_is_byte_identical_to_reference(P, tmp_path, w, h, bins):
    """dump_tensor of the device tensor == the reference's dump_tensor of the same BinMap
    (integral.cpp:619-633), and both load back (either loader) to the same tensor."""
    bm = oracle.random_binmap(w, h, bins, 900 + w)
    t = P.build_integral_histogram(bm, bins)
    mine, ref = tmp_path / "mine.iht", tmp_path / "ref.iht"
    P.dump_tensor(t, mine)
    if oracle.have_ref():
        oracle.RefTensor(bm, bins).dump(ref)
        assert mine.read_bytes() == ref.read_bytes()
        assert np.array_equal(oracle.RefTensor.load(mine).array(), oracle.build_ih(bm, bins))
        assert np.array_equal(P.load_tensor(ref).padded_u64(), oracle.build_ih(bm, bins))
    assert np.array_equal(P.load_tensor(mine).padded_u64(), oracle.build_ih(bm, bins))


def test_iht1_chunked_and_elem4(P, tmp_path):
    """A plane larger than one 32 MiB staging chunk, and the elem_bytes = 4 extension."""
    w, h, bins = 2304, 1900, 3
    img = oracle.smooth_image(w, h, 77)
    t = P.build_integral_histogram(img, bins)
    want = t.padded_u64()
    p8, p4 = tmp_path / "t8.iht", tmp_path / "t4.iht"
    P.dump_tensor(t, p8)
    P.dump_tensor(t, p4, elem_bytes=4)
    assert p8.stat().st_size == 20 + want.size * 8 and p4.stat().st_size == 20 + want.size * 4
    hdr = np.frombuffer(p8.read_bytes()[:20][4:], np.uint32)
    assert list(hdr) == [bins, h, w, 8]
    assert np.array_equal(np.fromfile(p8, np.uint64, offset=20).reshape(want.shape), want)
    assert np.array_equal(P.load_tensor(p8).padded_u64(), want)
    assert np.array_equal(P.load_tensor(p4).padded_u64(), want)


def test_iht1_weighted_tensor_round_trip(P, tmp_path):
    """A weighted tensor with cells beyond 2^32 dumps like the reference and loads back
    with uint64 cells (a WeightedTensor), as the reference's load_tensor keeps them."""
    rng = np.random.default_rng(3)
    bm = rng.integers(0, 5, (23, 31)).astype(np.uint16)
    wts = (np.uint64(1) << np.uint64(31)) + rng.integers(0, 1 << 20, (23, 31)).astype(np.uint64)
    wt = P.swih.build_weighted_tensor(bm, wts, 5)
    path = str(tmp_path / "w.iht")
    want = wt.padded_u64()
    header = np.array([5, 23, 31, 8], "<u4").tobytes()
    with open(path, "wb") as f:  # the reference's IHT1 layout (integral.cpp:619-631)
        f.write(b"IHT1" + header + want.astype("<u8").tobytes())
    got = P.load_tensor(path)
    assert isinstance(got, P.swih.WeightedTensor)
    assert np.array_equal(got.padded_u64(), want)
    assert want.max() > (1 << 32)


def test_iht1_load_rejects_bad_payloads(P, tmp_path):
    bm = oracle.random_binmap(9, 6, 4, 3)
    t = P.build_integral_histogram(bm, 4)
    good = tmp_path / "g.iht"
    P.dump_tensor(t, good)
    raw = bytearray(good.read_bytes())
    (tmp_path / "trunc.iht").write_bytes(bytes(raw[:-8]))
    with pytest.raises(P.SpctError, match="truncated tensor payload"):  # integral.cpp:655
        P.load_tensor(tmp_path / "trunc.iht")
    pad = bytearray(raw)
    pad[20:28] = (1).to_bytes(8, "little")  # cell (0, 0, 0) is padding
    (tmp_path / "pad.iht").write_bytes(bytes(pad))
    with pytest.raises(P.SpctError, match="nonzero padding"):
        P.load_tensor(tmp_path / "pad.iht")
    big = bytearray(raw)
    off = 20 + 8 * (1 * 10 + 1)  # plane 0, row 1, column 1
    big[off:off + 8] = (1 << 33).to_bytes(8, "little")
    (tmp_path / "big.iht").write_bytes(bytes(big))
    wt = P.load_tensor(tmp_path / "big.iht")  # cells beyond 2^32: uint64 cells, as the reference keeps them
    assert isinstance(wt, P.swih.WeightedTensor) and int(wt.padded_u64()[0, 1, 1]) == 1 << 33
    with pytest.raises(P.SpctError, match="cannot write tensor"):
        P.dump_tensor(t, "/nonexistent/dir/t.iht")


# ------------------------------------------------------------------ map consumers (§8(f) #2)

def _consumer_maps(seed):
    rng = np.random.default_rng(seed)
    img = oracle.smooth_image(301, 211, seed)
    qb = oracle.quantize(img, 24)
    th = _crop_template(qb, 24, 120, 80, 40, 30)
    lmap = oracle.hist_match_map_direct(qb, 24, th, 40, 30, 1.0)
    return [lmap, rng.random((211, 301)), np.round(rng.random((211, 301)) * 3) / 3, np.full((211, 301), 0.37)]


@pytest.mark.parametrize("seed", [4, 5])
def test_fuse_maps_bit_exact(P, seed):
    maps = _consumer_maps(seed)
    dm = [torch.from_numpy(m).cuda() for m in maps]
    for wts in (None, [0.1, 0.2, 0.3, 0.4], [0.0, 1.0, 0.0, 3.0]):
        assert np.array_equal(P.fuse_maps(dm, wts).cpu().numpy(), oracle.fuse_maps(maps, wts))
    many = [dm[i % 4] for i in range(11)]  # more maps than one fuse launch takes
    assert np.array_equal(P.fuse_maps(many).cpu().numpy(), oracle.fuse_maps([maps[i % 4] for i in range(11)]))
    with pytest.raises(P.ContractError):
        P.fuse_maps([dm[0], dm[1]], [1.0])
    with pytest.raises(P.ContractError):
        P.fuse_maps([dm[0]], [-1.0])


@pytest.mark.parametrize("seed", [4, 5])
def test_find_peaks_and_score_bit_exact(P, seed):
    for m in _consumer_maps(seed) + [np.random.default_rng(seed).random((600, 700))]:
        xs, ys, hs = (t.cpu().numpy() for t in P.find_peaks(torch.from_numpy(m).cuda()))
        wx, wy, wh = oracle.find_peaks(m)
        assert np.array_equal(xs, wx) and np.array_equal(ys, wy) and np.array_equal(hs, wh)
        h, w = m.shape
        for g in [(0, 0, 5, 5), (w // 3, h // 4, w // 3, h // 2), (w - 6, h - 5, 6, 5)]:
            assert P.score_map(torch.from_numpy(m).cuda(), *g) == oracle.score_map(m, *g)


def test_score_map_ties_and_empty_rects(P):
    """Equal-height peaks rank in row-major order (stable_sort, likelihood.cpp:319-321);
    a rect without a peak scores peak count + 1 (:337-338)."""
    m = np.zeros((90, 120))
    bumps = [(20, 10), (90, 10), (20, 60), (90, 60), (55, 35)]
    for i, (x, y) in enumerate(bumps):
        m[y - 2:y + 3, x - 2:x + 3] = 0.5 if i < 4 else 0.25
    md = torch.from_numpy(m).cuda()
    for g in [(85, 5, 10, 10), (15, 55, 10, 10), (50, 30, 10, 10), (0, 80, 120, 10), (100, 40, 20, 5),
              (0, 0, 120, 90)]:
        assert P.score_map(md, *g) == oracle.score_map(m, *g), g


def test_camshift_bit_exact(P):
    maps = _consumer_maps(6)
    rng = np.random.default_rng(6)
    starts = np.c_[rng.uniform(0, 300, 64), rng.uniform(0, 210, 64)]
    for m in maps:
        c, it, zm = P.camshift_batch(torch.from_numpy(m).cuda(), starts, 33, 21)
        for q, (cx, cy) in enumerate(starts):
            wcx, wcy, wit, wzm = oracle.camshift(m, cx, cy, 33, 21)
            assert (c[q, 0], c[q, 1], it[q], zm[q]) == (wcx, wcy, wit, wzm)
    imp = np.zeros((12, 12))
    imp[7, 5] = 1.0
    assert P.camshift_refine(torch.from_numpy(imp).cuda(), 3.0, 3.0, 9, 9)[:2] == (5.0, 7.0)  # test_tracker.cpp:151-158
    with pytest.raises(P.ContractError):
        P.camshift_refine(torch.from_numpy(imp).cuda(), 12.0, 3.0, 9, 9)


# ------------------------------------------------------------------ SWIH (§8(f) #1)

SWIH_KERNELS = [(1, 1), (2, 2), (3, 3), (4, 4), (5, 3), (1, 7), (8, 1), (9, 9), (6, 10)]  # test_swih.cpp:100-101


def test_weighted_tensor_bit_exact(P):
    bm = oracle.random_binmap(131, 77, 9, 5)
    wts = np.random.default_rng(5).integers(0, 1 << 40, bm.size, dtype=np.uint64).reshape(bm.shape)
    t = P.swih.build_weighted_tensor(bm, wts, 9)
    assert np.array_equal(t.padded_u64(), oracle.weighted_ih(bm, wts, 9))
    with pytest.raises(P.ContractError):
        P.swih.build_weighted_tensor(bm, wts, 8)  # bin index out of range (integral.cpp:337-343)


@pytest.mark.parametrize("kw,kh", SWIH_KERNELS)
def test_swlh_query_bit_exact(P, kw, kh):
    """test_swih.cpp:98-114 / acceptance criterion 3: the device quadrant query equals the
    brute force (device and oracle), 16.16 fixed point, bit for bit."""
    w, h, nb = 40, 36, 8
    bm = oracle.random_binmap(w, h, nb, 606 + kw * 10 + kh)
    s = P.swih.build_quadrant_set(bm, nb, kw, kh)
    rng = np.random.default_rng(kw * 100 + kh)
    cs = [(kw // 2 + int(rng.integers(0, w - kw + 1)), kh // 2 + int(rng.integers(0, h - kh + 1))) for _ in range(25)]
    fast = P.swih.swlh_query_fixed(s, cs)
    slow = P.swih.brute_force_swlh_fixed(bm, nb, cs, kw, kh)
    want = np.stack([oracle.swlh_fixed(bm, nb, cx, cy, kw, kh) for cx, cy in cs])
    assert np.array_equal(fast, want) and np.array_equal(slow, want)
    q = P.swih.swlh_query(s, cs)
    ref = np.stack([oracle.swlh(bm, nb, cx, cy, kw, kh) for cx, cy in cs])
    assert np.all(np.abs(q - ref) <= 2.3e-16 * np.abs(ref))  # FP64 vs x87 long double: <= 1 ulp
    with pytest.raises(P.ContractError):
        P.swih.swlh_query_fixed(s, [(0, 0)] if kw > 1 or kh > 1 else [(w, 0)])  # window outside the image


def test_swlh_quadrant_tensors_match_reference_fields(P):
    """build_quadrant_set's four tensors == build_weighted_tensor of quadrant_weight_fields."""
    w, h, nb, kw, kh = 33, 21, 5, 7, 4
    bm = oracle.random_binmap(w, h, nb, 17)
    s = P.swih.build_quadrant_set(bm, nb, kw, kh)
    sx, sy = int(kw >= 3), int(kh >= 3)
    x, y = np.meshgrid(np.arange(w), np.arange(h))
    fields = [1 + sx * x + sy * y, 1 + sx * (w - 1 - x) + sy * y, 1 + sx * x + sy * (h - 1 - y),
              1 + sx * (w - 1 - x) + sy * (h - 1 - y)]  # NW, NE, SW, SE (swih.cpp:45-53)
    for t, f in zip(s.tensors, fields):
        assert np.array_equal(t.padded_u64(), oracle.weighted_ih(bm, (f.astype(np.uint64) << np.uint64(16)), nb))


@pytest.mark.parametrize("kw,kh,w,h", [(9, 7, 64, 48), (4, 4, 37, 29), (1, 1, 12, 9), (20, 30, 15, 12)])
def test_swlh_distance_map(P, kw, kh, w, h):
    """The tracker's swlh-distance channel (track_loop.cpp:264-283) vs the C restatement."""
    nb = 8
    img = oracle.smooth_image(w, h, kw + w)
    bm = oracle.quantize(img, nb)
    if w >= kw and h >= kh:
        model = oracle.swlh(bm, nb, w // 2, h // 2, kw, kh)
    else:
        model = np.full(nb, 1.0 / nb)
    want = oracle.swlh_map(bm, nb, model, kw, kh)
    quad = P.swih.swlh_distance_map(bm, nb, model, kw, kh, method="quadrant").cpu().numpy()
    assert close(quad, want)
    got = P.swih.swlh_distance_map(bm, nb, model, kw, kh).cpu().numpy()
    assert np.array_equal(got, quad)  # the direct sweep reproduces the quadrant path bit for bit
    if w >= kw and h >= kh:
        assert got[h // 2, w // 2] == 1.0


@pytest.mark.parametrize("w,h,nb,kw,kh", [(300, 170, 32, 31, 31), (260, 150, 70, 17, 40), (140, 300, 5, 128, 9),
                                           (129, 130, 16, 2, 255), (64, 40, 33, 1, 1), (200, 90, 8, 64, 64)])
def test_swlh_direct_map_matches_quadrant_path(P, w, h, nb, kw, kh):
    """The single-sweep swlh map (many bands, several bin groups, kernel extremes) equals
    the quadrant-tensor path exactly."""
    rng = np.random.default_rng(w * h + kw)
    bm = rng.integers(0, nb, (h, w)).astype(np.uint16)
    model = rng.random(nb)
    model /= model.sum()
    if h < kh:
        return
    quad = P.swih.swlh_distance_map(bm, nb, model, kw, kh, method="quadrant").cpu().numpy()
    got = P.swih.swlh_distance_map(bm, nb, model, kw, kh).cpu().numpy()
    assert np.array_equal(got, quad)


# ------------------------------------------------------------------ joint-IH median (§8(f) #4)

@pytest.mark.parametrize("w,h,bins,m,n,nf,nslide", [(23, 17, 8, 3, 5, 5, 0), (140, 131, 16, 7, 7, 3, 4),
                                                      (9, 9, 4, 1, 1, 1, 2), (260, 150, 32, 5, 3, 7, 1),
                                                      (300, 40, 5, 9, 9, 5, 3)])
def test_median_background_bit_exact(P, w, h, bins, m, n, nf, nslide):
    rng = np.random.default_rng(w * h + bins)
    frames = [rng.integers(0, bins, (h, w), dtype=np.uint8) for _ in range(nf + nslide)]
    bg = P.motion.MedianBackgroundIH(frames[:nf], bins, m, n)
    for f in frames[nf:]:
        bg.slide(f)
    assert np.array_equal(bg.background().cpu().numpy(), oracle.median_bg_ih(frames, nf, bins, m, n))
    assert np.array_equal(P.motion.median_background_sort(frames[:nf]).cpu().numpy(), oracle.median_bg_sort(frames[:nf]))
    with pytest.raises(P.ContractError):
        P.motion.MedianBackgroundIH(frames[:nf], max(1, int(frames[0].max())), m, n)  # value exceeds bin count
    with pytest.raises(P.ContractError):
        P.motion.MedianBackgroundIH(frames[:2], bins, m, n)  # even window


def test_channel_graph_replays_exactly(P):
    """The CUDA-graph replay of a frame's five channels equals the eager calls."""
    from paper_1711_01656_b200.channels import ChannelGraph

    w, h, nbins, kw, kh = 300, 200, 32, 32, 24
    frames = [oracle.noise_color(w, h, 40 + i) for i in range(3)]
    srcs = P.channel_sources(*frames[0], nbins)
    tdev = {}
    for c, s in srcs.items():
        qb = s if c == "orientation" else P.quantize(s, nbins)
        crop = qb[90:90 + kh, 120:120 + kw].to(torch.int64).reshape(-1) & 0xFFFF
        tdev[c] = (torch.bincount(crop, minlength=nbins).to(torch.float64) / crop.numel()).contiguous()
    g = ChannelGraph(w, h, nbins, tdev, kw, kh, device="cuda")
    for r, gg, b in frames:
        got = {c: m.clone() for c, m in g.run(torch.from_numpy(r).cuda(), torch.from_numpy(gg).cuda(),
                                             torch.from_numpy(b).cuda()).items()}
        want = P.likelihood_channels(r, gg, b, nbins, None, kw, kh, 1.0, tmpl_dev=tdev)
        for c in P.CHANNELS:
            assert torch.equal(got[c], want[c]), c


@pytest.mark.parametrize("bins,p,metric,store", [(32, 1.0, 0, True), (48, 2.0, 0, False), (32, 1.0, 2, True),
                                                  (200, 1.0, 0, True)])
def test_build_match_map_multi_matches_single(P, bins, p, metric, store):
    """spct_cu_ih_build_match_map_multi (batched carries / preps, per-source sweeps) equals
    one spct_cu_ih_build_match_map per source: 8-bit frames beside a uint16 BinMap, a crop
    template and a random one; above 128 bins the batch runs source by source."""
    w, h, kw, kh = 300, 190, 64, 48
    imgs = [oracle.smooth_image(w, h, 30 + i) for i in range(3)]
    bm = oracle.random_binmap(w, h, bins, 77)
    srcs = [torch.from_numpy(x).cuda() for x in imgs] + [torch.from_numpy(bm.astype(np.int16)).cuda()]
    rng = np.random.default_rng(bins)
    tm = [_crop_template(oracle.quantize(imgs[0], bins), bins, 40, 30, kw, kh), rng.random(bins) + 0.05,
          _crop_template(oracle.quantize(imgs[2], bins), bins, 100, 60, kw, kh), rng.random(bins) + 0.05]
    tm = [t / t.sum() for t in tm]
    tds = [torch.from_numpy(t).cuda() for t in tm]
    outs = [P.IntegralHistogramTensor(w, h, bins) for _ in srcs]
    if not store:
        for t in outs:
            t.desc.data = None
    maps = [torch.empty((h, w), dtype=torch.float64, device="cuda") for _ in srcs]
    P.api.build_and_match_map_multi(srcs, bins, tds, kw, kh, p, metric, outs=outs, lmaps=maps)
    for i, s in enumerate(srcs):
        t1 = P.IntegralHistogramTensor(w, h, bins)
        if not store:
            t1.desc.data = None
        _, m1 = P.build_and_match_map(s, bins, None, kw, kh, p, metric, out=t1, tmpl_dev=tds[i])
        assert torch.equal(maps[i], m1), i
        if store:
            assert np.array_equal(outs[i].padded_u64(), t1.padded_u64()), i
    assert close(maps[3].cpu().numpy(), oracle.hist_match_map_direct(bm, bins, tm[3], kw, kh, p, metric))


@pytest.mark.parametrize("w,h,bins", [(520, 300, 64), (700, 130, 16), (129, 517, 40)])
def test_joint_tensor_after_slides_bit_exact(P, w, h, bins, band_rows):
    """The one-pass slide (J += IH(new) - IH(old), spct_cu_ih_slide) keeps the joint tensor
    equal to the sum of the window frames' integral histograms, cell by cell, across
    strips and (forced short) bands."""
    band_rows(37)
    rng = np.random.default_rng(w + bins)
    frames = [rng.integers(0, bins, (h, w), dtype=np.uint8) for _ in range(7)]
    bg = P.motion.MedianBackgroundIH(frames[:3], bins, 3, 3)
    for i in range(3, 7):
        bg.slide(frames[i])
        want = sum(oracle.build_ih(f.astype(np.uint16), bins) for f in frames[i - 2:i + 1])
        assert np.array_equal(bg.joint.padded_u64(), want), i


@pytest.mark.parametrize("w,bins,pitch", [(1001, 32, 1008), (1003, 16, 1004), (998, 32, 1000), (1022, 20, 1024)])
def test_fused_wide_staging_pitched_edges(P, w, bins, pitch):
    """4- and 8-strip CTAs stage four 8-bit columns per thread from 4-byte aligned rows (SK 3):
    a pitched frame whose last word straddles the image edge (garbage in the pitch padding)
    keeps the reference bins, tensor and map."""
    import ctypes as C

    import torch

    from paper_1711_01656_b200 import _capi as A
    from paper_1711_01656_b200 import api

    h, kw, kh = 150, 64, 40
    img = oracle.smooth_image(w, h, 77 + w)
    buf = np.full((h, pitch), 255, np.uint8)
    buf[:, :w] = img
    dev = torch.from_numpy(buf).cuda()
    qb = oracle.quantize(img, bins)
    th = _crop_template(qb, bins, (w - kw) // 2, (h - kh) // 3, kw, kh)
    t = P.IntegralHistogramTensor(w, h, bins)
    lmap = torch.empty((h, w), dtype=torch.float64, device="cuda")
    tdev = api._tmpl(th, bins, w, h, kw, kh, 1.0).cuda()
    src = api._source(A.SRC_GRAY_U8, [dev], w, h, bins, pitch=pitch)
    ws = C.c_size_t()
    api.check(A.lib().spct_cu_ih_build_workspace(C.byref(src), t.bin0, t.bins, C.byref(ws)))
    wbuf = torch.empty(max(ws.value, 256), dtype=torch.uint8, device="cuda")
    api.check(A.lib().spct_cu_ih_build_match_map(C.byref(src), C.byref(t.desc), api._ptr(tdev), kw, kh, 1.0,
                                                 A.METRIC_MINKOWSKI, api._ptr(lmap), api._ptr(wbuf), wbuf.numel(),
                                                 api._stream(None)))
    torch.cuda.synchronize()
    assert close(lmap.cpu().numpy(), oracle.hist_match_map_direct(qb, bins, th, kw, kh, 1.0))
    assert np.array_equal(t.padded_u64(), oracle.build_ih(qb, bins))
