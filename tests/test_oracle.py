"""Pin the CPU oracle before trusting it (CPU-only, no GPU).

1. The C restatement (oracle/spct_oracle.c) reproduces every known answer the
   reference's own tests assert (tests/golden/known_answers.json).
2. It reproduces the committed outputs of the unmodified reference
   (tests/golden/ref_vectors.npz) bit for bit.
3. When oracle/_ref is built (always in the build container), it agrees with the
   live reference on fresh seeded inputs, including every schedule kind.
"""
import numpy as np
import pytest

import oracle


def test_known_ih_2x2(golden):
    k = golden[0]["ih_2x2"]
    t = oracle.build_ih(np.array(k["binmap"], np.uint16), k["bins"])
    for kk, y, x, v in k["expect_at"]:
        assert t[kk, y, x] == v
    assert not t[:, 0, :].any() and not t[:, :, 0].any()


def test_known_ih_1x1(golden):
    k = golden[0]["ih_1x1"]
    t = oracle.build_ih(np.array(k["binmap"], np.uint16), k["bins"])
    nz = np.argwhere(t)
    assert nz.tolist() == [e[:3] for e in k["nonzero"]]
    assert t[5, 1, 1] == 1


def test_known_quantize_and_gray(golden):
    kn = golden[0]
    q = kn["quantize_32"]
    img = np.array([q["pixels"]], np.uint8)
    assert oracle.quantize(img, q["bins"], q["lo"], q["hi"]).tolist() == [q["expect"]]
    c = kn["quantize_clamp"]
    out = oracle.quantize(img, c["bins"], c["lo"], c["hi"])
    assert out[0, 0] == c["expect_first"] and out[0, -1] == c["expect_last"]
    for bins, lo, hi in kn["quantize_contract"]["bad"]:
        with pytest.raises(oracle.ContractError):
            oracle.quantize(img, bins, lo, hi)
    g = kn["grayscale"]
    rgb = np.array(g["rgb"], np.uint8)
    gray = oracle.to_grayscale(rgb[None, :, 0], rgb[None, :, 1], rgb[None, :, 2])
    assert gray.tolist() == [g["expect"]]


def test_known_hist_fixture(golden):
    k = golden[0]["hist_fixture_0p7"]
    img = np.array(k["image"], np.uint8)
    t = oracle.build_ih(oracle.quantize(img, k["bins"]), k["bins"])
    m = oracle.hist_distance_map(t, k["template"], k["kw"], k["kh"], k["p"])
    x, y = k["at"]
    assert abs(m[y, x] - k["expect"]) <= k["eps"] * max(1.0, k["expect"])


def test_known_stats_and_memory(golden):
    kn = golden[0]
    for c in kn["schedule_stats"]["cases"]:
        s = oracle.schedule_stats(*c["args"])
        assert s.wavefront_iterations == c["iters"] and s.tile_count == c["tiles"]
        if "eff_lo" in c:
            assert c["eff_lo"] < s.scan_efficiency < c["eff_hi"]
    for bad in kn["schedule_stats"]["bad"]:
        with pytest.raises(oracle.ContractError):
            oracle.schedule_stats(*bad)
    for c in kn["estimate_memory"]["cases"]:
        pad, raw, deg = oracle.estimate_memory(*c["args"])
        if "raw" in c:
            assert raw == c["raw"]
        if "padded" in c:
            assert pad == c["padded"]
        assert deg == c["degenerate"] if "degenerate" in c else True
    for bad in kn["estimate_memory"]["bad"]:
        with pytest.raises(oracle.ContractError):
            oracle.estimate_memory(*bad)


def test_known_budget_reject(golden):
    k = golden[0]["budget_reject"]
    bm = oracle.random_binmap(k["w"], k["h"], k["bins"], 3)
    with pytest.raises(oracle.ContractError):
        oracle.validate_build(bm, k["bins"], budget=k["budget"])
    oracle.validate_build(bm, k["bins"])
    bad = bm.copy()
    bad[0, 7] = k["bins"]
    with pytest.raises(oracle.ContractError):
        oracle.validate_build(bad, k["bins"])


def test_oracle_matches_reference_vectors(golden):
    vec = golden[1]
    for key in [k for k in vec if k.endswith("_tensor")]:
        bm = vec[key.replace("_tensor", "_bins")]
        t = oracle.build_ih(bm, 16)
        assert np.array_equal(t, vec[key]), key
        t32 = oracle.build_ih(bm, 16, dtype=np.uint32)
        assert np.array_equal(t32.astype(np.uint64), vec[key]), key
    t = oracle.build_ih(vec["region_bins"], 32)
    for r, want in zip(vec["region_rects"], vec["region_hists"]):
        assert np.array_equal(oracle.region_histogram(t, *map(int, r)), want)
    qb = oracle.quantize(vec["lmap_noise_img"], 8)
    t = oracle.build_ih(qb, 8)
    tmpl = np.full(8, 1.0 / 8)
    # same operation order as likelihood.cpp:211-221 -> bit-identical maps
    assert np.array_equal(oracle.hist_distance_map(t, tmpl, 7, 5, 2.0), vec["lmap_noise_p2"])
    assert np.array_equal(oracle.hist_distance_map(t, tmpl, 7, 5, 1.0), vec["lmap_noise_p1"])
    qb = oracle.quantize(vec["lmap_smooth_img"], 16)
    t = oracle.build_ih(qb, 16)
    th = vec["lmap_smooth_tmpl"]
    assert np.array_equal(oracle.hist_distance_map(t, th, 20, 16, 1.0), vec["lmap_smooth_p1"])
    assert np.array_equal(oracle.hist_distance_map(t, th, 20, 16, 3.0), vec["lmap_smooth_p3"])
    # the tensor-free sliding-window map is the same arithmetic per window
    assert np.array_equal(oracle.hist_match_map_direct(qb, 16, th, 20, 16, 1.0), vec["lmap_smooth_p1"])
    gray = oracle.to_grayscale(vec["color_r"], vec["color_g"], vec["color_b"])
    assert np.array_equal(gray, vec["color_gray"])
    assert np.array_equal(oracle.quantize(gray, 32), vec["color_q32"])
    assert np.array_equal(oracle.quantize(gray, 7, 30.0, 200.0), vec["color_q7_lohi"])


def test_grayscale_quantize_integer_shortcuts():
    """(r+g+b+1)//3 and (v*b)>>8 are exact restatements."""
    s = np.arange(0, 766)
    r = np.minimum(s, 255)
    g = np.minimum(np.maximum(s - 255, 0), 255)
    b = np.maximum(s - 510, 0)
    gray = oracle.to_grayscale(r[None].astype(np.uint8), g[None].astype(np.uint8), b[None].astype(np.uint8))
    assert np.array_equal(gray[0], ((s + 1) // 3).astype(np.uint8))
    v = np.arange(256, dtype=np.uint8)[None]
    for bins in [1, 2, 3, 7, 16, 32, 100, 128, 255, 256, 257, 1000, 1024, 65536]:
        assert np.array_equal(oracle.quantize(v, bins)[0], ((v[0].astype(np.int64) * bins) >> 8).astype(np.uint16))


def test_slab_partial_sums_recompose():
    """Bin-slab sharding: per-slab partial p-sums add up to the full map."""
    img = oracle.smooth_image(40, 30, 5)
    qb = oracle.quantize(img, 12)
    crop = qb[5:14, 8:19]
    th = np.bincount(crop.reshape(-1), minlength=12).astype(np.float64) / crop.size
    for p in (1.0, 2.0):
        full = oracle.hist_match_map_direct(qb, 12, th, 11, 9, p)
        parts = [oracle.hist_partial(qb, 12, th, 11, 9, p, k0, k0 + 4) for k0 in (0, 4, 8)]
        got = oracle.hist_finalize(parts[0] + parts[1] + parts[2], 40, 30, 11, 9, p)
        assert np.allclose(got, full, rtol=1e-12, atol=1e-12)


ref = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


@ref
@pytest.mark.parametrize("w,h,bins", [(1, 1, 4), (5, 3, 16), (33, 31, 16), (70, 129, 16), (97, 61, 37)])
def test_oracle_vs_live_reference_all_schedules(w, h, bins):
    bm = oracle.random_binmap(w, h, bins, 4242 + w)
    mine = oracle.build_ih(bm, bins)
    for kind in (oracle.SEQUENTIAL, oracle.STS, oracle.CW_TIS, oracle.WF_TIS):
        for tile, threads in ((32, 1), (64, 4)):
            assert np.array_equal(oracle.RefTensor(bm, bins, kind, tile, threads).array(), mine)


@ref
def test_oracle_vs_live_reference_maps():
    img = oracle.noise_image(57, 43, 3)
    qb = oracle.ref_quantize(img, 9)
    t = oracle.RefTensor(qb, 9)
    crop = qb[10:21, 5:18]
    th = np.bincount(crop.reshape(-1), minlength=9).astype(np.float64) / crop.size
    mine_t = oracle.build_ih(qb, 9)
    for p in (1.0, 1.5, 2.0):
        want = t.hist_distance_map(th, 13, 11, p)
        assert np.array_equal(oracle.hist_distance_map(mine_t, th, 13, 11, p), want)
        assert np.array_equal(oracle.hist_match_map_direct(qb, 9, th, 13, 11, p), want)
    with pytest.raises(oracle.ContractError):
        t.hist_distance_map(th * 2, 13, 11, 1.0)
    with pytest.raises(oracle.ContractError):
        t.hist_distance_map(th, 13, 11, 0.5)


@ref
@pytest.mark.parametrize("w,h,sigma,bins", [(1, 1, 1.0, 8), (5, 3, 0.0, 9), (64, 48, 1.0, 32), (131, 97, 1.5, 16),
                                            (200, 150, 0.7, 36)])
def test_orientation_bins_vs_live_reference(w, h, sigma, bins):
    """Orientation channel of the tracking batch: the C restatement of gradient_maps
    (features.cpp:78-93) + orientation_bin (phog.cpp:15-20) equals the reference."""
    for img in (oracle.smooth_image(w, h, w + h), oracle.noise_image(w, h, 7 * w + h)):
        assert np.array_equal(oracle.orientation_bins(img, bins, sigma), oracle.ref_orientation_bins(img, bins, sigma))
    flat = np.full((h, w), 77, np.uint8)  # flat: fold_orientation gives 0 degrees -> the middle bin
    assert np.all(oracle.orientation_bins(flat, bins, sigma) == min(bins - 1, (90 * bins) // 180))
    with pytest.raises(oracle.ContractError):
        oracle.ref_orientation_bins(flat, bins, -1.0)


# ------------------------------------------------------------------ map consumers (§8(f) #2)

def _bump_map(w, h, bumps):
    """test_likelihood.cpp:325-336 bump_map."""
    m = np.zeros((h, w))
    for (rx, ry, rw, rh), v in bumps:
        for y in range(ry, ry + rh):
            for x in range(rx, rx + rw):
                m[y, x] = max(m[y, x], v * (1.0 - 0.15 * (abs(x - (rx + rw // 2)) + abs(y - (ry + rh // 2)))))
    return m


def test_consumers_known_answers():
    """test_likelihood.cpp:296-362 and test_tracker.cpp:150-176 on the C restatement."""
    a, b = np.full((3, 4), 0.2), np.full((3, 4), 0.8)
    assert np.array_equal(oracle.fuse_maps([a]), a)
    assert np.allclose(oracle.fuse_maps([a, a], [0.3, 0.7]), 0.2)
    assert np.allclose(oracle.fuse_maps([a, b]), 0.5)
    for bad in ([a, np.full((3, 5), 0.1)], []):
        with pytest.raises(oracle.ContractError):
            oracle.fuse_maps(bad)
    with pytest.raises(oracle.ContractError):
        oracle.fuse_maps([a, b], [1.0])
    m = _bump_map(30, 24, [((10, 8, 5, 5), 1.0)])
    xs, ys, hs = oracle.find_peaks(m)
    assert len(xs) and np.all(np.diff(hs) <= 0)
    assert oracle.score_map(m, 9, 7, 8, 8) == 1
    two = _bump_map(40, 30, [((5, 5, 5, 5), 1.0), ((28, 20, 5, 5), 0.6)])
    assert oracle.score_map(two, 26, 18, 9, 9) == 2
    assert oracle.score_map(two, 20, 2, 4, 4) == len(oracle.find_peaks(two)[0]) + 1
    assert oracle.score_map(two * 0.25, 26, 18, 9, 9) == 2
    with pytest.raises(oracle.ContractError):
        oracle.score_map(two, 38, 28, 5, 5)
    imp = np.zeros((12, 12))
    imp[7, 5] = 1.0
    cx, cy, it, zm = oracle.camshift(imp, 3.0, 3.0, 9, 9)
    assert (cx, cy, zm) == (5.0, 7.0, False) and it >= 1
    assert oracle.camshift(np.zeros((10, 10)), 4.0, 4.0, 5, 5)[3]
    assert oracle.camshift(np.full((20, 20), 0.25), 10.0, 9.0, 5, 5)[:2] == (10.0, 9.0)


@ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_consumers_vs_live_reference(seed):
    rng = np.random.default_rng(seed)
    maps = [rng.random((37, 53)), np.round(rng.random((37, 53)) * 3) / 3, _bump_map(53, 37, [((4, 4, 9, 9), 0.9)])]
    for wts in (None, [0.2, 0.5, 0.3], [0.0, 2.0, 1.0]):
        assert np.array_equal(oracle.fuse_maps(maps, wts), oracle.ref_fuse_maps(maps, wts))
    for m in maps + [np.full((9, 11), 0.4)]:
        mine, ref_ = oracle.find_peaks(m), oracle.ref_find_peaks(m)
        assert all(np.array_equal(p, q) for p, q in zip(mine, ref_))
        h, w = m.shape
        for g in [(0, 0, 5, 5), (w // 3, h // 4, w // 3, h // 2), (w - 6, h - 5, 6, 5)]:
            assert oracle.score_map(m, *g) == oracle.ref_score_map(m, *g)


# ------------------------------------------------------------------ SWIH (§8(f) #1)

SWIH_KERNELS = [(1, 1), (2, 2), (3, 3), (4, 4), (5, 3), (1, 7), (8, 1), (9, 9), (6, 10)]  # test_swih.cpp:100-101


@ref
def test_weighted_ih_vs_live_reference():
    bm = oracle.random_binmap(23, 17, 6, 11)
    wts = np.random.default_rng(11).integers(0, 1 << 30, bm.size, dtype=np.uint64).reshape(bm.shape)
    assert np.array_equal(oracle.weighted_ih(bm, wts, 6), oracle.ref_weighted_ih(bm, wts, 6))


@ref
@pytest.mark.parametrize("kw,kh", SWIH_KERNELS)
def test_swlh_brute_force_vs_live_reference(kw, kh):
    """The C brute force (swih.cpp:166-178) == the reference's exact quadrant query
    (test_swih.cpp:98-114, acceptance criterion 3), fixed and normalised."""
    w, h, nb = 40, 36, 8
    bm = oracle.random_binmap(w, h, nb, 606 + kw * 10 + kh)
    rng = np.random.default_rng(kw * 100 + kh)
    cs = [(kw // 2 + int(rng.integers(0, w - kw + 1)), kh // 2 + int(rng.integers(0, h - kh + 1))) for _ in range(25)]
    fixed = oracle.ref_swlh_query_fixed(bm, nb, cs, kw, kh)
    norm = oracle.ref_swlh_query(bm, nb, cs, kw, kh)
    for i, (cx, cy) in enumerate(cs):
        assert np.array_equal(oracle.swlh_fixed(bm, nb, cx, cy, kw, kh), fixed[i])
        assert np.array_equal(oracle.swlh(bm, nb, cx, cy, kw, kh), norm[i])


def test_swlh_degenerate_known_answers():
    """test_swih.cpp:116-135."""
    bm = np.full((12, 12), 2, np.uint16)
    q = oracle.swlh(bm, 4, 6, 6, 5, 5)
    assert q[2] == 1.0 and q[0] == 0.0
    bm = oracle.random_binmap(9, 9, 5, 81)
    for y in range(9):
        for x in range(9):
            q = oracle.swlh(bm, 5, x, y, 1, 1)
            assert q[bm[y, x]] == 1.0 and q.sum() == 1.0


# ------------------------------------------------------------------ joint-IH median (§8(f) #4)

@ref
@pytest.mark.parametrize("w,h,bins,m,n,nf,nslide", [(23, 17, 8, 3, 5, 5, 0), (40, 31, 16, 7, 7, 3, 4),
                                                      (9, 9, 4, 1, 1, 1, 2), (31, 20, 32, 5, 3, 7, 1)])
def test_median_bg_vs_live_reference(w, h, bins, m, n, nf, nslide):
    rng = np.random.default_rng(w * h + bins)
    frames = [rng.integers(0, bins, (h, w), dtype=np.uint8) for _ in range(nf + nslide)]
    assert np.array_equal(oracle.median_bg_ih(frames, nf, bins, m, n), oracle.median_bg_ih(frames, nf, bins, m, n, True))
    assert np.array_equal(oracle.median_bg_sort(frames[:nf]), oracle.median_bg_sort(frames[:nf], True))
    with pytest.raises(oracle.ContractError):
        oracle.median_bg_ih(frames, nf, bins - 1 if bins > 1 else 0, m, n, True)  # value exceeds bin count


def test_extension_metrics_pinned_to_published_implementations():
    """Intersection / Bhattacharyya / chi-square (absent from the reference):
    the oracle's definitions against fixtures computed with scipy.spatial.distance
    (braycurtis, sqeuclidean) and sklearn.metrics.pairwise.additive_chi2_kernel
    (tests/golden/make_metric_golden.py)."""
    import os

    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "metric_vectors.npz"))
    for name in ("crop", "random", "sparse"):
        w, h, bins, kw, kh = (int(v) for v in d[f"{name}_dims"])
        bm, t = d[f"{name}_binmap"], d[f"{name}_template"]
        for key, metric in (("intersection", oracle.INTERSECTION), ("bhattacharyya", oracle.BHATTACHARYYA),
                            ("chisq", oracle.CHISQ)):
            got = oracle.hist_match_map_direct(bm, bins, t, kw, kh, 1.0, metric)
            assert np.abs(got - d[f"{name}_{key}"]).max() <= 1e-12, (name, key)
            ih = oracle.build_ih(bm, bins)
            assert np.array_equal(oracle.hist_match_map(ih, t, kw, kh, 1.0, metric), got), (name, key)
