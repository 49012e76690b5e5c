"""Full-size BASELINE configs through size-independent properties (GPU).

The oracle restatement is exact but too slow for the full sizes, so at C1-C5 scale the
device results are checked against properties that hold at any size and against direct
recomputation of sampled pieces:
  * integral histogram: the bin planes of a cell sum to y * x (every pixel has one bin);
    the last row of plane k is the running column count of bin k (so its last cell is the
    bin's pixel count); random rectangles equal direct counts of the quantised frame;
  * likelihood map: the fused single pass equals the map computed from the stored tensor
    (bit-exact for p = 1 with an integral template); sampled windows equal a direct FP64
    recomputation; the template's own crop scores exactly 1.0;
  * bin-slab sharding (C4): the partial maps of the slabs, summed and finalised, equal the
    single-pass map of the whole histogram (within 1e-12: the partials round separately);
  * tracking batch (C5): every channel map equals its tensor-path map; the orientation
    BinMap equals the oracle restatement at 2048^2.
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1711_01656_b200 as P

    return P


def frame(w, h, seed):
    return np.random.default_rng(seed).integers(0, 256, size=(h, w), dtype=np.uint8)


def qbins(img, nbins):
    return (img.astype(np.int64) * nbins) >> 8  # quantize(img, nbins), default range


def crop_template(qb, nbins, x0, y0, kw, kh):
    c = qb[y0:y0 + kh, x0:x0 + kw]
    return np.bincount(c.reshape(-1), minlength=nbins).astype(np.float64) / c.size


def check_tensor(P, t, qb_dev, nbins, rng, nrect=64):
    """Plane sums, last row = running column counts, random rectangles."""
    h, w = qb_dev.shape
    planes = t.planes()  # (bins, h, row_pitch) int32 view, unpadded: cell (y, x) = H(y + 1, x + 1)
    for y in (0, h // 3, h - 1):
        s = planes[:, y, :w].to(torch.int64).sum(0)
        want = (y + 1) * torch.arange(1, w + 1, device=s.device, dtype=torch.int64)
        assert torch.equal(s, want), y
    flat = qb_dev.to(torch.int64) * w + torch.arange(w, device=qb_dev.device).expand(h, w)
    col = torch.bincount(flat.reshape(-1), minlength=nbins * w).view(nbins, w)
    assert torch.equal(planes[:, h - 1, :w].to(torch.int64), col.cumsum(1))
    for _ in range(nrect):
        x0, y0 = int(rng.integers(0, w)), int(rng.integers(0, h))
        rw, rh = int(rng.integers(0, w - x0 + 1)), int(rng.integers(0, h - y0 + 1))
        got = np.asarray(P.region_histogram(t, x0, y0, rw, rh), np.int64)
        want = torch.bincount(qb_dev[y0:y0 + rh, x0:x0 + rw].reshape(-1).to(torch.int64), minlength=nbins)
        assert np.array_equal(got, want.cpu().numpy()), (x0, y0, rw, rh)


def direct_windows(qb, nbins, tmpl, kw, kh, pts):
    """L at window top-left (u, v), FP64 in the reference's order (likelihood.cpp:208-221)."""
    out = []
    for u, v in pts:
        c = np.bincount(qb[v:v + kh, u:u + kw].reshape(-1), minlength=nbins).astype(np.float64)
        tot = c.sum()
        d = 0.0
        for k in range(nbins):
            d += abs(c[k] / tot - tmpl[k])
        out.append(min(max(1.0 - d / 2.0, 0.0), 1.0))
    return np.array(out)


def map_at(lmap, pts, kw, kh):
    return np.array([lmap[v + (kh - 1) // 2, u + (kw - 1) // 2] for u, v in pts])


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_full_size_ih_and_map(P, cfg):
    rng = np.random.default_rng(7)
    if cfg == "C1":  # 512^2 8-bit gray, 16 bins
        w = h = 512
        nbins, kw, kh = 16, 32, 32
        img = frame(w, h, 1)
        src = img
    elif cfg == "C2":  # 1024^2 RGB -> gray, 32 bins, 64 x 64 template at (480, 480)
        w = h = 1024
        nbins, kw, kh = 32, 64, 64
        rgb = [frame(w, h, s) for s in (1, 2, 3)]
        img = ((rgb[0].astype(np.int64) + rgb[1] + rgb[2] + 1) // 3).astype(np.uint8)  # to_grayscale
        src = tuple(torch.from_numpy(c).cuda() for c in rgb)
    else:  # 4096^2, 128 bins, 64 x 64
        w = h = 4096
        nbins, kw, kh = 128, 64, 64
        img = frame(w, h, 1)
        src = img
    qb = qbins(img, nbins)
    x0 = y0 = 480 if cfg == "C2" else (w - kw) // 2
    tmpl = crop_template(qb, nbins, x0, y0, kw, kh)
    t, lmap = P.build_and_match_map(src, nbins, tmpl, kw, kh, 1.0)
    qb_dev = torch.from_numpy(qb.astype(np.int16)).cuda()
    check_tensor(P, t, qb_dev, nbins, rng)
    lm = lmap.cpu().numpy()
    # the map from the stored tensor (the unfused matcher) is the same bits
    assert np.array_equal(P.hist_distance_map(t, tmpl, kw, kh, 1.0, exact=True).cpu().numpy(), lm)
    assert lm[y0 + (kh - 1) // 2, x0 + (kw - 1) // 2] == 1.0
    pts = [(int(rng.integers(0, w - kw + 1)), int(rng.integers(0, h - kh + 1))) for _ in range(48)]
    pts += [(0, 0), (w - kw, h - kh), (x0, y0)]
    assert np.array_equal(map_at(lm, pts, kw, kh), direct_windows(qb, nbins, tmpl, kw, kh, pts))


def test_full_size_c4_bin_slabs(P):
    """8192^2, 256 bins in eight 32-bin slabs (the 8-GPU partition) on one device."""
    w = h = 8192
    nbins, kw, kh, nslab = 256, 64, 64, 8
    img = frame(w, h, 4)
    qb = qbins(img, nbins)
    tmpl = crop_template(qb, nbins, (w - kw) // 2, (h - kh) // 2, kw, kh)
    full = P.IntegralHistogramTensor(w, h, nbins)
    full.desc.data = None  # map only: the 68.7 GB tensor is not stored
    _, lmap = P.build_and_match_map(img, nbins, tmpl, kw, kh, 1.0, out=full)
    nu, nv = w - kw + 1, h - kh + 1
    acc = torch.zeros((nv, nu), dtype=torch.float64, device="cuda")
    part = torch.empty_like(acc)
    qb_dev = torch.from_numpy(qb.astype(np.int16)).cuda()
    rng = np.random.default_rng(3)
    from paper_1711_01656_b200.sharding import slab_bounds

    for r in range(nslab):
        k0, k1 = slab_bounds(nbins, nslab, r)
        slab = P.IntegralHistogramTensor(w, h, nbins, k0, k1 - k0)
        P.build_and_match(img, nbins, tmpl, kw, kh, 1.0, bin0=k0, bins=k1 - k0, out=slab, partial=part)
        acc += part
        if r in (0, nslab - 1):  # slab tensor: its planes' last row are the slab bins' column counts
            planes = slab.planes()
            for kk in (0, k1 - k0 - 1):
                colk = (qb_dev == k0 + kk).to(torch.int64).sum(0)
                assert torch.equal(planes[kk, h - 1, :w].to(torch.int64), colk.cumsum(0))
            x, y = int(rng.integers(0, w - 100)), int(rng.integers(0, h - 100))
            got = np.asarray(P.region_histogram(slab, x, y, 100, 100), np.int64)
            want = torch.bincount(qb_dev[y:y + 100, x:x + 100].reshape(-1).to(torch.int64), minlength=nbins)
            assert np.array_equal(got, want[k0:k1].cpu().numpy())
    got = P.hist_finalize(acc, w, h, kw, kh, 1.0).cpu().numpy()
    want = lmap.cpu().numpy()
    assert np.all(np.abs(got - want) <= 1e-12)


def test_full_size_c5_channels(P):
    """One 2048^2 RGB frame, 32 bins: the five channel maps equal their tensor-path maps, and
    the orientation BinMap equals the oracle restatement."""
    w = h = 2048
    nbins, kw, kh = 32, 64, 64
    rgb = [frame(w, h, s) for s in (11, 12, 13)]
    dev = [torch.from_numpy(c).cuda() for c in rgb]
    srcs = P.channel_sources(*dev, nbins)
    gray = ((rgb[0].astype(np.int64) + rgb[1] + rgb[2] + 1) // 3).astype(np.uint8)
    assert np.array_equal(srcs["intensity"].cpu().numpy(), gray)
    ob = P.api.as_numpy_u16(srcs["orientation"])
    assert np.array_equal(ob, oracle.orientation_bins(gray, nbins, 1.0))
    qbs = {"intensity": qbins(gray, nbins), "orientation": ob.astype(np.int64), "red": qbins(rgb[0], nbins),
           "green": qbins(rgb[1], nbins), "blue": qbins(rgb[2], nbins)}
    tmpls = {c: crop_template(q, nbins, 992, 992, kw, kh) for c, q in qbs.items()}
    maps = P.likelihood_channels(*dev, nbins, tmpls, kw, kh)
    for c in P.CHANNELS:
        t = P.build_integral_histogram(torch.from_numpy(qbs[c].astype(np.int16)).cuda(), nbins)
        want = P.hist_distance_map(t, tmpls[c], kw, kh, 1.0, exact=True).cpu().numpy()
        assert np.array_equal(maps[c].cpu().numpy(), want), c
