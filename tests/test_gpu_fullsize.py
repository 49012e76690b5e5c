"""Cell-by-cell parity at the BASELINE headline sizes (GPU), against the CPU oracle.

test_gpu_properties.py checks the full sizes through size-independent properties; this
file compares EVERY cell with the oracle restatement (oracle/spct_oracle.c, pinned to the
compiled reference in test_oracle.py):

  * C3 (4096^2 x 128 bins): the fused build+match tensor, plane group by plane group,
    against or_ih_build_u32 (integral.cpp:348-361) — 0 mismatching cells; the finished
    likelihood map against or_hist_match_map_direct (likelihood.cpp:193-225 + spread_valid
    :44-58) computed in window-row bands on the host threads — bit-exact for the crop
    template (p = 1, kw*kh a power of two) and within 1e-5 relative for a general
    template at p = 2;
  * C4 (8192^2 x 256 bins, the sharded config on one GPU: two 128-bin groups whose partial
    sums are accumulated): every IH cell of every bin, and the full map.

Host work runs in ctypes calls that release the GIL, so the oracle bands and plane
groups run on all host threads.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 1e-5
THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1711_01656_b200 as P

    return P


def _frame(side, seed):
    return np.random.default_rng(seed).integers(0, 256, size=(side, side), dtype=np.uint8)


def _crop_template(qb, nbins, kw, kh):
    h, w = qb.shape
    y0, x0 = (h - kh) // 2, (w - kw) // 2
    c = qb[y0:y0 + kh, x0:x0 + kw]
    return np.bincount(c.reshape(-1), minlength=nbins).astype(np.float64) / c.size


def _ih_mismatches(t, qb, nbins, group=4):
    """Count device cells != oracle cells over every plane (groups of `group` planes)."""
    h, w = qb.shape
    planes = t.planes()

    def one(k0):
        k1 = min(nbins, k0 + group)
        want = oracle.build_ih(qb, nbins, k0, k1, dtype=np.uint32)
        got = planes[k0:k1, :, :w].cpu().numpy().view(np.uint32)
        bad = int(np.count_nonzero(got != want[:, 1:, 1:]))
        pad = int(np.count_nonzero(want[:, 0, :])) + int(np.count_nonzero(want[:, :, 0]))
        return bad + pad

    with ThreadPoolExecutor(min(THREADS, 8)) as ex:
        return sum(ex.map(one, range(0, nbins, group)))


def _valid_grid(qb, nbins, tmpl, kw, kh, p, metric=0):
    """The reference's per-window values (the valid grid, nv x nu), computed by the oracle
    in window-row bands: band [v0, v1) needs bin-map rows [v0, v1 + kh - 1)."""
    h, w = qb.shape
    nu, nv = w - kw + 1, h - kh + 1
    cy, cx = (kh - 1) // 2, (kw - 1) // 2
    grid = np.empty((nv, nu), np.float64)
    step = -(-nv // (4 * THREADS))

    def band(v0):
        v1 = min(nv, v0 + step)
        m = oracle.hist_match_map_direct(qb[v0:v1 + kh - 1], nbins, tmpl, kw, kh, p, metric)
        grid[v0:v1] = m[cy:cy + v1 - v0, cx:cx + nu]

    with ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(band, range(0, nv, step)))
    return grid


def _spread(grid, w, h, kw, kh):
    """spread_valid (likelihood.cpp:44-58): every map cell takes the clamped valid window."""
    nv, nu = grid.shape
    cy, cx = (kh - 1) // 2, (kw - 1) // 2
    ys = np.clip(np.arange(h) - cy, 0, nv - 1)
    xs = np.clip(np.arange(w) - cx, 0, nu - 1)
    return grid[ys][:, xs]


def _compare_map(got, want, exact):
    if exact:
        bad = int(np.count_nonzero(got != want))
        assert bad == 0, f"{bad} map cells differ from the reference arithmetic"
    err = np.abs(got - want)
    rel = err / np.maximum(np.abs(want), 1e-12)
    assert rel.max() <= RTOL, f"max relative error {rel.max():.3g}"


def test_c3_every_cell(P):
    side, nbins, kw, kh = 4096, 128, 64, 64
    img = _frame(side, 1)
    qb = oracle.quantize(img, nbins)
    tmpl = _crop_template(qb, nbins, kw, kh)
    t, lmap = P.build_and_match_map(torch.from_numpy(img).cuda(), nbins, tmpl, kw, kh, 1.0)
    got = lmap.cpu().numpy()
    assert _ih_mismatches(t, qb, nbins) == 0
    want = _spread(_valid_grid(qb, nbins, tmpl, kw, kh, 1.0), side, side, kw, kh)
    _compare_map(got, want, exact=True)


def test_c3_general_template_p2_every_window(P):
    side, nbins, kw, kh = 4096, 128, 64, 64
    img = _frame(side, 1)
    qb = oracle.quantize(img, nbins)
    r = np.random.default_rng(3).random(nbins) + 0.1
    tmpl = r / r.sum()
    _, lmap = P.build_and_match_map(torch.from_numpy(img).cuda(), nbins, tmpl, kw, kh, 2.0)
    want = _spread(_valid_grid(qb, nbins, tmpl, kw, kh, 2.0), side, side, kw, kh)
    _compare_map(lmap.cpu().numpy(), want, exact=False)


@pytest.mark.parametrize("p,metric", [(1.0, 0), (1.0, 1), (1.0, 2), (1.0, 3)])
def test_c3_general_template_every_window(P, p, metric):
    """A random normalised template at C3: the fractional-template integer path (p = 1,
    intersection) and the integer / FP32 terms (Bhattacharyya, chi-square), every window."""
    side, nbins, kw, kh = 4096, 128, 64, 64
    img = _frame(side, 1)
    qb = oracle.quantize(img, nbins)
    r = np.random.default_rng(3).random(nbins) + 0.1
    tmpl = r / r.sum()
    _, lmap = P.build_and_match_map(torch.from_numpy(img).cuda(), nbins, tmpl, kw, kh, p, metric)
    want = _spread(_valid_grid(qb, nbins, tmpl, kw, kh, p, metric), side, side, kw, kh)
    _compare_map(lmap.cpu().numpy(), want, exact=False)


def test_c4_every_cell(P):
    side, nbins, kw, kh = 8192, 256, 64, 64
    free = torch.cuda.mem_get_info()[0]
    if free < 80e9:
        pytest.skip(f"C4 needs ~72 GB of device memory ({free / 1e9:.0f} GB free)")
    img = _frame(side, 4)
    qb = oracle.quantize(img, nbins)
    tmpl = _crop_template(qb, nbins, kw, kh)
    t, lmap = P.build_and_match_map(torch.from_numpy(img).cuda(), nbins, tmpl, kw, kh, 1.0)
    got = lmap.cpu().numpy()
    del lmap
    assert _ih_mismatches(t, qb, nbins, group=2) == 0
    del t
    torch.cuda.empty_cache()
    want = _spread(_valid_grid(qb, nbins, tmpl, kw, kh, 1.0), side, side, kw, kh)
    _compare_map(got, want, exact=True)
