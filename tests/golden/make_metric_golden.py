"""Golden likelihood maps for the three extension metrics, from published implementations.

The reference implements only the Minkowski-p distance (likelihood.cpp:193-225).  The
thesis names histogram intersection and the Bhattacharyya coefficient as the other
bin-to-bin measures of its sliding-window matcher (ref. [67]); chi-square
is the third common one.  Their values here come from third-party library code, not from
this repository's definitions, so the oracle and the CUDA paths are pinned to a
published implementation:

* histogram intersection (Swain & Ballard 1991, "Color indexing"): sum_k min(q_k, t_k).
  For two histograms that each sum to 1 this is 1 - BC(q, t), BC the Bray-Curtis
  dissimilarity sum|q - t| / sum|q + t|: scipy.spatial.distance.braycurtis (scipy 1.18);
* Bhattacharyya coefficient (Bhattacharyya 1943; Comaniciu, Ramesh & Meer 2003 use it as
  the tracking likelihood): sum_k sqrt(q_k t_k) = 1 - ||sqrt(q) - sqrt(t)||^2 / 2 for
  normalised histograms: scipy.spatial.distance.sqeuclidean on the square roots;
* chi-square (the additive chi^2 kernel of Zhang, Marszalek, Lazebnik & Schmid 2007,
  sklearn.metrics.pairwise.additive_chi2_kernel = -sum_k (q_k - t_k)^2 / (q_k + t_k),
  terms with q_k + t_k = 0 skipped): L = 1 + additive_chi2_kernel(q, t) / 2, i.e.
  1 - half the chi^2 distance, clamped to [0, 1].

q = window histogram / window total, t = template; every value clamped to [0, 1]; the map
is the valid grid spread to the image as spread_valid (likelihood.cpp:44-58).  The window
histograms are counted here with numpy from the bin map (independent of the oracle).

Run from the repo root (needs scipy + scikit-learn, present in this image):
    python tests/golden/make_metric_golden.py
"""
from __future__ import annotations

import os

import numpy as np
import scipy
import sklearn
from scipy.spatial.distance import braycurtis, sqeuclidean
from sklearn.metrics.pairwise import additive_chi2_kernel

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [  # (name, w, h, bins, kw, kh, seed, template kind)
    ("crop", 47, 33, 6, 9, 7, 1, "crop"),
    ("random", 40, 29, 10, 11, 6, 2, "random"),
    ("sparse", 36, 30, 16, 8, 8, 3, "sparse"),   # many empty template bins: q + t = 0 terms
]


def window_hists(bm: np.ndarray, bins: int, kw: int, kh: int) -> np.ndarray:
    """(nv, nu, bins) float64 counts of every kw x kh window (numpy, no integral image)."""
    h, w = bm.shape
    onehot = (bm[..., None] == np.arange(bins)).astype(np.int64)
    ii = np.zeros((h + 1, w + 1, bins), np.int64)
    ii[1:, 1:] = onehot.cumsum(0).cumsum(1)
    c = ii[kh:, kw:] - ii[:-kh, kw:] - ii[kh:, :-kw] + ii[:-kh, :-kw]
    return c.astype(np.float64)


def spread(grid: np.ndarray, w: int, h: int, kw: int, kh: int) -> np.ndarray:
    nv, nu = grid.shape
    ys = np.clip(np.arange(h) - (kh - 1) // 2, 0, nv - 1)
    xs = np.clip(np.arange(w) - (kw - 1) // 2, 0, nu - 1)
    return grid[ys][:, xs]


def main() -> None:
    out = {"versions": np.array([f"scipy {scipy.__version__}", f"scikit-learn {sklearn.__version__}"])}
    for name, w, h, bins, kw, kh, seed, kind in CASES:
        rng = np.random.default_rng(seed)
        bm = rng.integers(0, bins, (h, w)).astype(np.uint16)
        if kind == "sparse":
            bm = (bm // 4 * 4).astype(np.uint16)  # only every 4th bin occurs
        c = window_hists(bm, bins, kw, kh)
        q = c / c.sum(-1, keepdims=True)
        if kind == "crop":
            t = c[5, 7] / c[5, 7].sum()
        elif kind == "random":
            r = rng.random(bins) + 0.05
            t = r / r.sum()
        else:
            r = np.zeros(bins)
            r[::4] = rng.random(bins // 4) + 0.1
            r[1] = 0.02  # a template bin that never occurs in the image
            t = r / r.sum()
        qs = q.reshape(-1, bins)
        inter = np.array([1.0 - braycurtis(a, t) for a in qs])
        bhat = np.array([1.0 - sqeuclidean(np.sqrt(a), np.sqrt(t)) / 2.0 for a in qs])
        chi = 1.0 + additive_chi2_kernel(qs, t[None, :])[:, 0] / 2.0
        nv, nu = c.shape[:2]
        for key, v in (("intersection", inter), ("bhattacharyya", bhat), ("chisq", chi)):
            grid = np.clip(v, 0.0, 1.0).reshape(nv, nu)
            out[f"{name}_{key}"] = spread(grid, w, h, kw, kh)
        out[f"{name}_binmap"] = bm
        out[f"{name}_template"] = t
        out[f"{name}_dims"] = np.array([w, h, bins, kw, kh])
    np.savez_compressed(os.path.join(OUT, "metric_vectors.npz"), **out)
    print("wrote", os.path.join(OUT, "metric_vectors.npz"))


if __name__ == "__main__":
    main()
