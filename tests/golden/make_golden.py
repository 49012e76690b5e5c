"""Generate the committed golden fixtures for the hot path.

Two kinds of fixtures, both committed next to this script:

* ``known_answers.json`` — the literal known answers the reference's own tests
  assert (file:line cited per entry).  They are transcribed, not computed.
* ``ref_vectors.npz``   — outputs of the UNMODIFIED reference (oracle/_ref, built
  from /root/reference/proj/src by oracle/Makefile) on small seeded inputs:
  padded uint64 integral histograms, region histograms and likelihood maps.
  They let the GPU box (where /root/reference does not exist) pin both the C
  oracle and the CUDA path against the reference itself.

Run from the repo root:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

KNOWN = {
    "ih_2x2": {
        "cite": "proj/tests/test_integral.cpp:40-57",
        "binmap": [[0, 1], [1, 0]], "bins": 2,
        "expect_at": [[0, 2, 2, 2], [1, 2, 2, 2], [0, 1, 1, 1], [1, 1, 1, 0]],  # (k, y, x, value)
        "padding_zero": True,
    },
    "ih_1x1": {
        "cite": "SPEC.md:121 (build example 3)",
        "binmap": [[5]], "bins": 8,
        "nonzero": [[5, 1, 1, 1]],
    },
    "quantize_32": {
        "cite": "proj/tests/test_imagecore.cpp:88-95",
        "pixels": [0, 64, 128, 255], "bins": 32, "lo": 0.0, "hi": 256.0, "expect": [0, 8, 16, 31],
    },
    "quantize_clamp": {
        "cite": "proj/tests/test_imagecore.cpp:97-101",
        "pixels": [0, 64, 128, 255], "bins": 4, "lo": 100.0, "hi": 200.0, "expect_first": 0, "expect_last": 3,
    },
    "quantize_contract": {
        "cite": "proj/tests/test_imagecore.cpp:102-106",
        "bad": [[0, 0.0, 256.0], [70000, 0.0, 256.0], [8, 10.0, 10.0]],
    },
    "grayscale": {
        "cite": "proj/tests/test_imagecore.cpp:48-50",
        "rgb": [[10, 20, 40], [255, 255, 255]], "expect": [23, 255],
    },
    "hist_fixture_0p7": {
        "cite": "proj/tests/test_likelihood.cpp:183-194",
        "image": [[0, 100], [100, 200], [200, 200]], "bins": 3,
        "template": [0.4, 0.4, 0.2], "kw": 2, "kh": 3, "p": 1.0,
        "at": [0, 1], "expect": 0.7, "eps": 1e-12,
    },
    "schedule_stats": {
        "cite": "proj/tests/test_integral.cpp:155-174, acceptance.cpp:242-256",
        "cases": [
            {"args": [1024, 1024, 32, 1024], "iters": 63, "tiles": 1024, "eff_lo": 0.29, "eff_hi": 0.31},
            {"args": [512, 512, 32, 512], "iters": 31, "tiles": 256},
            {"args": [70, 33, 32, 64], "iters": 4, "tiles": 6},
            {"args": [512, 512, 32, 1024], "iters": 31, "tiles": 256, "eff_lo": 0.29, "eff_hi": 0.31},
        ],
        "bad": [[0, 4, 32, 64], [4, 4, 32, 1]],
    },
    "estimate_memory": {
        "cite": "proj/tests/test_integral.cpp:176-188",
        "cases": [
            {"args": [2048, 2048, 64, 1], "raw": 2048 * 2048 * 64, "degenerate": False},
            {"args": [512, 512, 32, 8], "raw": 64 * 1024 * 1024, "padded": 32 * 513 * 513 * 8},
            {"args": [100, 100, 0, 8], "degenerate": True},
        ],
        "bad": [[-1, 4, 4, 4]],
    },
    "budget_reject": {
        "cite": "proj/tests/test_integral.cpp:196-198",
        "w": 16, "h": 16, "bins": 4, "budget": 64,
    },
}


def ref_vectors():
    """Reference outputs on seeded inputs (sizes from test_integral.cpp:74)."""
    if not oracle.have_ref():
        raise SystemExit("oracle/_ref/libspct_ref.so missing: run `make -C oracle` with /root/reference present")
    vec = {}
    sizes = [(1, 1), (5, 3), (33, 31), (64, 64), (70, 129), (256, 40)]
    for i, (w, h) in enumerate(sizes):
        bm = oracle.random_binmap(w, h, 16, 1000 + i)  # test_integral.cpp:76-78 seeds
        t = oracle.RefTensor(bm, 16, oracle.SEQUENTIAL)
        vec[f"ih_{w}x{h}_bins"] = bm
        vec[f"ih_{w}x{h}_tensor"] = t.array()
    # region queries on a 200x150/32 map (test_integral.cpp:107-121)
    bm = oracle.random_binmap(200, 150, 32, 7)
    t = oracle.RefTensor(bm, 32, oracle.WF_TIS, 32, 4)
    rng = np.random.default_rng(8)
    rects = []
    for _ in range(64):
        x1, y1 = int(rng.integers(0, 200)), int(rng.integers(0, 150))
        rects.append([x1, y1, int(rng.integers(0, 200 - x1 + 1)), int(rng.integers(0, 150 - y1 + 1))])
    rects = np.asarray(rects, np.int32)
    vec["region_bins"] = bm
    vec["region_rects"] = rects
    vec["region_hists"] = np.stack([t.region_histogram(*r) for r in rects])
    # likelihood maps: the hist-distance spot-check image (test_likelihood.cpp:196-215)
    img = oracle.noise_image(30, 22, 19)
    qb = oracle.ref_quantize(img, 8)
    t = oracle.RefTensor(qb, 8)
    tmpl = np.full(8, 1.0 / 8)
    vec["lmap_noise_img"] = img
    vec["lmap_noise_p2"] = t.hist_distance_map(tmpl, 7, 5, 2.0)
    vec["lmap_noise_p1"] = t.hist_distance_map(tmpl, 7, 5, 1.0)
    # a 96x80 smooth frame with a template cut from the frame itself (p = 1 and 3)
    img = oracle.smooth_image(96, 80, 21)
    qb = oracle.ref_quantize(img, 16)
    t = oracle.RefTensor(qb, 16)
    crop = qb[30:46, 40:60]
    th = np.bincount(crop.reshape(-1), minlength=16).astype(np.float64) / crop.size
    vec["lmap_smooth_img"] = img
    vec["lmap_smooth_tmpl"] = th
    vec["lmap_smooth_p1"] = t.hist_distance_map(th, 20, 16, 1.0)
    vec["lmap_smooth_p3"] = t.hist_distance_map(th, 20, 16, 3.0)
    # grayscale + quantize on a color frame (test_util.hpp:56-68 noise_color)
    r, g, b = oracle.noise_color(64, 48, 1)
    gray = oracle.ref_to_grayscale(r, g, b)
    vec["color_r"], vec["color_g"], vec["color_b"] = r, g, b
    vec["color_gray"] = gray
    vec["color_q32"] = oracle.ref_quantize(gray, 32)
    vec["color_q7_lohi"] = oracle.ref_quantize(gray, 7, 30.0, 200.0)
    return vec


def main():
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(KNOWN, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "ref_vectors.npz"), **ref_vectors())
    print("wrote", os.path.join(OUT, "known_answers.json"), os.path.join(OUT, "ref_vectors.npz"))


if __name__ == "__main__":
    main()
