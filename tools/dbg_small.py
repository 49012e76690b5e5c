import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_1711_01656_b200 as P
def run(img, bins, th, kw, kh, store):
    qb = oracle.quantize(img, bins)
    h, w = img.shape
    t = P.IntegralHistogramTensor(w, h, bins)
    if not store: t.desc.data = None
    _, lm = P.build_and_match_map(img, bins, np.array(th), kw, kh, 1.0, out=t)
    want = oracle.hist_match_map_direct(qb, bins, np.array(th), kw, kh, 1.0)
    return lm.cpu().numpy(), want
img = np.array([[0, 100], [100, 200], [200, 200]], np.uint8)
for store in (True, False):
    g, w = run(img, 3, [0.4, 0.4, 0.2], 2, 3, store); print('2x3', store, g.ravel()[:3], w.ravel()[:3])
rng = np.random.default_rng(1)
for (W, H, kw, kh) in [(2,3,2,3),(3,3,2,3),(4,4,2,2),(8,6,3,3),(20,10,5,4),(130,20,5,4),(300,40,64,8)]:
    img = rng.integers(0, 256, (H, W), dtype=np.uint8)
    th = rng.random(3); th /= th.sum()
    for store in (True, False):
        g, w = run(img, 3, th, kw, kh, store)
        print(W, H, kw, kh, store, 'maxerr', np.abs(g - w).max())
