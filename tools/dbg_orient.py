import sys; sys.path.insert(0, '.')
import numpy as np, oracle, paper_1711_01656_b200 as P
h, w = 20, 30
y, x = np.mgrid[0:h, 0:w]
for name, img in [("xramp", 3 * x), ("yramp", 3 * y), ("diag", x + y), ("smooth", oracle.smooth_image(w, h, 7))]:
    img = np.ascontiguousarray(img % 256, np.uint8)
    for s in (1.0, 0.0, 1.5):
        got = P.api.as_numpy_u16(P.orientation_bins(img, 32, s))
        want = oracle.orientation_bins(img, 32, s)
        print(name, s, int((got != want).sum()), got[10, 5:12].tolist(), want[10, 5:12].tolist())
