"""Device time of the SWIH build / map pieces (1024^2, 32 bins, 31x31)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_1711_01656_b200 as P  # noqa: E401,E402
n, nb, k = 1024, 32, 31
g = torch.Generator(device="cuda"); g.manual_seed(11)
bm = torch.randint(0, nb, (n, n), dtype=torch.int16, device="cuda", generator=g)
model = np.full(nb, 1.0 / nb)
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
s = P.swih.build_quadrant_set(bm, nb, k, k)
print("quadrant set: %.3f ms" % t(lambda: P.swih.build_quadrant_set(bm, nb, k, k)))
print("one tensor:   %.3f ms" % t(lambda: P.swih.build_weighted_tensor(bm, np.ones((n, n), np.uint64) << 16, nb)))
print("map (incl. set): %.3f ms" % t(lambda: P.swih.swlh_distance_map(bm, nb, model, k, k)))
