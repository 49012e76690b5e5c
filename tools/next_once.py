"""Run the 8(f) kernels once each after a warm-up (for ncu): SWIH quadrant build, direct
swlh map, orientation, find_peaks / score_map, camshift."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, paper_1711_01656_b200 as P  # noqa: E401,E402
g = torch.Generator(device="cuda"); g.manual_seed(11)
bm = torch.randint(0, 32, (1024, 1024), dtype=torch.int16, device="cuda", generator=g)
gray = torch.randint(0, 256, (2048, 2048), dtype=torch.uint8, device="cuda", generator=g)
m = torch.rand((4096, 4096), dtype=torch.float64, device="cuda", generator=g)
for _ in range(2):
    P.swih.build_quadrant_set(bm, 32, 31, 31)
    P.swih.swlh_distance_map(bm, 32, np.full(32, 1 / 32), 31, 31)
    P.orientation_bins(gray, 32, 1.0)
    P.find_peaks(m)
    P.score_map(m, 1000, 1000, 64, 64)
    P.camshift_batch(m, [[64 + 61 * i, 64 + 57 * i] for i in range(64)], 64, 64)
torch.cuda.synchronize()
