"""Device time of the orientation channel (2048^2, 32 bins, sigma 1) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1711_01656_b200 as P  # noqa: E401,E402
g = torch.randint(0, 256, (2048, 2048), dtype=torch.uint8, device="cuda")
for _ in range(3):
    P.orientation_bins(g, 32, 1.0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    P.orientation_bins(g, 32, 1.0)
b.record()
torch.cuda.synchronize()
print("orientation_bins 2048^2 x 32: %.1f us" % (a.elapsed_time(b) / 50 * 1e3))
