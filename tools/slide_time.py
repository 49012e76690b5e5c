"""Joint-IH slide at 1024^2 x 16 bins, 5 frames: device time per slide (spct_cu_ih_slide)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1711_01656_b200 as P
g = torch.Generator(device="cuda"); g.manual_seed(3)
n = 1024
fr = [torch.randint(0, 16, (n, n), dtype=torch.uint8, device="cuda", generator=g) for _ in range(8)]
mb = P.motion.MedianBackgroundIH(fr[:5], 16, 7, 7)
for i in range(3): mb.slide(fr[5 + i % 3])
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(20): mb.slide(fr[5 + i % 3])
b.record(); torch.cuda.synchronize()
print("slide ms", a.elapsed_time(b) / 20)
