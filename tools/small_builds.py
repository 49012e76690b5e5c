"""Device time of builds with few bins (C1 512^2 x 16, C2 1024^2 x 32, 1024^2 x 16) and the median slide."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1711_01656_b200 as P  # noqa: E401,E402
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for (n, nb) in [(512, 16), (1024, 32), (1024, 16), (2048, 32), (4096, 128)]:
    f = torch.randint(0, 256, (n, n), dtype=torch.uint8, device="cuda")
    tt = P.IntegralHistogramTensor(n, n, nb)
    ms = t(lambda: P.build_integral_histogram(f, nb, memory_budget=None, out=tt, validate=False))
    print(f"build {n}^2 x {nb}: {ms*1e3:.1f} us  {nb*n*n*4/ms/1e6:.0f} GB/s")
fr = [torch.randint(0, 16, (1024, 1024), dtype=torch.uint8, device="cuda") for _ in range(8)]
mb = P.motion.MedianBackgroundIH(fr[:5], 16, 7, 7)
it = iter(range(10**9))
print("median slide: %.1f us" % (t(lambda: mb.slide(fr[5 + next(it) % 3])) * 1e3))
