"""C3 tensor matcher (hist_match_map of a tensor without a source frame): ms per call with
an L2 flush, and the map compared bit for bit with the fused map of the same frame.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P  # noqa: E401,E402

dev = torch.device("cuda", 0)
fh = bench.make_frame(4096, 4096)
tmpl = bench.template_hist(fh, 128, 64, 64)
frame = torch.from_numpy(fh).to(dev)
t = P.IntegralHistogramTensor(4096, 4096, 128, device=dev)
ref = torch.empty((4096, 4096), dtype=torch.float64, device=dev)
P.build_and_match_map(frame, 128, None, 64, 64, 1.0, out=t, lmap=ref, tmpl_dev=torch.from_numpy(tmpl).to(dev))
t.source = None
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ms = []
for i in range(12):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    m = P.hist_match_map(t, tmpl, 64, 64, 1.0)
    b.record()
    torch.cuda.synchronize()
    if i >= 2:
        ms.append(a.elapsed_time(b))
m = P.hist_match_map(t, tmpl, 64, 64, 1.0)
mt = m if isinstance(m, torch.Tensor) else torch.as_tensor(m, device=dev)
print("tmatch ms", round(sorted(ms)[len(ms) // 2], 4), "min", round(min(ms), 4),
      "bit-equal to fused map:", bool(torch.equal(mt.to(dev), ref)))
