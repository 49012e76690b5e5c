"""C4 (8192^2 x 256 bins, one GPU) fused build + map: device time per step (L2-flushed)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P
dev = torch.device("cuda", 0)
side, nb = 8192, 256
fh = bench.make_frame(side, side, seed=4)
frame = torch.from_numpy(fh).to(dev)
t = P.IntegralHistogramTensor(side, side, nb, device=dev)
lmap = torch.empty((side, side), dtype=torch.float64, device=dev)
td = torch.from_numpy(bench.template_hist(fh, nb, 64, 64)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fn = lambda: P.build_and_match_map(frame, nb, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=td)
for _ in range(2): fn()
ms = []
for _ in range(5):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
print(json.dumps({"c4_ms": sorted(ms)[2], "checksum": float(lmap[::97, ::89].sum())}))
