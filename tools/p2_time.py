"""C3 fused map with a random (non-integral) template at p = 2: ms per step (L2-flushed),
and the max relative difference to the FP64 path (SPCT_P2_MODE3=1 selects the full-warp MODE 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P  # noqa: E401,E402

dev = torch.device("cuda", 0)
side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 128
fh = bench.make_frame(side, side)
frame = torch.from_numpy(fh).to(dev)
t = P.IntegralHistogramTensor(side, side, nb, device=dev)
lmap = torch.empty((side, side), dtype=torch.float64, device=dev)
g = torch.from_numpy(bench.general_template(nb)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
fn = lambda: P.build_and_match_map(frame, nb, None, 64, 64, 2.0, 0, out=t, lmap=lmap, tmpl_dev=g)
for _ in range(3): fn()
ms = []
for _ in range(10):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
got = lmap.clone()
print(side, nb, "p2 ms", round(sorted(ms)[5], 4), "map checksum", float(got[::61, ::67].sum()))
