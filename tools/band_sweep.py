"""C3 fused step time against forced band heights (SPCT_BAND_ROWS), device-timed with an L2 flush."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P

dev = torch.device("cuda", 0)
W = H = 4096; nb = 128
fh = bench.make_frame(W, H)
frame = torch.from_numpy(fh).to(dev)
t = P.IntegralHistogramTensor(W, H, nb, device=dev)
lmap = torch.empty((H, W), dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ti = torch.from_numpy(bench.template_hist(fh, nb, 64, 64)).to(dev)
res = {}
for br in [int(x) for x in (sys.argv[1:] or ["0", "455", "410", "342", "293", "228", "152", "111", "86"])]:
    if br:
        os.environ["SPCT_BAND_ROWS"] = str(br)
    else:
        os.environ.pop("SPCT_BAND_ROWS", None)
    fn = lambda: P.build_and_match_map(frame, nb, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=ti)
    for _ in range(3): fn()
    ms = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    res[br] = round(sorted(ms)[5], 4)
print(json.dumps(res))
