"""Per-rank work of C3 strong scaling on one GPU: the fused sweep of a bin slab (16/32/64/128
of 128 bins) writing its tensor slab and partial window sums; device time + roofline."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P
dev = torch.device("cuda", 0)
W = H = 4096; nb = 128
fh = bench.make_frame(W, H)
frame = torch.from_numpy(fh).to(dev)
tm = torch.from_numpy(bench.template_hist(fh, nb, 64, 64)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
part = torch.empty((H - 63, W - 63), dtype=torch.float64, device=dev)
res = {}
for k in (128, 64, 32, 16):
    t = P.IntegralHistogramTensor(W, H, nb, bin0=0, bins=k, device=dev)
    fn = lambda: P.build_and_match(frame, nb, None, 64, 64, 1.0, bin0=0, bins=k, out=t, partial=part, tmpl_dev=tm)
    for _ in range(3): fn()
    ms = []
    for _ in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    m = sorted(ms)[4]
    alg = k * W * H * 4 + W * H + (W - 63) * (H - 63) * 8
    res[k] = {"ms": round(m, 4), "tb_s": round(alg / m / 1e9, 2)}
    del t
print(json.dumps(res))
