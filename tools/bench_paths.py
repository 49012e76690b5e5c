"""Time the fused sweep's code paths at C3 (4096^2 x 128 bins, 64x64 window): the integer
path (integral template) against the FP64 path (non-integral template / p != 1 / other
metrics).  Device-timed, L2 flushed between steps."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_01656_b200 as P

dev = torch.device("cuda", 0)
W = H = 4096
nb, kw, kh = 128, 64, 64
frame = torch.from_numpy(bench.make_frame(W, H)).to(dev)
t = P.IntegralHistogramTensor(W, H, nb, device=dev)
lmap = torch.empty((H, W), dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
integral = bench.template_hist(bench.make_frame(W, H), nb, kw, kh)
fh = bench.make_frame(W, H)
crop = (fh[2000:2063, 2000:2064].astype(np.int64) * nb) >> 8  # 63 x 64 crop: non-integral s_k
nonint = np.bincount(crop.reshape(-1), minlength=nb).astype(np.float64) / crop.size
gen = bench.general_template(nb)
cases = {"integer p=1": (integral, 1.0, 0), "frac p=1 (non-integral crop)": (nonint, 1.0, 0),
         "frac p=1 (random tmpl)": (gen, 1.0, 0), "frac intersection (random)": (gen, 1.0, 1),
         "p=2 (random)": (gen, 2.0, 0), "bhattacharyya (random)": (gen, 1.0, 2), "chi2 (random)": (gen, 1.0, 3),
         "fp64 p=1.5 (random)": (gen, 1.5, 0)}
res = {}
for name, (tm, p, metric) in cases.items():
    td = torch.from_numpy(tm).to(dev)
    for _ in range(2):
        P.build_and_match_map(frame, nb, None, kw, kh, p, metric, out=t, lmap=lmap, tmpl_dev=td)
    ms = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); P.build_and_match_map(frame, nb, None, kw, kh, p, metric, out=t, lmap=lmap, tmpl_dev=td); b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    res[name] = round(sorted(ms)[len(ms) // 2], 3)
print(json.dumps(res))
