"""Run one C3 kernel a few times (for ncu): `build` (ih_sweep), `fused` (sweep_match), `carries`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P  # noqa: E401,E402
mode = sys.argv[1] if len(sys.argv) > 1 else "build"
dev = torch.device("cuda", 0)
frame = torch.from_numpy(bench.make_frame(4096, 4096)).to(dev)
t = P.IntegralHistogramTensor(4096, 4096, 128, device=dev)
lmap = torch.empty((4096, 4096), dtype=torch.float64, device=dev)
td = torch.from_numpy(bench.template_hist(bench.make_frame(4096, 4096), 128, 64, 64)).to(dev)
for _ in range(3):
    if mode == "fused":
        P.build_and_match_map(frame, 128, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=td)
    else:
        P.build_integral_histogram(frame, 128, memory_budget=None, out=t, validate=False)
torch.cuda.synchronize()
