"""Run one bench workload a few times (for ncu launch lists): c3 | c4 | c5 | tmatch | gen_p1 | gen_p2 | gen_bhat."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench, paper_1711_01656_b200 as P  # noqa: E401,E402
from paper_1711_01656_b200.sharding import ShardedMapStep  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
if mode == "c5":
    class A: pass
    print(bench.run_c5(P, dev, torch.cuda.current_stream(), frames=reps))
    raise SystemExit
side, nb = (8192, 256) if mode == "c4" else (4096, 128)
fh = bench.make_frame(side, side, seed=4 if mode == "c4" else 1)
tmpl = bench.template_hist(fh, nb, 64, 64)
frame = torch.from_numpy(fh).to(dev)
if mode in ("c3", "c4"):
    st = ShardedMapStep(side, side, nb, tmpl, 64, 64, 1.0, device=dev)
    for _ in range(reps):
        st.step(frame)
else:
    t = P.IntegralHistogramTensor(side, side, nb, device=dev)
    lmap = torch.empty((side, side), dtype=torch.float64, device=dev)
    P.build_and_match_map(frame, nb, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=torch.from_numpy(tmpl).to(dev))
    if mode == "tmatch":
        t.source = None
        for _ in range(reps):
            P.hist_match_map(t, tmpl, 64, 64, 1.0)
    else:
        p, metric = {"gen_p1": (1.0, 0), "gen_p2": (2.0, 0), "gen_bhat": (1.0, 2)}[mode]
        g = torch.from_numpy(bench.general_template(nb)).to(dev)
        for _ in range(reps):
            P.build_and_match_map(frame, nb, None, 64, 64, p, metric, out=t, lmap=lmap, tmpl_dev=g)
torch.cuda.synchronize()
print("done", mode)
