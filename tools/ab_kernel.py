"""A/B of library builds on one box: `python tools/ab_kernel.py libA.so libB.so [rounds]`.
Each build runs in its own process (SPCT_LIB_PATH) and times, device-side with CUDA events
and a 256 MiB L2 flush between steps, the C3 calls: fused integer map, fused fractional
(random template) map, plain build; and the C5 batch per frame."""
import json, os, subprocess, sys

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, bench, paper_1711_01656_b200 as P
dev = torch.device("cuda", 0)
W = H = 4096; nb = 128
fh = bench.make_frame(W, H)
frame = torch.from_numpy(fh).to(dev)
t = P.IntegralHistogramTensor(W, H, nb, device=dev)
lmap = torch.empty((H, W), dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ti = torch.from_numpy(bench.template_hist(fh, nb, 64, 64)).to(dev)
tg = torch.from_numpy(bench.general_template(nb)).to(dev)
def timeit(fn, reps=10):
    for _ in range(3): fn()
    ms = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return round(sorted(ms)[len(ms) // 2], 4)
res = {}
res["c3_int"] = timeit(lambda: P.build_and_match_map(frame, nb, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=ti))
res["c3_frac"] = timeit(lambda: P.build_and_match_map(frame, nb, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=tg))
res["c3_build"] = timeit(lambda: P.build_integral_histogram(frame, nb, memory_budget=None, out=t, validate=False))
if os.environ.get("AB_C5", "1") == "1":
    res["c5_ms_per_frame"] = bench.run_c5(P, dev, torch.cuda.current_stream(), frames=20)["ms_per_frame"]
print(json.dumps(res))
'''

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for r in range(rounds):
    for lib in libs:
        env = dict(os.environ, SPCT_LIB_PATH=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        print(os.path.basename(lib), line, flush=True)
