import sys, os, json
sys.path.insert(0, '.')
import torch, bench, paper_1711_01656_b200 as P
dev = torch.device("cuda", 0)
def timer(fn, steps, warmup=2, flush=False):
    for _ in range(warmup): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(steps):
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return sorted(ms)[len(ms)//2]
pk = {"hbm_gbs": 6500.0}
print(json.dumps(bench.run_c2(P, dev, timer, pk)))
