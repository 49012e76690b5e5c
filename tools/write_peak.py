"""Write-only and copy HBM bandwidth on this GPU (torch fill / copy kernels, CUDA events)."""
import json
import torch

n = 8_589_934_592 // 4  # 8.59 GB of uint32, the C3 tensor size
x = torch.empty(n, dtype=torch.int32, device="cuda")
y = torch.empty(n // 2, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for name, fn, nbytes in [("fill", lambda: x.fill_(7), 4 * n), ("copy", lambda: y.copy_(x[: n // 2]), 4 * n)]:
    ts = []
    for i in range(8):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    t = min(ts)
    res[name] = {"ms": t, "GBs": nbytes / t / 1e6}
print(json.dumps(res))
