"""C3 step shapes: fused sweep vs build + no-store map (sequential and on two streams)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P  # noqa: E401,E402

dev = torch.device("cuda", 0)
fr = bench.make_frame(4096, 4096)
frame = torch.from_numpy(fr).to(dev)
t = P.IntegralHistogramTensor(4096, 4096, 128, device=dev)
t_ns = P.IntegralHistogramTensor(4096, 4096, 128, device=dev)
t_ns.desc.data = None
lmap = torch.empty((4096, 4096), dtype=torch.float64, device=dev)
lmap2 = torch.empty_like(lmap)
td = torch.from_numpy(bench.template_hist(fr, 128, 64, 64)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s1 = torch.cuda.Stream(dev)
lo, hi = torch.cuda.Stream.priority_range()
s2 = torch.cuda.Stream(dev, priority=hi)
s3 = torch.cuda.Stream(dev, priority=lo)


def fused():
    P.build_and_match_map(frame, 128, None, 64, 64, 1.0, out=t, lmap=lmap, tmpl_dev=td)


def build(stream=None):
    P.build_integral_histogram(frame, 128, memory_budget=None, out=t, validate=False, stream=stream)


def mapo(stream=None):
    P.build_and_match_map(frame, 128, None, 64, 64, 1.0, out=t_ns, lmap=lmap2, tmpl_dev=td, stream=stream)


def both(sa, sb, map_first):
    cur = torch.cuda.current_stream(dev)
    sa.wait_stream(cur)
    sb.wait_stream(cur)
    if map_first:
        mapo(sb)
        build(sa)
    else:
        build(sa)
        mapo(sb)
    cur.wait_stream(sa)
    cur.wait_stream(sb)


cases = {
    "fused": fused,
    "build": build,
    "map_nostore": mapo,
    "build+map seq": lambda: (build(), mapo()),
    "two streams (map hi prio, first)": lambda: both(s3, s2, True),
    "two streams (build first, map hi)": lambda: both(s3, s2, False),
    "two streams (same prio)": lambda: both(s1, torch.cuda.Stream(dev), True),
}
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{name:40s} median {ts[5]:.4f} ms  min {ts[0]:.4f}", flush=True)
ok = torch.equal(lmap, lmap2)
print("map equal fused vs no-store:", ok)
