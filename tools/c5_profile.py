"""Run a few config-5 frames (for ncu launch lists / timing of the tracking batch)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1711_01656_b200 as P

class A: pass
dev = torch.device("cuda", 0)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t0 = time.perf_counter()
r = bench.run_c5(P, dev, torch.cuda.current_stream(), A(), frames=frames)
print(r, "wall", time.perf_counter() - t0)
