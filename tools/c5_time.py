"""C5 tracking batch ms/frame (bench.run_c5), e.g. SPCT_NO_SIDE_STREAMS=1 python tools/c5_time.py."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench, paper_1711_01656_b200 as P  # noqa: E401,E402

dev = torch.device("cuda", 0)
r = [bench.run_c5(P, dev, torch.cuda.current_stream(), frames=100)["ms_per_frame"] for _ in range(3)]
print("c5 ms/frame", r, "side streams", "off" if os.environ.get("SPCT_NO_SIDE_STREAMS") else "on")
