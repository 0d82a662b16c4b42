"""One trajectory call (traj1 size) repeated, for ncu: python tools/prof_traj.py [split]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11359_b200 as P  # noqa: E402

split = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g = torch.Generator(device="cuda").manual_seed(0)
sig = torch.randn(16000, device="cuda", generator=g)
rirs = torch.randn((100, 32, 11200), device="cuda", generator=g) * 1e-2
out = torch.empty((32, 16000 + 11200 - 1), device="cuda")
for _ in range(4):
    P.simulate_trajectory(sig, rirs, out=out, split=split)
torch.cuda.synchronize()
print("ok")
