"""One small call, repeated (for ncu -s/-c): python tools/prof_small.py cfg1|cfg2_0.7|cfg4a [mode] [split]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
mode = sys.argv[2] if len(sys.argv) > 2 else "poly"
split = int(sys.argv[3]) if len(sys.argv) > 3 else 0
sc = {"cfg1": W.cfg1, "cfg2_0.7": lambda: W.cfg2(0.7), "cfg2_2.0": lambda: W.cfg2(2.0), "cfg4a": lambda: W.cfg4("a"),
      "cfg4b": lambda: W.cfg4("b")}[name]()
beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
nb = P.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
src = torch.from_numpy(sc.pos_src).cuda()
rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).cuda() if sc.orV_rcv is not None else None
out = torch.empty((src.shape[0], rcv.shape[0], P.nsamples(sc.Tmax, sc.fs)), device="cuda")
for _ in range(8):
    P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv, mic_pattern=sc.pattern,
                   mode=mode, seed=sc.seed, out=out, split=split)
torch.cuda.synchronize()
print("ok", name, mode, split)
