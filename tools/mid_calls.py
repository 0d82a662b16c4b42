"""Mid-size polyphase calls (--graph: 10 calls per CUDA graph) (config 3 (i) with M receivers): device time per call (CUDA events over 20
back-to-back calls after warm-up) for the automatic plan and for forced persistent CTAs (split = -1).
  python tools/mid_calls.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def timed(sc, split, reps=20):
    beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    nb = P.t2n(sc.Tdiff, sc.room, sc.c)
    src = torch.from_numpy(sc.pos_src).cuda()
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
    orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).cuda()
    out = torch.empty((1, rcv.shape[0], P.nsamples(sc.Tmax, sc.fs)), device="cuda")
    f = lambda: P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,  # noqa
                               mic_pattern=sc.pattern, mode="poly", seed=sc.seed, out=out, split=split)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:  # 10 calls per CUDA graph: device time per call without the host's launch overhead
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            f()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    f()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(reps // 10):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / (reps // 10 * 10) * 1000.0, out.clone()
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000.0, out.clone()


GRAPH = "--graph" in sys.argv
Ms = (1, 2, 4, 8, 12, 16, 24, 32, 48, 64, 96, 128, 192, 256) if GRAPH else (4, 8, 16, 32, 48, 64, 96, 128, 192, 256)
if "--large" in sys.argv:
    Ms = (64, 96, 128, 192, 256, 384, 512, 768, 1024, 2048)
for M in Ms:
    sc = W.cfg3(M, "diffuse")
    ta, oa = timed(sc, 0)
    tp, op = timed(sc, -1)
    same = bool(torch.equal(oa, op))
    print(f"M={M:4d} auto {ta:7.1f} us  persistent {tp:7.1f} us  same_bits={same}", flush=True)
