"""Small calls from CUDA graphs: µs per call when each replay holds 1 call and when one graph holds n calls back to
back (graph replays are quantised at ~2.05 µs per launch, tools/replay_quantum.py; kernels inside one graph are not)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def call_of(sc):
    beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    nb = P.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
    src = torch.from_numpy(sc.pos_src).cuda()
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
    out = torch.empty((1, rcv.shape[0], P.nsamples(sc.Tmax, sc.fs)), device="cuda")
    return lambda: P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, mode="poly",
                                  seed=sc.seed, out=out)


def us_per_call(fn, calls, reps=30):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(calls):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000.0 / (reps * calls)


if __name__ == "__main__":
    for name, sc in (("cfg1", W.cfg1()), ("cfg2_0.7", W.cfg2(0.7)), ("cfg2_2.0", W.cfg2(2.0))):
        fn = call_of(sc)
        r = [f"{n} per graph {us_per_call(fn, n):6.2f}" for n in (1, 2, 5, 10)]
        print(f"{name:9s} us per call: " + "   ".join(r), flush=True)
