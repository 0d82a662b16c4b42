"""Small (latency-bound) calls — configs 1, 2 and 4 — device time per call with CUDA events (back-to-back and
isolated) and host time per call; run under `ncu --metrics gpu__time_duration.sum` for the kernels' own
durations.  Prints one line per case.

  python tools/small_calls.py [--reps N]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def case(sc, mode, split=0):
    beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    nb = P.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
    src = torch.from_numpy(sc.pos_src).cuda()
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
    orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).cuda() if sc.orV_rcv is not None else None
    out = torch.empty((src.shape[0], rcv.shape[0], P.nsamples(sc.Tmax, sc.fs)), device="cuda")
    return lambda: P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                                  mic_pattern=sc.pattern, mode=mode, seed=sc.seed, out=out, split=split)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    cases = [("cfg1", W.cfg1(), "fp32", 0), ("cfg1", W.cfg1(), "poly", 0), ("cfg1", W.cfg1(), "poly", -1),
             ("cfg2_0.7", W.cfg2(0.7), "poly", 0), ("cfg2_2.0", W.cfg2(2.0), "poly", 0),
             ("cfg2_2.0", W.cfg2(2.0), "poly", -1), ("cfg4a", W.cfg4("a"), "poly", 0), ("cfg4b", W.cfg4("b"), "poly", 0)]
    for name, sc, mode, split in cases:
        fn = case(sc, mode, split)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        host = (time.perf_counter() - t) / a.reps * 1e6
        b2b = e0.elapsed_time(e1) * 1e3 / a.reps
        iso = []
        for _ in range(a.reps):
            torch.cuda.synchronize()
            x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x.record()
            fn()
            y.record()
            torch.cuda.synchronize()
            iso.append(x.elapsed_time(y) * 1e3)
        # the same call captured once into a CUDA graph, replayed back to back (launch overhead of one graph)
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            fn()
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            fn()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        gr = e0.elapsed_time(e1) * 1e3 / a.reps
        print(f"{name:10s} {mode:5s} split={split:3d}  back-to-back {b2b:7.1f} us/call  isolated {np.median(iso):7.1f} us  "
              f"host {host:7.1f} us/call  graph replay {gr:7.1f} us/call", flush=True)


if __name__ == "__main__":
    main()
