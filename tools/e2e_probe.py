"""Timeline of bench.py's e2e loop (cfg3, 16384 RIRs per step): per-step kernel / D2H events on two streams,
to see how much of the 734 MB D2H overlaps the next step's kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def main(n=6):
    sc = W.cfg3(16384, "diffuse")
    dev = torch.device("cuda", 0)
    beta, _ = P.beta_sabine(sc.room, sc.T60)
    nb = P.t2n(sc.Tdiff, sc.room, sc.c)
    nS = P.nsamples(sc.Tmax, sc.fs)
    h_src = torch.from_numpy(sc.pos_src).pin_memory()
    h_rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).pin_memory()
    h_orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).pin_memory()
    h_out = [torch.empty((1, 16384, nS)).pin_memory() for _ in range(2)]
    d_out = [torch.empty((1, 16384, nS), device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def run(mode):
        torch.cuda.synchronize()
        t0 = E()
        t0.record(torch.cuda.current_stream())
        for s in streams:
            s.wait_event(t0)
        evs = []
        for i in range(n):
            s = streams[i % 2]
            with torch.cuda.stream(s):
                a, b, c = E(), E(), E()
                d_src = h_src.to(dev, non_blocking=True)
                d_rcv = h_rcv.to(dev, non_blocking=True)
                d_orv = h_orv.to(dev, non_blocking=True)
                a.record(s)
                if mode != "copy":
                    P.simulate_rir(sc.room, beta, d_src, d_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=d_orv,
                                   mic_pattern=sc.pattern, seed=sc.seed, out=d_out[i % 2], stream=s)
                b.record(s)
                if mode != "kernel":
                    h_out[i % 2].copy_(d_out[i % 2], non_blocking=True)
                c.record(s)
                evs.append((a, b, c))
        torch.cuda.synchronize()
        tot = max(t0.elapsed_time(c) for _, _, c in evs)
        print(f"{mode:8s} total {tot:8.2f} ms  per step {tot / n:6.2f} ms")
        for i, (a, b, c) in enumerate(evs):
            print(f"   step {i}: kernel {t0.elapsed_time(a):8.2f} -> {t0.elapsed_time(b):8.2f}   "
                  f"D2H -> {t0.elapsed_time(c):8.2f}")

    for mode in ("kernel", "copy", "both", "both"):
        run(mode)


if __name__ == "__main__":
    main()
