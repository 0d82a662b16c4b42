"""Time gpurir_simulate_rir_host against its parts (run on the GPU box): wall time per call at several M,
pinned vs pageable output, and the device call + a plain D2H of the same bytes for comparison."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
import oracle  # noqa: E402


def main():
    for M in (2048, 4096, 16384):
        sc = W.cfg3(M, "diffuse")
        beta, _ = oracle.beta_sabine(sc.room, sc.T60)
        beta = beta.astype(np.float32)
        nb = oracle.t2n(sc.Tdiff, sc.room, sc.c)
        nS = P.nsamples(sc.Tmax, sc.fs)
        src, rcv, orv = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (sc.pos_src, sc.pos_rcv, sc.orV_rcv))
        out = torch.empty((1, M, nS), dtype=torch.float32).pin_memory()
        kw = dict(c=sc.c, orV_rcv=orv, mic_pattern=sc.pattern, mode="poly", seed=sc.seed)
        for rep in range(4):
            t = time.perf_counter()
            P.simulate_rir_host(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, out=out, **kw)
            dt = time.perf_counter() - t
            print(f"M={M} host call pinned rep{rep}: {dt*1e3:.2f} ms  ({M/dt:.0f} RIRs/s)", flush=True)
        d = torch.empty((1, M, nS), dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        t = time.perf_counter()
        out.copy_(d)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"M={M} plain D2H {out.numel()*4/1e6:.0f} MB: {dt*1e3:.2f} ms ({out.numel()*4/dt/1e9:.1f} GB/s)", flush=True)
        dsrc, drcv, dorv = src.cuda(), rcv.cuda(), orv.cuda()
        torch.cuda.synchronize()
        t = time.perf_counter()
        P.simulate_rir(sc.room, beta, dsrc, drcv, nb, sc.Tdiff, sc.Tmax, sc.fs, out=d, c=sc.c, orV_rcv=dorv,
                       mic_pattern=sc.pattern, mode="poly", seed=sc.seed)
        torch.cuda.synchronize()
        print(f"M={M} device call: {(time.perf_counter()-t)*1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
