import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1810_11359_b200 as P, workloads as W
for v in ("a", "b"):
    sc = W.cfg4(v)
    beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    nb = P.t2n(sc.Tdiff, sc.room, sc.c)
    src = torch.from_numpy(sc.pos_src).cuda(); rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
    out = torch.empty((1, rcv.shape[0], P.nsamples(sc.Tmax, sc.fs)), device="cuda")
    f = lambda: P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, mic_pattern=sc.pattern, mode="poly", seed=sc.seed, out=out)
    for _ in range(3): f()
    torch.cuda.synchronize()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        f(); g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10): f()
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"cfg4{v} {a.elapsed_time(b) / 50 * 1000:.1f} us per call  sum {float(out.double().abs().sum()):.6f}", flush=True)
