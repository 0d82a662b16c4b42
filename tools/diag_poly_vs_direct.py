"""Diagnose poly vs direct fp32 at the bench size: per-RIR max difference, and both vs the oracle on the worst RIRs."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1810_11359_b200 as P, oracle
import workloads as W
from helpers import derive, rel_err
sc = W.cfg3(16384, "diffuse"); beta, nb = derive(oracle, sc)
src = torch.from_numpy(np.ascontiguousarray(sc.pos_src)).cuda(); rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
ov = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).cuda()
kw = dict(c=sc.c, orV_rcv=ov, mic_pattern=sc.pattern, seed=sc.seed, sync=True)
a = P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, mode="poly", **kw)[0]
b = P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, mode="fp32", **kw)[0]
err = ((a - b).abs().amax(dim=1) / b.abs().amax(dim=1)).cpu().numpy()
nISM = 2800
errI = ((a[:, :nISM] - b[:, :nISM]).abs().amax(dim=1) / b.abs().amax(dim=1)).cpu().numpy()
print("all max", err.max(), "ism-part max", errI.max(), "p99.9", np.quantile(err, 0.999), "n>5e-5", (err > 5e-5).sum())
for m in [int(err.argmax()), int(errI.argmax())]:
    rj = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[m:m+1], nb, sc.Tdiff, sc.Tmax, fs=sc.fs, pattern=sc.pattern,
                             orV_rcv=sc.orV_rcv[m:m+1], seed=sc.seed, rir_index_base=m)[0, 0]
    A = a[m].cpu().double().numpy(); B = b[m].cpu().double().numpy(); pk = np.abs(rj).max()
    print(m, "poly-oracle", np.abs(A - rj).max() / pk, "at", int(np.abs(A - rj).argmax()), "fp32-oracle", np.abs(B - rj).max() / pk,
          "at", int(np.abs(B - rj).argmax()), "poly ism", np.abs(A - rj)[:nISM].max() / pk, "fp32 ism", np.abs(B - rj)[:nISM].max() / pk)
