"""Per-RIR parity of the bench workload's RIRs [a, b) (config 3 (i), M = 16384) for the polyphase and direct kernels
against the oracle, with where in the RIR the worst sample sits (GPU box).  usage: tools/diag_worst_rir.py a b"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from helpers import derive, run_gpu, run_oracle  # noqa: E402

a, b = int(sys.argv[1]), int(sys.argv[2])
sc = W.cfg3(16384, "diffuse")
beta, nb = derive(oracle, sc)
rcv, orv = sc.pos_rcv[a:b], sc.orV_rcv[a:b]
ref = run_oracle(oracle, sc, beta, nb, pos_rcv=rcv, orv=orv, rir_index_base=a)
for mode in ("poly", "fp32"):
    g = run_gpu(P, sc, beta, nb, mode=mode, split=-1, pos_rcv=rcv, orv=orv, rir_index_base=a)
    g, r2 = g.reshape(-1, g.shape[-1]), ref.reshape(-1, ref.shape[-1])
    d = np.abs(g - r2)
    pk = np.abs(r2).max(axis=1)
    e = d.max(axis=1) / pk
    i = int(np.argmax(e))
    k = int(np.argmax(d[i]))
    print(f"{mode}: worst RIR {a + i} err/peak {e[i]:.3e} at sample {k} (|ref| {abs(r2[i, k]):.3e}, peak {pk[i]:.3e}, "
          f"nISM {int(sc.Tdiff * sc.fs)}); median {np.median(e):.3e}; >3e-5: {int((e > 3e-5).sum())} RIRs")
