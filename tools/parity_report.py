"""Parity report: max per-RIR |h_gpu - h_oracle| / max|h_oracle| for every config and mode (GPU box).

Writes one line per (config, mode, kernel) to stdout; used for profiles/r01_parity.txt.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402
from helpers import TOL, derive, rel_err, run_gpu, run_oracle  # noqa: E402


def report(name, sc, modes=("fp32", "lut", "fp16", "lut_tex", "poly"), kernels=(0, -1)):
    beta, nb = derive(oracle, sc)
    r = run_oracle(oracle, sc, beta, nb)
    for mode in modes:
        for k in kernels:
            g = run_gpu(P, sc, beta, nb, mode=mode, split=k)
            e = rel_err(g, r)
            kn = "persistent" if k == -1 else "auto"
            flag = "OK" if e.max() <= TOL[mode] else "FAIL"
            print(f"{name:28s} {mode:5s} {kn:10s} M={e.size:4d} max_err/peak={e.max():.3e} "
                  f"median={np.median(e):.3e} tol={TOL[mode]:.0e} {flag}", flush=True)


def main():
    report("cfg1", W.cfg1())
    for T60 in (0.2, 0.5, 1.0, 2.0):
        report(f"cfg2_T60_{T60}", W.cfg2(T60), modes=("fp32",))
    report("cfg3_diffuse_M32", W.cfg3(32, "diffuse"))
    sc = W.cfg3(8, "full")
    report("cfg3_full_M8", sc)
    sc = W.cfg4("a")
    sc.pos_rcv = sc.pos_rcv[:8]
    report("cfg4a_48k_M8", sc)
    sc = W.cfg4("b")
    sc.pos_rcv = sc.pos_rcv[:4]
    report("cfg4b_48k_fullISM_M4", sc)


if __name__ == "__main__":
    main()
