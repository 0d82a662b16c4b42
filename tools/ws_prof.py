"""Per-role cycle breakdown of the persistent ISM kernel (profiling build only).

  tools/build_variant.sh prof -DGPURIR_WS_PROF
  GPURIR_LIB=build/prof.so python tools/ws_prof.py
Runs bench.py's workload (cfg3, 16384 receivers) and prints where producer and consumer warps spend cycles.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11359_b200 as P  # noqa: E402
from paper_1810_11359_b200 import _lib  # noqa: E402
import workloads as W  # noqa: E402


def main():
    sc = W.cfg3(16384, "diffuse")
    dev = torch.device("cuda", 0)
    beta, _ = P.beta_sabine(sc.room, sc.T60)
    nb = P.t2n(sc.Tdiff, sc.room, sc.c)
    src = torch.from_numpy(sc.pos_src).to(dev)
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).to(dev)
    orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).to(dev)
    out = torch.empty((1, 16384, P.nsamples(sc.Tmax, sc.fs)), device=dev)
    lib = _lib.lib()
    fn = lib.gpurir_debug_ws_prof
    fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
    buf = (C.c_ulonglong * 64)()

    def run():
        P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                       mic_pattern=sc.pattern, seed=sc.seed, out=out)
        torch.cuda.synchronize()
    run()
    fn(buf, 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    fn(buf, 0)
    v = list(buf)
    ms = a.elapsed_time(b)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n_ctas = 2 * sms
    per_warp_cycles = ms * 1e-3 * 1.965e9
    pw = n_ctas * 8
    print(f"call {ms:.3f} ms; per-warp budget {per_warp_cycles:.3g} cycles; {pw} producer warps, {pw} consumer warps")
    names = {0: "publish (sort+handoff)", 1: "  of which EMPTY wait", 2: "tile setup (serial + barriers)",
             3: "column phase", 4: "image loop (+ full-window publishes)"}
    for i, nm in names.items():
        print(f"producer {nm:40s} {v[i] / pw / per_warp_cycles * 100:6.1f} %")
    tot_wait = sum(v[16:24]); tot_work = sum(v[24:32])
    print(f"consumer FULL wait {tot_wait / pw / per_warp_cycles * 100:6.1f} %   work {tot_work / pw / per_warp_cycles * 100:6.1f} %")
    for t in range(8):
        n = v[40 + t] / pw
        if n:
            print(f"  tile {t}: windows/warp {n:8.1f}  wait {v[16 + t] / pw / per_warp_cycles * 100:6.1f} %  "
                  f"work {v[24 + t] / pw / per_warp_cycles * 100:6.1f} %")


if __name__ == "__main__":
    main()
