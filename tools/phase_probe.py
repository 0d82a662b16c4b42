"""Phase timing of small polyphase calls (diagnostic): run with GPURIR_LIB=build/phase.so (tools/build_variant.sh phase
-DGPURIR_PHASE_TIMING); the kernel prints one PT line per CTA of the last call.  Summarises per-phase spans.

  GPURIR_LIB=build/phase.so python tools/phase_probe.py cfg1 [split] > log; python tools/phase_probe.py --parse log
"""
import os
import sys

import numpy as np


def parse(path):
    rows = [l.split()[1:] for l in open(path) if l.startswith("PT ")]
    a = np.array([[int(x) for x in r] for r in rows], dtype=np.float64)
    if not len(a):
        print("no PT lines")
        return
    # keep the last call: the CTAs whose start lies after the last gap of > 50 us between consecutive starts
    o = np.argsort(a[:, 4])
    st = a[o, 4]
    gaps = np.where(np.diff(st) > 50e3)[0]
    if len(gaps):
        a = a[o[gaps[-1] + 1:]]
    t = a[:, 4:12]
    base = t[:, 0].min()
    t = (t - base) / 1e3  # us
    print(f"{len(a)} CTAs; kernel span {t[:, 7].max():.2f} us (first mark to last end)")
    names = ["start", "setup", "bz", "aggr", "Gsync", "merge/v", "fir", "end"]
    for i, n in enumerate(names):
        print(f"  {n:8s} min {t[:, i].min():7.2f}  median {np.median(t[:, i]):7.2f}  max {t[:, i].max():7.2f}")
    # the CTA that ends last: its phase times
    k = int(np.argmax(t[:, 7]))
    print("last CTA", a[k, :4].astype(int).tolist(), " ".join(f"{x:.2f}" for x in t[k]), "te", int(a[k, 12]))
    for te in sorted(set(a[:, 12].astype(int))):
        s = a[:, 12] == te
        print(f"  tile te={te:6d}: {s.sum():4d} CTAs  aggr done max {t[s, 3].max():7.2f}  end max {t[s, 7].max():7.2f}")
    if a.shape[1] >= 18:  # thread-0 setup sub-steps in SM clocks from entry (1.965 GHz)
        u = (a[:, 14:18] - a[:, 13:14]) / 1965.0
        for i, n in enumerate(["P loaded", "decoded", "geom", "set up"]):
            print(f"  setup {n:9s} min {u[:, i].min():7.2f}  median {np.median(u[:, i]):7.2f}  max {u[:, i].max():7.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "--parse":
        parse(sys.argv[2])
        sys.exit(0)
    import torch
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, ROOT)
    sys.argv = [sys.argv[0], sys.argv[1], "poly", sys.argv[2] if len(sys.argv) > 2 else "0"]
    sys.stdout.flush()
    exec(open(os.path.join(ROOT, "tools", "prof_small.py")).read())
