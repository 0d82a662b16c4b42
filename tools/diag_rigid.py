"""Diagnose the rigid-cube 48 kHz polyphase error: error location and size for the default poly path, the
two-word scheme (split -2), the direct fp32 kernel, and (if GPURIR_LIB_OLD is set) an older library build."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1810_11359_b200 as P  # noqa: E402

fs, T = 48000.0, 0.3
room = np.array([2.0, 2.0, 2.0], np.float32)
src = np.array([[1.0, 1.0, 1.0]], np.float32)
for rcv_ in ([[1.0, 1.0, 1.5]], [[1.0, 1.0, 1.0 + 2.0 ** -10], [1.0, 1.0, 1.5]]):
    rcv = np.array(rcv_, np.float32)
    nb = oracle.t2n(T, room, 343.0)
    beta = np.full(6, 1.0, np.float32)
    r = oracle.simulate_rir(room, beta, src, rcv, nb, T, T, fs=fs)
    for mode, split in (("poly", -1), ("poly", -2), ("fp32", 0)):
        g = P.simulate_rir(room, beta, torch.from_numpy(src).cuda(), torch.from_numpy(rcv).cuda(), nb, T, T, fs,
                           mode=mode, split=split, sync=True).cpu().numpy().astype(np.float64)
        for i in range(len(rcv)):
            e = np.abs(g[0, i] - r[0, i])
            k = int(e.argmax())
            print(f"M={len(rcv)} rcv{i} {mode} split={split}: err/peak {e.max() / np.abs(r[0, i]).max():.3e} at {k} "
                  f"(gpu {g[0, i, k]:.6e} oracle {r[0, i, k]:.6e}); errs near: "
                  f"{[round(float(v), 9) for v in e[max(0, k - 3):k + 4]]}", flush=True)
