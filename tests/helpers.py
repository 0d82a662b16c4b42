"""Shared test helpers: run one workloads.Scene through the CUDA path and the oracle on identical inputs.

beta and nb_img are derived ONCE with the oracle's helpers and fed to both sides
(no oracle input comes from the CUDA path).
"""
from __future__ import annotations

import numpy as np

TOL = {"fp32": 1e-4, "lut": 5e-3, "fp16": 2e-2, "lut_tex": 5e-3, "poly": 1e-4}  # north_star (lut_tex = LUT, poly = fp32), per RIR, relative to max|h_oracle| (C20)


def derive(oracle, sc):
    beta, clamped = oracle.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    beta = beta.astype(np.float32)
    nb = oracle.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
    return beta, nb


def run_gpu(P, sc, beta, nb, mode="fp32", split=0, rir_index_base=0, pos_rcv=None, orv=None):
    import torch
    src = torch.from_numpy(np.ascontiguousarray(sc.pos_src)).cuda()
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv if pos_rcv is None else pos_rcv)).cuda()
    o = sc.orV_rcv if orv is None else orv
    ov = torch.from_numpy(np.ascontiguousarray(o)).cuda() if o is not None else None
    h = P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=ov,
                       mic_pattern=sc.pattern, mode=mode, seed=sc.seed, rir_index_base=rir_index_base, split=split,
                       sync=True)
    torch.cuda.synchronize()
    return h.cpu().numpy().astype(np.float64)


def run_oracle(oracle, sc, beta, nb, pos_rcv=None, orv=None, rir_index_base=0):
    o = sc.orV_rcv if orv is None else orv
    return oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv if pos_rcv is None else pos_rcv, nb, sc.Tdiff,
                               sc.Tmax, fs=sc.fs, c=sc.c, pattern=sc.pattern, orV_rcv=o, seed=sc.seed,
                               rir_index_base=rir_index_base)


def rel_err(g: np.ndarray, r: np.ndarray) -> np.ndarray:
    """Per-RIR max |g - r| / max |r| (reading C20)."""
    g = g.reshape(-1, g.shape[-1])
    r = r.reshape(-1, r.shape[-1])
    peak = np.max(np.abs(r), axis=1)
    peak = np.where(peak > 0, peak, 1.0)
    return np.max(np.abs(g - r), axis=1) / peak
