"""Tiny calls of every kernel for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
cluster-split direct kernel (cfg1-like, fp32 / lut / fp16 / lut_tex), persistent warp-specialised kernel
(split -1), polyphase kernel (split -1, single- and two-word, fused tail, the count guard's redo), tail
kernel, batch call (polyphase with fused tail; fp32 with tail_kernel), the polyphase cluster items of small calls,
trajectory filter (tcgen05 kernel with TMA- and register-fed B, K shares; CUDA-core kernel).  Small sizes:
racecheck tracks every shared-memory access."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402


def run(sc, mode, split=0, M=None):
    beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    nb = P.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
    rcv = sc.pos_rcv if M is None else sc.pos_rcv[:M]
    orv = None if sc.orV_rcv is None else (sc.orV_rcv if M is None else sc.orV_rcv[:M])
    h = P.simulate_rir(sc.room, beta, torch.from_numpy(sc.pos_src).cuda(),
                       torch.from_numpy(np.ascontiguousarray(rcv)).cuda(), nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c,
                       orV_rcv=None if orv is None else torch.from_numpy(np.ascontiguousarray(orv)).cuda(),
                       mic_pattern=sc.pattern, mode=mode, seed=sc.seed, split=split, sync=True)
    assert torch.isfinite(h).all()
    print(f"ok {sc.name} {mode} split={split} M={h.shape[1]}", flush=True)


def main():
    small = W.cfg2(0.3)  # 6x4x3 m, ISM to 75 ms + tail to 0.3 s, one RIR
    for mode in ("fp32", "lut", "fp16", "lut_tex"):
        run(small, mode)                  # cluster-split direct kernel + tail kernel
        run(small, mode, split=-1)        # persistent warp-specialised kernel
    run(small, "poly", split=-1)          # polyphase, fused tail
    run(small, "poly", split=-2)          # polyphase, two-word scheme
    c3 = W.cfg3(8, "diffuse")
    c3.Tdiff, c3.Tmax = 0.05, 0.1
    run(c3, "poly", split=-3)             # polyphase, count guard redo (two words)
    run(c3, "poly")                       # 8 cardioid RIRs: 8 x 1 tile -> direct kernels
    rb = W.cfg5(6)
    rooms, off = [], 0
    for i in range(rb.n):
        beta, _ = P.beta_sabine(rb.room[i], rb.T60[i])
        Tm = min(float(rb.Tmax[i]), 0.25)
        rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i],
                          nb_img=P.t2n(Tm / 4, rb.room[i]), Tdiff=Tm / 4, Tmax=Tm, out_offset=off))
        off += P.nsamples(Tm, rb.fs)
    for mode, split in (("poly", -1), ("fp32", 0)):
        out = torch.empty((off,), device="cuda")
        P.simulate_rir_batch(rooms, rb.fs, out, seed=rb.seed, mode=mode, split=split, sync=True)
        assert torch.isfinite(out).all()
        print(f"ok batch {mode}", flush=True)
    run(small, "poly")                    # lone RIR: cluster items (1024-thread CTAs, L2 slab exchange), fused tail
    run(small, "poly", split=8)           # forced cluster of 8 (512-thread CTAs)
    run(W.cfg4("a"), "poly", M=4)         # 48 kHz cluster items (runtime plane stride)
    sig = torch.randn(777, device="cuda")
    for shape, split in (((3, 2, 301), 0), ((3, 2, 300), 0), ((3, 8, 300), 0), ((3, 8, 300), 3), ((3, 8, 300), -1)):
        # L % 4 != 0: CUDA-core kernel; 2 mics: tensor cores, B through registers; 8 mics: TMA-fed B; 3 K shares
        # (the ordered partial sum); -1: the CUDA-core kernel
        rirs = torch.randn(shape, device="cuda")
        y = P.simulate_trajectory(sig, rirs, sync=True, split=split)
        assert torch.isfinite(y).all()
        print(f"ok trajectory {shape} split={split}", flush=True)


if __name__ == "__main__":
    main()
