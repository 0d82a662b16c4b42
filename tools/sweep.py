"""Throughput sweeps on one B200 (GPU box): the paper's #RIR and T60 sweeps (BASELINE.json configs 2-5).

Device time per gpurir_simulate_rir call with CUDA events (inputs resident, L2 flushed between calls),
median of `reps` calls after warm-up.  Prints one JSON object per line and a final summary object.

  python tools/sweep.py [--quick] > profiles/r01_sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1810_11359_b200 as P  # noqa: E402
import workloads as W  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def time_call(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def scene_call(sc, mode="fp32"):
    beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
    nb = P.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
    src = torch.from_numpy(sc.pos_src).to(dev)
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).to(dev)
    orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).to(dev) if sc.orV_rcv is not None else None
    nS = P.nsamples(sc.Tmax, sc.fs)
    out = torch.empty((src.shape[0], rcv.shape[0], nS), dtype=torch.float32, device=dev)

    def fn():
        P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                       mic_pattern=sc.pattern, mode=mode, seed=sc.seed, out=out)
    return fn, nb


def emit(d):
    print(json.dumps(d), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    reps = 3 if args.quick else 5
    rows = []

    # config 1: latency of the single-RIR ISM-only call
    for mode in ("fp32", "lut", "fp16", "lut_tex", "poly"):
        fn, nb = scene_call(W.cfg1(), mode)
        ms = time_call(fn, reps=20, warm=5)
        rows.append(dict(cfg="cfg1", mode=mode, M=1, ms=ms, rirs_per_s=1e3 / ms))
        emit(rows[-1])

    # config 2: T60 sweep, 1 RIR (latency bound at low T60)
    for T60 in W.CFG2_T60:
        fn, nb = scene_call(W.cfg2(T60))
        ms = time_call(fn, reps=10, warm=3)
        rows.append(dict(cfg="cfg2", T60=T60, M=1, ms=ms, rirs_per_s=1e3 / ms,
                         lattice_per_s=float(np.prod(nb.astype(float))) / ms * 1e3))
        emit(rows[-1])

    # config 3: #RIR sweep (diffuse and full ISM), 3 modes
    Ms = [1, 16, 128, 1024, 4096, 16384]
    for variant in ("diffuse", "full"):
        for mode in ("fp32", "lut", "fp16", "lut_tex", "poly"):
            for M in Ms:
                if variant == "full" and M > 4096 and args.quick:
                    continue
                sc = W.cfg3(M, variant)
                fn, nb = scene_call(sc, mode)
                ms = time_call(fn, reps=reps if M < 4096 else 3, warm=2 if M < 4096 else 1)
                rows.append(dict(cfg=f"cfg3_{variant}", mode=mode, M=M, ms=ms, rirs_per_s=M / ms * 1e3,
                                 lattice_per_s=M * float(np.prod(nb.astype(float))) / ms * 1e3))
                emit(rows[-1])

    # config 4: 32-mic array at 48 kHz, three modes
    for variant in ("a", "b"):
        for mode in ("fp32", "lut", "fp16", "lut_tex", "poly"):
            fn, nb = scene_call(W.cfg4(variant), mode)
            ms = time_call(fn, reps=reps, warm=2)
            rows.append(dict(cfg=f"cfg4{variant}", mode=mode, M=32, ms=ms, rirs_per_s=32 / ms * 1e3,
                             lattice_per_s=32 * float(np.prod(nb.astype(float))) / ms * 1e3))
            emit(rows[-1])

    # config 5: independent rooms through the batch API (one GPU)
    n_rooms = 20000 if args.quick else 100000
    rb = W.cfg5(n_rooms)
    t0 = time.time()
    rooms, off = [], 0
    lattice = 0.0
    for i in range(rb.n):
        beta, _ = P.beta_sabine(rb.room[i], rb.T60[i])
        nb = P.t2n(rb.Tdiff[i], rb.room[i])
        lattice += float(np.prod(nb.astype(float)))
        rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i], nb_img=nb,
                          Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], out_offset=off))
        off += P.nsamples(rb.Tmax[i], rb.fs)
    arr = P.room_array(rooms)
    plan_s = time.time() - t0
    out = torch.empty(off, dtype=torch.float32, device=dev)
    for mode in ("fp32", "poly"):
        fn = lambda: P.simulate_rir_batch(arr, rb.fs, out, seed=rb.seed, mode=mode)  # noqa: E731
        ms = time_call(fn, reps=3, warm=1)
        rows.append(dict(cfg="cfg5", mode=mode, M=rb.n, ms=ms, rirs_per_s=rb.n / ms * 1e3,
                         lattice_per_s=lattice / ms * 1e3, samples=off, host_plan_s=plan_s,
                         note="time includes the call's host planning + job-table upload (batch API synchronises)"))
        emit(rows[-1])
    # NEXT row f1: moving source, 1 s at 16 kHz, 100 trajectory points x 32 mics, 0.7 s RIRs (cfg3 length)
    n_sig, n_pts, n_mics, L = 16000, 100, 32, 11200
    sig = torch.randn(n_sig, device=dev)
    rirs = torch.randn((n_pts, n_mics, L), device=dev) * 1e-2
    outb = torch.empty((n_mics, n_sig + L - 1), device=dev)
    ms = time_call(lambda: P.simulate_trajectory(sig, rirs, out=outb), reps=5, warm=2)
    macs = n_sig * L * n_mics
    rows.append(dict(cfg="traj_f1", n_sig=n_sig, points=n_pts, mics=n_mics, L=L, ms=ms, macs=macs,
                     fma_per_s=macs / ms * 1e3, frac_fp32_fma_peak=macs / ms * 1e3 / (148 * 128 * 1.965e9)))
    emit(rows[-1])
    emit({"summary": True, "device": torch.cuda.get_device_name(0), "rows": len(rows)})


if __name__ == "__main__":
    main()
