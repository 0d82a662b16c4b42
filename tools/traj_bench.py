"""Timing of NEXT row f1 (trajectory filtering) on one B200: device time per gpurir_simulate_trajectory call
(CUDA events, L2 flushed between calls, median).  MACs = n_sig x L x n_mics (each input sample meets every tap
once per microphone); the bound is the FP32 FMA issue rate (148 SMs x 128 lanes x clock).

  python tools/traj_bench.py [--clock-mhz 1965]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_11359_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--clock-mhz", type=float, default=1965.0)
    ap.add_argument("--splits", default="0,-1", help="opts.split values: 0 auto (tcgen05), -1 CUDA cores, k > 0 K split")
    args = ap.parse_args()
    splits = [int(x) for x in args.splits.split(",")]
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    peak = 148 * 128 * args.clock_mhz * 1e6
    g = torch.Generator(device=dev).manual_seed(0)
    for n_sig, n_pts, n_mics, L in [(16000, 100, 32, 11200), (48000, 300, 32, 11200), (160000, 64, 4, 4000),
                                    (16000, 16, 1, 11200)]:
        sig = torch.randn(n_sig, device=dev, generator=g)
        rirs = torch.randn((n_pts, n_mics, L), device=dev, generator=g) * 1e-2
        out = torch.empty((n_mics, n_sig + L - 1), device=dev)
        for split in splits:
            for _ in range(3):
                P.simulate_trajectory(sig, rirs, out=out, split=split)
            ts = []
            for _ in range(7):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                P.simulate_trajectory(sig, rirs, out=out, split=split)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = float(np.median(ts))
            macs = n_sig * L * n_mics
            print(json.dumps(dict(cfg="traj_f1", split=split, kernel="cuda_cores" if split < 0 else "tcgen05",
                                  n_sig=n_sig, points=n_pts, mics=n_mics, L=L, ms=ms, macs=macs,
                                  fma_per_s=macs / ms * 1e3, frac_fp32_fma_peak=macs / ms * 1e3 / peak)), flush=True)


if __name__ == "__main__":
    main()
