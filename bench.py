#!/usr/bin/env python
"""bench.py — RIR-synthesis throughput of the B200 ISM engine (contract: see DESIGN.md §Measurement).

Workload (BASELINE.json config 3, the paper's #RIR sweep room): 3x4x2.5 m, T60 = 0.7 s
(beta = -0.9397, Sabine), source (1.5, 1.0, 1.2), M = 16384 cardioid receivers per GPU uniform in the
room (seed 3) with random orientations, fs = 16 kHz, ISM to Tdiff = 0.175 s + diffuse tail to 0.7 s,
polyphase mode by default (fp32 arithmetic and tolerance, reading R11; --mode fp32 selects the
direct-tap kernel, which the line also reports as `direct_fp32`).  One step = one gpurir_simulate_rir call
over the rank's 16384 receivers (ISM kernel + tail kernel).  Weak scaling: rank r owns receivers [16384 r, 16384 (r+1)) of the N*16384-receiver workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--mode poly|fp32|lut|fp16|lut_tex]
                  [--workload ism|trajectory|cfg5] [--no-sweep] [--no-cpu-baseline]

The default line also carries `sweep`: the points behind the metric's axes (the cfg3 #RIR sweep 1-16384 in
both variants, the cfg2 T60 sweep, cfg4 (a/b) in every mode, the cfg1 single-RIR latency, config 5's 100 000
rooms in one batch call, the trajectory job), device-timed in the same run, and `parity`: the timed step's
output checked against the oracle RIRs that cpu_baseline computes.

--workload cfg5 (BASELINE.json config 5, dataset generation): 100 000 random rooms LPT-sharded over the ranks
(SURVEY §8(e)), one gpurir_simulate_rir_batch call per rank per step, no collective; strong scaling.

--impl reference times the CPU oracle (oracle/, test infrastructure) on the host cores: the paper's
comparison arm for this tier.

--workload trajectory (NEXT row f1, workloads.traj1): one step = one moving-source job: the 100 x 32
RIRs of the trajectory (ISM + tail kernels) and the filtering of 1 s of signal through them
(traj_kernel); value = trajectories/s.  Weak scaling: every rank runs its own trajectory.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

M_PER_GPU = 16384
METRIC = "RIRs/s and image contributions/s vs T60 and #RIRs at 1/2/4/8 B200"
TRAJ_METRIC = "moving-source trajectories/s (RIR synthesis + trajectory filtering, NEXT row f1)"
ISSUE_SLOTS_PER_TAP = 13  # algorithmic FP32-pipe issue slots per in-window tap (direct kernels)
# Polyphase kernel (mode poly, reading R11 / §5.5): algorithmic lane-ops per in-range image (Eqs. 1-4:
# 13, the 8 Chebyshev channel values: 14, their 8 deposits) and per output sample (the FIR: 2H taps x 8 MACs)
POLY_OPS_PER_IMAGE = 35


def workload_name(mode="fp32"):
    """The workload (BASELINE.json config 3, diffuse variant); the evaluation mode is a separate config key."""
    return f"cfg3_diffuse_M{M_PER_GPU}perGPU_T60_0.7_fs16k_cardioid"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def count_taps(room, src, rcv, nb, nISM, fs, c, H, images=False):
    """Algorithmic work: in-window (image, sample) pairs for samples [0, nISM) (Eqs. 5-6 support); with
    images=True also the number of images with at least one such tap."""
    lo = [-(int(n) // 2) for n in nb]
    hi = [(int(n) + 1) // 2 for n in nb]
    ax = []
    for a in range(3):
        n = np.arange(lo[a], hi[a])
        q = np.where(n % 2 == 0, n * room[a] + src[a], (n + 1) * room[a] - src[a]) - rcv[a]
        ax.append(q * q)
    d2 = ax[0][None, None, :] + ax[1][None, :, None] + ax[2][:, None, None]
    x = np.sqrt(d2).ravel() * fs / c
    k0 = np.maximum(np.floor(x - H) + 1, 0)
    k1 = np.minimum(np.ceil(x + H) - 1, nISM - 1)
    n = np.maximum(k1 - k0 + 1, 0)
    return (float(n.sum()), float((n > 0).sum())) if images else float(n.sum())


class RawEvent:
    """A cudaEvent_t created through the CUDA runtime torch already loaded (the library records it)."""
    _rt = None

    @classmethod
    def rt(cls):
        if cls._rt is None:
            import ctypes
            cls._rt = ctypes.CDLL("libcudart.so.12")
        return cls._rt

    def __init__(self):
        import ctypes
        self.h = ctypes.c_void_p()
        assert self.rt().cudaEventCreate(ctypes.byref(self.h)) == 0
        self.cuda_event = self.h.value

    def elapsed_ms(self, end) -> float:
        import ctypes
        ms = ctypes.c_float()
        assert self.rt().cudaEventElapsedTime(ctypes.byref(ms), self.h, end.h) == 0
        return float(ms.value)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
            # nvidia-smi's NVML start-up can take longer than a fixed sleep and stalls the driver meanwhile (a cfg5
            # step that plans on the host saw its first timed call take 117 ms instead of 40): wait for its first
            # sample before the timed region starts
            t_end = time.time() + 5.0
            while time.time() < t_end and os.path.getsize(self.path) == 0:
                time.sleep(0.02)
            time.sleep(0.1)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def lib_record(P, allow_override):
    """Which libgpurir.so this run timed: path, sha256 prefix, version.  A GPURIR_LIB override (A/B variant
    builds, tools/build_variant.sh) or a variant build is refused unless --ab-lib is given."""
    import hashlib
    path = os.path.abspath(P.LIB_PATH)
    with open(path, "rb") as f:
        sha = hashlib.sha256(f.read()).hexdigest()[:16]
    ver = P.version()
    default = os.path.abspath(os.path.join(ROOT, "paper_1810_11359_b200", "libgpurir.so"))
    overridden = path != default or "variant" in ver
    if overridden and not allow_override:
        raise SystemExit(f"bench.py: refusing to time {path} ({ver}): not the in-tree build (pass --ab-lib for A/B)")
    return {"path": os.path.relpath(path, ROOT), "sha256_16": sha, "version": ver, "override": overridden}


# ----------------------------------------------------------------------------- oracle arms

def oracle_rate(sc, beta, nb, n_rir, base_index=0, nthreads=0):
    """Time the CPU oracle (as it stands) on the first n_rir receivers of the workload; (RIRs/s, s, RIRs)."""
    import oracle
    t = time.perf_counter()
    h = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[:n_rir], nb, sc.Tdiff, sc.Tmax, fs=sc.fs, c=sc.c,
                            pattern=sc.pattern, orV_rcv=sc.orV_rcv[:n_rir], seed=sc.seed, rir_index_base=base_index,
                            nthreads=nthreads)
    dt = time.perf_counter() - t
    return n_rir / dt, dt, h


def cpu_baseline(sc, gpu_rows=None, budget_s=15.0, kernel=None):
    """The oracle (oracle/, -O3 -march=native built on this host) on the host cores, on a bounded sample of the
    workload: all cores, then one thread.  With gpu_rows (the timed step's output rows [M, nS] as a host array)
    it also returns the step's parity against the oracle RIRs it just computed (reading C20)."""
    import oracle
    oracle.use_native()
    beta, _ = oracle.beta_sabine(sc.room, sc.T60)
    beta = beta.astype(np.float32)
    nb = oracle.t2n(sc.Tdiff, sc.room, sc.c)
    cores = oracle.max_threads()
    n0 = max(cores, 8)
    r0, dt0, _ = oracle_rate(sc, beta, nb, n0, nthreads=cores)
    n = int(min(len(sc.pos_rcv), max(n0, round(r0 * budget_s / cores) * cores)))
    if gpu_rows is not None:
        n = min(n, len(gpu_rows))
    r, dt, h = oracle_rate(sc, beta, nb, n, nthreads=cores)
    n1 = max(1, int(round(r / cores * 3.0)))  # about 3 s on one thread
    r1, dt1, _ = oracle_rate(sc, beta, nb, n1, nthreads=1)
    out = {"value": r, "unit": "RIRs/s", "cores": cores, "kind": "oracle",
           "sample": f"first {n} of the {len(sc.pos_rcv)} receivers of the workload ({dt:.1f} s, OpenMP over RIRs, "
                     f"fp64 C oracle, {oracle.build_flags()})",
           "single_thread": {"value": r1, "unit": "RIRs/s", "sample": f"first {n1} receivers, 1 thread ({dt1:.1f} s)"},
           "cpu_model": oracle.cpu_model(), "build": oracle.build_flags()}
    parity = None
    if gpu_rows is not None:
        g = gpu_rows[:n].astype(np.float64)
        r_ = h.reshape(n, -1)
        peak = np.abs(r_).max(axis=1)
        err = np.abs(g - r_).max(axis=1) / np.where(peak > 0, peak, 1.0)
        parity = {"max_err_over_peak": float(err.max()), "median_err_over_peak": float(np.median(err)), "n": n,
                  "tol": 1e-4, "ok": bool(err.max() <= 1e-4),
                  "what": f"the timed step's RIRs 0..{n - 1} (all samples, tail included) vs the oracle's (C20)",
                  "kernel": kernel}
    return out, parity


def traj_oracle_times(sc, sig, n_rir, n_mic):
    """Oracle seconds for n_rir of the trajectory's RIRs and for filtering n_mic microphones (random RIR
    values of the right shape: the filter's cost does not depend on them)."""
    import oracle
    beta, _ = oracle.beta_sabine(sc.room, sc.T60)
    beta = beta.astype(np.float32)
    nb = oracle.t2n(sc.Tdiff, sc.room, sc.c)
    L = oracle.nsamples(sc.Tmax, sc.fs)
    n_src = max(1, n_rir // len(sc.pos_rcv))
    t = time.perf_counter()
    oracle.simulate_rir(sc.room, beta, sc.pos_src[:n_src], sc.pos_rcv[:max(1, n_rir // n_src)], nb, sc.Tdiff, sc.Tmax,
                        fs=sc.fs, c=sc.c, pattern=sc.pattern, seed=sc.seed)
    t_rir = time.perf_counter() - t
    n_rir = n_src * max(1, n_rir // n_src)
    rirs = np.random.default_rng(0).standard_normal((len(sc.pos_src), n_mic, L)) * 1e-2
    t = time.perf_counter()
    oracle.simulate_trajectory(sig, rirs)
    t_f = time.perf_counter() - t
    per_traj = t_rir * (len(sc.pos_src) * len(sc.pos_rcv)) / n_rir + t_f * len(sc.pos_rcv) / n_mic
    return per_traj, n_rir, n_mic, t_rir + t_f


def traj_oracle_sample(sc, sig, cores, budget_s):
    """Sample sizes (RIRs, microphones) so that one oracle pass over them takes about budget_s."""
    per_traj, _, _, _ = traj_oracle_times(sc, sig, cores, 2)
    f = min(1.0, budget_s / per_traj)
    nr = int(min(sc.M, max(cores, round(f * sc.M / cores) * cores)))
    nm = int(min(len(sc.pos_rcv), max(2, round(f * len(sc.pos_rcv)))))
    return nr, nm


def run_reference_trajectory(args):
    import oracle
    sc = W.traj1()
    sig = W.traj_signal(sc.meta["n_sig"])
    cores = oracle.max_threads()
    nr, nm = traj_oracle_sample(sc, sig, cores, 150.0 / max(1, args.steps + args.warmup))
    times = []
    for i in range(args.warmup + args.steps):
        per_traj, nr, nm, _ = traj_oracle_times(sc, sig, nr, nm)
        if i >= args.warmup:
            times.append(per_traj)
    ms = 1000.0 * float(np.mean(times))
    value = 1000.0 / ms
    line = {"impl": "reference", "metric": TRAJ_METRIC, "value": value, "unit": "trajectories/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": sc.name, "reference_arm": "CPU oracle (oracle/oracle.c); each step times "
                       f"{nr} of the {sc.M} RIRs and the filtering of {nm} of {len(sc.pos_rcv)} microphones and "
                       "scales both to one trajectory"},
            "cpu_baseline": {"value": value, "unit": "trajectories/s", "cores": cores, "kind": "oracle",
                             "sample": f"{nr} RIRs + {nm} microphones filtered per step"},
            "e2e": {"value": value, "unit": "trajectories/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cfg3_config(mode, sc, beta, nb, nS, nISM):
    """The bench line's config for the cfg3 workload (both arms print the same dict)."""
    return {"workload": workload_name(mode), "M_per_gpu": M_PER_GPU, "room": [3, 4, 2.5], "T60": 0.7,
            "beta": float(beta[0]), "nb_img": [int(v) for v in nb], "fs": sc.fs, "Tdiff": sc.Tdiff,
            "Tmax": sc.Tmax, "pattern": "cardioid", "mode": mode, "nSamples": nS, "nISM": nISM,
            "l2": "256 MB buffer written between timed steps (L2 126 MB); step output 734 MB"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload == "trajectory":
        run_reference_trajectory(args)
        return
    import oracle
    oracle.use_native()
    sc = W.cfg3(M_PER_GPU, "diffuse")
    beta, _ = oracle.beta_sabine(sc.room, sc.T60)
    beta = beta.astype(np.float32)
    nb = oracle.t2n(sc.Tdiff, sc.room, sc.c)
    cores = oracle.max_threads()
    per_step = max(cores, 16)
    r0, dt0, _ = oracle_rate(sc, beta, nb, per_step, nthreads=cores)
    # size each step so warmup + steps finish in ~2-3 minutes
    target = 150.0 / max(1, args.steps + args.warmup)
    per_step = int(min(M_PER_GPU, max(cores, round(r0 * target / cores) * cores)))
    times = []
    for i in range(args.warmup + args.steps):
        off = (i * per_step) % (M_PER_GPU - per_step + 1)
        t = time.perf_counter()
        oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[off:off + per_step], nb, sc.Tdiff, sc.Tmax,
                            fs=sc.fs, c=sc.c, pattern=sc.pattern, orV_rcv=sc.orV_rcv[off:off + per_step],
                            seed=sc.seed, rir_index_base=off)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = per_step / (ms / 1000.0)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "RIRs/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(cfg3_config(args.mode, sc, beta, nb, oracle.nsamples(sc.Tmax, sc.fs),
                                       oracle.nsamples(sc.Tdiff, sc.fs)),
                           reference_arm=f"CPU oracle (oracle/oracle.c), each step {per_step} receivers of the workload"),
            "cpu_baseline": {"value": value, "unit": "RIRs/s", "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} RIRs per step x {args.steps} steps",
                             "build": oracle.build_flags(), "cpu_model": oracle.cpu_model()},
            "e2e": {"value": value, "unit": "RIRs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--mode", default="poly", choices=["fp32", "lut", "fp16", "lut_tex", "poly"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the N>1 host path with several ranks on one GPU")
    ap.add_argument("--workload", default="ism", choices=["ism", "trajectory", "cfg5"])
    ap.add_argument("--no-sweep", action="store_true", help="skip the `sweep` points (configs 1-5)")
    ap.add_argument("--ab-lib", action="store_true", help="allow timing a GPURIR_LIB override / variant build")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    import torch
    import paper_1810_11359_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    local_dev = local % torch.cuda.device_count()
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    lib = lib_record(P, args.ab_lib)
    if args.workload == "trajectory":
        run_trajectory(args, P, torch, dev, rank, world, dist, local_dev, lib)
        return
    if args.workload == "cfg5":
        run_cfg5(args, P, torch, dev, rank, world, dist, local_dev, lib)
        return

    # ---- workload (weak scaling: this rank's 16384 receivers of the N*16384 workload) ----
    sc = W.cfg3(M_PER_GPU * world, "diffuse")
    sl = slice(rank * M_PER_GPU, (rank + 1) * M_PER_GPU)
    beta, _ = P.beta_sabine(sc.room, sc.T60)           # library helpers on the product path
    nb = P.t2n(sc.Tdiff, sc.room, sc.c)
    nS, nISM = P.nsamples(sc.Tmax, sc.fs), P.nsamples(sc.Tdiff, sc.fs)
    src = torch.from_numpy(sc.pos_src).to(dev)
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv[sl])).to(dev)
    orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv[sl])).to(dev)
    out = torch.empty((1, M_PER_GPU, nS), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    base = rank * M_PER_GPU

    def step(ev=None, ev_tail=None):
        P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                       mic_pattern=sc.pattern, mode=args.mode, seed=sc.seed, rir_index_base=base, out=out,
                       stream=stream, ev_ism=ev, ev_tail=ev_tail)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    n_ev = args.steps
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    ism_s = [RawEvent() for _ in range(n_ev)]
    ism_e = [RawEvent() for _ in range(n_ev)]
    tail_s = [RawEvent() for _ in range(n_ev)]
    tail_e = [RawEvent() for _ in range(n_ev)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_dev) as clk:
        for i in range(args.steps):
            flush.zero_()                       # L2 flushed between timed steps (outside the events)
            ev_s[i].record(stream)
            step((ism_s[i], ism_e[i]), (tail_s[i], tail_e[i]))
            ev_e[i].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev_s, ev_e)]
    ism_ms = [a.elapsed_ms(b) for a, b in zip(ism_s, ism_e)]
    tail_ms = [a.elapsed_ms(b) for a, b in zip(tail_s, tail_e)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    ms_per_step = total_ms / args.steps
    value = world * M_PER_GPU * args.steps / (total_ms / 1000.0)

    # ---- end to end through the C ABI with HOST buffers: gpurir_simulate_rir_host ----
    # A dataset-generation loop: every step is one call that takes the positions from pinned host memory and
    # returns the full RIR tensor in pinned host memory (its H2D and D2H copies inside the call, the D2H of
    # each 2048-RIR chunk overlapping the next chunk's kernels).  CUDA events on the call's stream bracket
    # the K synchronous calls.
    e2e_steps = max(2, args.e2e_steps)
    h_src = torch.from_numpy(sc.pos_src).pin_memory()
    h_rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv[sl])).pin_memory()
    h_orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv[sl])).pin_memory()
    h_out = [torch.empty((1, M_PER_GPU, nS), dtype=torch.float32).pin_memory() for _ in range(2)]
    # one untimed call first: it sizes the library's per-device scratch and creates its copy stream
    P.simulate_rir_host(sc.room, beta, h_src, h_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=h_orv,
                        mic_pattern=sc.pattern, mode=args.mode, seed=sc.seed, rir_index_base=base,
                        out=h_out[1], stream=stream)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_steps):
        P.simulate_rir_host(sc.room, beta, h_src, h_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=h_orv,
                            mic_pattern=sc.pattern, mode=args.mode, seed=sc.seed, rir_index_base=base,
                            out=h_out[i % 2], stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64,
                          device=dev if args.dist_backend == "nccl" else "cpu")
    if dist:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * M_PER_GPU * e2e_steps / (float(e2e_ms.item()) / 1000.0)
    h2d = (h_src.numel() + h_rcv.numel() + h_orv.numel()) * 4
    d2h = h_out[0].numel() * 4
    # the host copy of the last step equals the device-timed result (same inputs, deterministic kernels)
    assert torch.equal(h_out[(e2e_steps - 1) % 2][0, :4].to(dev), out[0, :4])

    # the same loop through the device API with torch copies, pipelined ACROSS steps (two device output
    # buffers, D2H of step i on a copy stream while step i+1 computes): context for the host call's number
    d_out = [out, torch.empty_like(out)]
    cs, xs = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    cs.wait_event(p0)
    xs.wait_event(p0)
    copied = []
    for i in range(e2e_steps):
        with torch.cuda.stream(cs):
            if i >= 2:
                cs.wait_event(copied[i - 2])  # d_out[i % 2] is free once step i-2's D2H is done
            d_src = h_src.to(dev, non_blocking=True)
            d_rcv = h_rcv.to(dev, non_blocking=True)
            d_orv = h_orv.to(dev, non_blocking=True)
            P.simulate_rir(sc.room, beta, d_src, d_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=d_orv,
                           mic_pattern=sc.pattern, mode=args.mode, seed=sc.seed, rir_index_base=base,
                           out=d_out[i % 2], stream=cs)
            done = torch.cuda.Event()
            done.record(cs)
        xs.wait_event(done)
        with torch.cuda.stream(xs):
            h_out[i % 2].copy_(d_out[i % 2], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(xs)
            copied.append(ev)
    stream.wait_event(copied[-1])
    p1.record(stream)
    torch.cuda.synchronize()
    pipe_ms = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64,
                           device=dev if args.dist_backend == "nccl" else "cpu")
    if dist:
        dist.all_reduce(pipe_ms, op=dist.ReduceOp.MAX)
    e2e_pipe_value = world * M_PER_GPU * e2e_steps / (float(pipe_ms.item()) / 1000.0)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (the ISM accumulation kernel) ----
    sample = np.linspace(0, M_PER_GPU - 1, 256).astype(int)
    H = 4e-3 * sc.fs / 2
    r64 = sc.pos_rcv[sl].astype(np.float64)
    ti_sample = [count_taps(sc.room.astype(np.float64), sc.pos_src[0].astype(np.float64), r64[m], nb, nISM,
                            sc.fs, sc.c, H, images=True) for m in sample]
    taps_per_rir = float(np.mean([t for t, _ in ti_sample]))
    imgs_per_rir = float(np.mean([i for _, i in ti_sample]))
    taps_launch = taps_per_rir * M_PER_GPU
    imgs_launch = imgs_per_rir * M_PER_GPU
    ism_avg_s = float(np.mean(ism_ms)) / 1000.0
    pk, pk_kind = peaks()
    f_clk = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    issue_peak = 148 * 128 * f_clk  # FP32 lane issue slots / s (B200_PROFILING.md unit counts)
    fir = P.poly_fir_table(4e-3, sc.fs)  # the FIR the kernel runs (reading R13): 4 ntaps + 4 nn MACs per output
    fir_macs = 4 * fir["far"].shape[1] + 4 * fir["nn"]
    poly_ops = imgs_launch * POLY_OPS_PER_IMAGE + M_PER_GPU * nISM * fir_macs
    if args.mode == "poly":
        achieved = poly_ops / ism_avg_s
        basis = (f"{POLY_OPS_PER_IMAGE} lane-ops per in-range image x {imgs_launch:.4g} images + {fir_macs} MACs per "
                 f"output sample (rotated low-rank FIR, R13: 4 channels x {fir['far'].shape[1]} taps + 4 x {fir['nn']}) "
                 f"x {M_PER_GPU * nISM} samples per launch (exact image count on 256 sampled receivers); peak = 148 SM x "
                 f"128 lanes x {f_clk / 1e6:.0f} MHz ({pk_kind} sm_max_mhz); the kernel's time includes the fused "
                 f"diffuse tail, not counted as work")
        kname = "ism_poly_kernel"
    else:
        achieved = taps_launch * ISSUE_SLOTS_PER_TAP / ism_avg_s
        basis = (f"{ISSUE_SLOTS_PER_TAP} issue slots per in-window tap (SURVEY §8(d)) x {taps_launch:.4g} taps per "
                 f"launch (exact count on 256 sampled receivers x {M_PER_GPU}); peak = 148 SM x 128 lanes x "
                 f"{f_clk / 1e6:.0f} MHz ({pk_kind} sm_max_mhz)")
        kname = "ism_ws_kernel<0>" if args.mode == "fp32" else f"ism_ws_kernel ({args.mode})"
    lattice = float(np.prod(nb.astype(np.float64)))
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ism_profile.json")) as f:
            prof = json.load(f)
    except Exception:
        pass
    traffic = (prof["dram_read_bytes"] + prof["dram_write_bytes"]) if prof else None
    tail_bytes = M_PER_GPU * (nS - nISM) * 4
    # polyphase mode writes the diffuse tail inside the ISM kernel (fs <= 102.4 kHz: the 10 ms envelope
    # window fits the last 1024-sample tile); the tail events then bracket nothing
    fused_tail = args.mode == "poly" and round(0.010 * sc.fs) <= 1024  # GPURIR_FUSE_MIN_PER_SM = 0 (abi.cu)
    tail_avg_s = max(float(np.mean(tail_ms)), 1e-9) / 1000.0
    hbm_peak = float(pk.get("hbm_gbs", 6650.0))

    # the polyphase kernel's binding resource is the shared-memory pipe: its roofline counts
    # shared-memory wavefronts per launch (one per SM per clock), the bank-conflict-free count as the
    # algorithmic figure and the measured one (conflict replays included) as the traffic, both from the ncu
    # capture of this step's launch (profiles/r02_ism_profile.json), over the live kernel time
    wf_peak = 148 * f_clk
    if args.mode == "poly" and prof.get("smem_wavefronts"):
        roof_main = {"bound": "smem", "achieved": prof["smem_wavefronts_ideal"] / ism_avg_s / 1e9,
                     "peak": wf_peak / 1e9, "unit": "G shared-memory wavefronts/s",
                     "frac": prof["smem_wavefronts_ideal"] / ism_avg_s / wf_peak,
                     "traffic": prof["smem_wavefronts"], "traffic_unit": "wavefronts per launch (measured)",
                     "frac_measured": prof["smem_wavefronts"] / ism_avg_s / wf_peak,
                     "kernel": kname, "dram_traffic": traffic,
                     "basis": f"bank-conflict-free wavefronts per launch {prof['smem_wavefronts_ideal']:.4g} "
                              f"(measured {prof['smem_wavefronts']:.4g}, {prof['smem_bank_conflicts']:.3g} of them "
                              f"conflict replays; ncu, profiles/r02_ism_profile.json) / live ism_ms; peak = 148 SM x 1 "
                              f"wavefront/clk x {f_clk / 1e6:.0f} MHz ({pk_kind} sm_max_mhz)"}
    else:
        roof_main = {"bound": "alu", "achieved": achieved / 1e12, "peak": issue_peak / 1e12,
                     "unit": "T FP32-lane-issue-slots/s", "frac": achieved / issue_peak, "traffic": traffic,
                     "kernel": kname, "basis": basis}
    line = {
        "metric": METRIC, "value": value, "unit": "RIRs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.mode != "fp16" else "f16x2-taps/f32-acc", "data": "synthetic",
        "config": cfg3_config(args.mode, sc, beta, nb, nS, nISM),
        "image_contributions_per_s": value * lattice,
        "taps_per_s": world * taps_launch / ism_avg_s if world == 1 else None,
        "ism_ms": float(np.mean(ism_ms)),
        "roofline": roof_main,
        "roofline_alu": {"bound": "alu", "achieved": achieved / 1e12, "peak": issue_peak / 1e12,
                         "unit": "T FP32-lane-issue-slots/s", "frac": achieved / issue_peak, "traffic": traffic,
                         "traffic_note": "DRAM bytes per launch from profiles/r02_ism_profile.json (ncu --set full)",
                         "kernel": kname, "basis": basis},
        "tail_kernel": ({"fused_into": "ism_poly_kernel", "bytes": tail_bytes,
                         "note": "the CTA that finishes a RIR's last (end-aligned) ISM tile writes its diffuse tail; "
                                 "its time is inside ism_ms"} if fused_tail else
                        {"ms": float(np.mean(tail_ms)), "bytes": tail_bytes, "GB_per_s": tail_bytes / tail_avg_s / 1e9,
                         "frac_of_hbm": tail_bytes / tail_avg_s / 1e9 / hbm_peak, "bound": "hbm (write)",
                         "peak_GB_per_s": hbm_peak}),
        "e2e": {"value": e2e_value, "unit": "RIRs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "call": "gpurir_simulate_rir_host (pinned host buffers; D2H of each 2048-RIR "
                "chunk overlaps the next chunk's kernels)",
                "stream_pipelined": {"value": e2e_pipe_value, "unit": "RIRs/s", "note": "device API + torch copies, "
                                     "D2H of step i overlapping the kernels of step i+1 (context)"}},
        "gpu_launches": (1 if fused_tail else 2) * args.steps,
        "clocks": clk.summary(),
        "paper_context": "gpuRIR V100 fp32, 1024 RIRs, T60 0.7 s diffuse: 195.69 ms = 5,233 RIRs/s (P:362); "
                         "different fs/positions/pattern, context only",
    }
    # the timed step's RIRs for the parity leg, read before the direct-kernel A/B below reuses `out`
    rows = out[0, :8192].cpu().numpy() if not args.no_cpu_baseline and world == 1 else None
    if args.mode == "poly":  # the direct-tap fp32 kernel on the same step, for the A/B (not part of `value`)
        line["direct_fp32"] = direct_ab(P, torch, sc, beta, nb, src, rcv, orv, base, out, flush, stream,
                                        taps_launch, issue_peak)
    line["lib"] = lib
    if rows is not None:
        line["cpu_baseline"], line["parity"] = cpu_baseline(W.cfg3(M_PER_GPU, "diffuse"), gpu_rows=rows, kernel=kname)
    if not args.no_sweep and world == 1:
        line["sweep"] = sweep(P, torch, dev, flush)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _time_calls(torch, fn, flush, reps=5, warm=2, events=None):
    """Median device ms of fn() over reps calls (CUDA events on the current stream, L2 flushed between calls
    outside the events).  With events=(start, end) RawEvent pairs from fn, those bracket the device work."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ev = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_ms(ev[1]) if isinstance(ev, tuple) else a.elapsed_time(b))
    return float(np.median(ts))


def _latency_us(torch, fn, n=50):
    """Back-to-back calls (no flush): device µs per call, the small-call latency of configs 1, 2, 4."""
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000.0 / n


def _graph_latency_us(torch, fn, n=50, calls=1):
    """The same call captured into a CUDA graph (`calls` times back to back) and replayed: device µs per call without
    the Python / ctypes / launch overhead of an eager call (the library is stream-ordered and capturable).  A graph
    replay costs a whole number of ~2.05 µs steps (tools/replay_quantum.py: any kernel, cluster or not), so one call
    per graph rounds the kernel up; with several calls per graph only the kernels and their gaps remain."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(calls):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000.0 / (n * calls)


def sweep(P, torch, dev, flush):
    """The points behind the metric's axes (BASELINE.json configs 1-5: #RIRs and T60), device-timed in this run:
    median ms per call, RIRs/s and lattice image contributions/s (the paper's work unit)."""
    rows = []

    def scene(sc, mode):
        beta, _ = P.beta_sabine(sc.room, sc.T60, clamp=sc.clamp)
        nb = P.t2n(sc.nb_time if sc.nb_time is not None else max(sc.Tdiff, 1e-6), sc.room, sc.c)
        src = torch.from_numpy(sc.pos_src).to(dev)
        rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).to(dev)
        orv = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).to(dev) if sc.orV_rcv is not None else None
        out = torch.empty((src.shape[0], rcv.shape[0], P.nsamples(sc.Tmax, sc.fs)), dtype=torch.float32, device=dev)

        def fn():
            P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                           mic_pattern=sc.pattern, mode=mode, seed=sc.seed, out=out)
        return fn, float(np.prod(nb.astype(np.float64))), src.shape[0] * rcv.shape[0]

    def point(cfg, sc, mode, reps=5, warm=2, **kw):
        fn, lat, M = scene(sc, mode)
        ms = _time_calls(torch, fn, flush, reps, warm)
        rows.append(dict(cfg=cfg, mode=mode, M=M, ms=ms, rirs_per_s=M / ms * 1e3, lattice_per_s=M * lat / ms * 1e3, **kw))
        return fn

    t0 = time.time()
    for mode in ("poly", "fp32", "lut", "fp16", "lut_tex"):  # config 1: one RIR, ISM only — latency
        fn = point("cfg1", W.cfg1(), mode, reps=10, warm=3)
        rows[-1]["us_per_call_back_to_back"] = _latency_us(torch, fn)
        rows[-1]["us_per_call_graph_replay"] = _graph_latency_us(torch, fn)
        if mode == "poly":
            rows[-1]["us_per_call_graph_10_calls"] = _graph_latency_us(torch, fn, 10, calls=10)
    for T60 in W.CFG2_T60:  # config 2: T60 sweep, one RIR, ISM + tail
        fn = point("cfg2", W.cfg2(T60), "poly", reps=7, warm=3, T60=T60)
        rows[-1]["us_per_call_back_to_back"] = _latency_us(torch, fn, 20)
        rows[-1]["us_per_call_graph_replay"] = _graph_latency_us(torch, fn, 20)
        rows[-1]["us_per_call_graph_10_calls"] = _graph_latency_us(torch, fn, 5, calls=10)
    for M in (1, 4, 16, 64, 256, 1024, 4096, 16384):  # config 3 (i): #RIR sweep, diffuse
        point("cfg3_diffuse", W.cfg3(M, "diffuse"), "poly", reps=5 if M < 4096 else 3)
    for mode in ("fp32", "lut", "fp16", "lut_tex"):
        point("cfg3_diffuse", W.cfg3(4096, "diffuse"), mode, reps=3, warm=1)
    for M in (1, 16, 128, 1024):  # config 3 (ii): #RIR sweep, full ISM to 0.7 s
        point("cfg3_full", W.cfg3(M, "full"), "poly", reps=3, warm=1)
    point("cfg3_full", W.cfg3(128, "full"), "fp32", reps=3, warm=1)
    for variant in ("a", "b"):  # config 4: 32-mic array at 48 kHz, every mode
        for mode in ("poly", "fp32", "lut", "fp16", "lut_tex"):
            fn = point(f"cfg4{variant}", W.cfg4(variant), mode, reps=5, warm=2)
            if mode == "poly":
                rows[-1]["us_per_call_graph_replay"] = _graph_latency_us(torch, fn, 20)
    # config 5: 100 000 rooms in one batch call (device time between the call's first and last kernel events;
    # the host planning of the call is reported beside it)
    rb = W.cfg5(100_000)
    th = time.time()
    rooms, off, lattice = [], 0, 0.0
    for i in range(rb.n):
        beta, _ = P.beta_sabine(rb.room[i], rb.T60[i])
        nb = P.t2n(rb.Tdiff[i], rb.room[i])
        lattice += float(np.prod(nb.astype(np.float64)))
        rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i], nb_img=nb,
                          Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], out_offset=off))
        off += P.nsamples(rb.Tmax[i], rb.fs)
    arr = P.room_array(rooms)
    build_s = time.time() - th
    outb = torch.empty(off, dtype=torch.float32, device=dev)
    for mode in ("poly", "fp32"):
        def fn5(mode=mode):
            e = (RawEvent(), RawEvent()), (RawEvent(), RawEvent())
            P.simulate_rir_batch(arr, rb.fs, outb, seed=rb.seed, mode=mode, ev_ism=e[0], ev_tail=e[1])
            return e[0][0], e[1][1]
        tc = time.time()
        ms = _time_calls(torch, fn5, flush, reps=3, warm=1, events=True)
        call_s = (time.time() - tc) / 4
        rows.append(dict(cfg="cfg5", mode=mode, M=rb.n, ms=ms, rirs_per_s=rb.n / ms * 1e3,
                         lattice_per_s=lattice / ms * 1e3, samples=off, host_call_ms=call_s * 1e3,
                         note="device time from the ISM kernel's start event to the tail's end event; the call's "
                              "host planning + staging (host_call_ms) precedes it"))
    del outb
    # NEXT row f1: the trajectory filter alone, 1 s at 16 kHz, 100 points x 32 mics, 0.7 s RIRs
    n_sig, n_pts, n_mics, L = 16000, 100, 32, 11200
    g = torch.Generator(device=dev).manual_seed(11)
    sig = torch.randn(n_sig, device=dev, generator=g)
    rirs = torch.randn((n_pts, n_mics, L), device=dev, generator=g) * 1e-2
    outt = torch.empty((n_mics, n_sig + L - 1), device=dev)
    ms = _time_calls(torch, lambda: P.simulate_trajectory(sig, rirs, out=outt), flush, reps=5, warm=2)
    ms_fma = _time_calls(torch, lambda: P.simulate_trajectory(sig, rirs, out=outt, split=-1), flush, reps=5, warm=2)
    pk, pk_kind = peaks()
    rows.append(dict(cfg="traj_f1", kernel="traj_tc_kernel (tcgen05)", n_sig=n_sig, points=n_pts, mics=n_mics, L=L,
                     ms=ms, macs_per_s=n_sig * L * n_mics / ms * 1e3,
                     roofline=traj_roofline(n_sig, n_pts, n_mics, L, ms, pk, pk_kind),
                     cuda_core_kernel_ms=ms_fma))
    return {"rows": rows, "seconds": time.time() - t0, "cfg5_room_list_build_s": build_s,
            "timing": "median device ms per call (CUDA events, inputs resident, 256 MB L2 flush between calls); "
                      "us_per_call_back_to_back = device time of 20-50 back-to-back calls / n"}


def direct_ab(P, torch, sc, beta, nb, src, rcv, orv, base, out, flush, stream, taps_launch, issue_peak, steps=5):
    """The same step through the direct-tap fp32 kernel (ism_ws_kernel<0>): RIRs/s and its own roofline."""
    ts, ism = [], []
    for i in range(steps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0, e1 = RawEvent(), RawEvent()
        a.record(stream)
        P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                       mic_pattern=sc.pattern, mode="fp32", seed=sc.seed, rir_index_base=base, out=out,
                       stream=stream, ev_ism=(e0, e1))
        b.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
            ism.append(e0.elapsed_ms(e1))
    ms, ism_ms = float(np.mean(ts)), float(np.mean(ism))
    ach = taps_launch * ISSUE_SLOTS_PER_TAP / (ism_ms / 1000.0)
    return {"value": M_PER_GPU / (ms / 1000.0), "unit": "RIRs/s", "ms_per_step": ms, "ism_ms": ism_ms,
            "roofline_frac": ach / issue_peak, "kernel": "ism_ws_kernel<0>", "steps": steps}


def traj_tc_chunks(n_sig, n_points, n_mics, L):
    """K chunks (128 outputs x 256 columns x 32) the tensor-core trajectory kernel issues per launch: the same integer
    walk as tc_tile_chunks in csrc/traj_tc_kernel.cu (segments padded to U = 4 ceil((e - j0) / 4) + 1 from the
    32-aligned start j0; chunk c of segment p touches a tile's blocks [a_lo, a_hi] when its RIR window overlaps [0, L))."""
    seglen = n_sig // n_points
    n_out = n_sig + L - 1
    nA = -(-n_out // 128)
    n_cols = nA * n_mics
    total = 0
    for tile in range(-(-n_cols // 256)):
        col0 = tile * 256
        a_lo, a_hi = col0 // n_mics, min(nA - 1, (col0 + 255) // n_mics)
        tlo, thi = 128 * a_lo, 128 * (a_hi + 1) - 1
        for p in range(n_points):
            jp = p * seglen
            ep = n_sig if p == n_points - 1 else jp + seglen
            if ep + L - 2 < tlo or jp > thi:
                continue
            j0 = jp - jp % 32
            U = 4 * ((ep - j0 + 3) // 4) + 1
            nC = (127 + U + 31) // 32
            off = -j0 - (U - 1)
            klo, khi = -(128 * a_hi + off), L - (128 * a_lo + off)
            lo = klo // 32 if klo > 0 else 0
            hi = min(nC - 1, (khi - 1) // 32) if khi > 0 else -1
            total += max(0, hi - lo + 1)
    return total


def traj_roofline(n_sig, n_pts, n_mics, L, ms, pk, pk_kind):
    """Roofline of the trajectory filter.  Tensor-core kernel (L % 4 == 0): bound "tensor" against the dense tf32
    peak (the measured bf16 cuBLAS peak x 0.5, the nominal tf32 : bf16 ratio); achieved = tf32 flops the kernel
    issues (3 products of the 3xTF32 split x 128 x 256 x 32 per chunk); useful = 2 n_sig L n_mics (the fp32 filter).
    CUDA-core kernel: FP32 FFMA issue (148 SMs x 128 lanes x clock)."""
    macs = float(n_sig) * L * n_mics
    if L % 4 == 0:
        peak = float(pk.get("bf16_tflops", 2250.0)) * 0.5e12
        issued = traj_tc_chunks(n_sig, n_pts, n_mics, L) * 3 * 128 * 256 * 32 * 2.0
        return {"bound": "tensor", "achieved": issued / (ms / 1e3) / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                "frac": issued / (ms / 1e3) / peak, "useful_frac": 2 * macs / (ms / 1e3) / peak, "traffic": None,
                "kernel": "traj_tc_kernel",
                "basis": f"{issued:.4g} tf32 flops issued per launch (3xTF32 over the signal's banded Toeplitz chunks), "
                         f"{2 * macs:.4g} useful; peak = measured bf16 {pk.get('bf16_tflops')} TF/s x 0.5 ({pk_kind})"}
    f_clk = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    issue_peak = 148 * 128 * f_clk
    return {"bound": "alu", "achieved": macs / (ms / 1e3) / 1e12, "peak": issue_peak / 1e12, "unit": "T FFMA/s",
            "frac": macs / (ms / 1e3) / issue_peak, "traffic": None, "kernel": "traj_kernel",
            "basis": f"n_sig x L x n_mics = {macs:.4g} MACs per launch (one FFMA each); peak = 148 SM x 128 lanes x "
                     f"{f_clk / 1e6:.0f} MHz ({pk_kind})"}


def run_trajectory(args, P, torch, dev, rank, world, dist, local_dev, lib):
    """--workload trajectory: one moving-source job per step (RIRs of all trajectory points + filtering)."""
    sc = W.traj1()
    n_sig = sc.meta["n_sig"]
    sig_h = W.traj_signal(n_sig)
    beta, _ = P.beta_sabine(sc.room, sc.T60)
    nb = P.t2n(sc.Tdiff, sc.room, sc.c)
    nS, nISM = P.nsamples(sc.Tmax, sc.fs), P.nsamples(sc.Tdiff, sc.fs)
    n_pts, n_mic = len(sc.pos_src), len(sc.pos_rcv)
    base = rank * n_pts * n_mic                # every rank's trajectory draws its own tail noise
    src = torch.from_numpy(sc.pos_src).to(dev)
    rcv = torch.from_numpy(sc.pos_rcv).to(dev)
    sig = torch.from_numpy(sig_h).to(dev)
    rirs = torch.empty((n_pts, n_mic, nS), dtype=torch.float32, device=dev)
    out = torch.empty((n_mic, n_sig + nS - 1), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(s_src, s_rcv, s_sig, s_rirs, s_out, st, ev=None, ev_tail=None, ev_tr=None):
        P.simulate_rir(sc.room, beta, s_src, s_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, mic_pattern=sc.pattern,
                       mode=args.mode, seed=sc.seed, rir_index_base=base, out=s_rirs, stream=st, ev_ism=ev,
                       ev_tail=ev_tail)
        if ev_tr is not None:
            ev_tr[0].record(st)
        P.simulate_trajectory(s_sig, s_rirs, out=s_out, stream=st)
        if ev_tr is not None:
            ev_tr[1].record(st)

    for _ in range(args.warmup):
        flush.zero_()
        step(src, rcv, sig, rirs, out, stream)
    torch.cuda.synchronize()
    K = args.steps
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    tr = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    ism = [(RawEvent(), RawEvent()) for _ in range(K)]
    tail = [(RawEvent(), RawEvent()) for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_dev) as clk:
        for i in range(K):
            flush.zero_()
            ev_s[i].record(stream)
            step(src, rcv, sig, rirs, out, stream, ism[i], tail[i], tr[i])
            ev_e[i].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev_s, ev_e)]
    ism_ms = float(np.mean([a.elapsed_ms(b) for a, b in ism]))
    tail_ms = float(np.mean([a.elapsed_ms(b) for a, b in tail]))
    tr_ms = float(np.mean([a.elapsed_time(b) for a, b in tr]))
    red_dev = dev if args.dist_backend == "nccl" else "cpu"
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=red_dev)
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    value = world * K / (total_ms / 1000.0)

    # ---- e2e: signal + positions from pinned host memory, filtered output back, 2 streams ----
    e2e_steps = max(2, args.e2e_steps)
    h_src, h_rcv = torch.from_numpy(sc.pos_src).pin_memory(), torch.from_numpy(sc.pos_rcv).pin_memory()
    h_sig = torch.from_numpy(sig_h).pin_memory()
    h_out = [torch.empty(out.shape, dtype=torch.float32).pin_memory() for _ in range(2)]
    d_rirs, d_out = [rirs, torch.empty_like(rirs)], [out, torch.empty_like(out)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for st_ in streams:
        st_.wait_event(e0)
    done = []
    for i in range(e2e_steps):
        st_ = streams[i % 2]
        with torch.cuda.stream(st_):
            step(h_src.to(dev, non_blocking=True), h_rcv.to(dev, non_blocking=True), h_sig.to(dev, non_blocking=True),
                 d_rirs[i % 2], d_out[i % 2], st_)
            h_out[i % 2].copy_(d_out[i % 2], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st_)
            done.append(ev)
    for ev in done[-2:]:
        stream.wait_event(ev)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
    if dist:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = world * e2e_steps / (float(e2e_ms.item()) / 1000.0)
    assert torch.equal(h_out[(e2e_steps - 1) % 2][:, :64].to(dev), out[:, :64])
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    pk, pk_kind = peaks()
    f_clk = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    issue_peak = 148 * 128 * f_clk
    H = 4e-3 * sc.fs / 2
    pairs = [(p, m) for p in range(0, n_pts, 7) for m in range(0, n_mic, 5)]
    ti = [count_taps(sc.room.astype(np.float64), sc.pos_src[p].astype(np.float64), sc.pos_rcv[m].astype(np.float64),
                     nb, nISM, sc.fs, sc.c, H, images=True) for p, m in pairs]
    taps = float(np.mean([t for t, _ in ti]))
    taps_launch = taps * n_pts * n_mic
    if args.mode == "poly":
        fir = P.poly_fir_table(4e-3, sc.fs)  # the FIR the kernel runs (reading R13)
        fir_macs = 4 * fir["far"].shape[1] + 4 * fir["nn"]
        ism_work = (float(np.mean([i for _, i in ti])) * POLY_OPS_PER_IMAGE + nISM * fir_macs) * n_pts * n_mic
    else:
        ism_work = taps_launch * ISSUE_SLOTS_PER_TAP
    ism_ach = ism_work / (ism_ms / 1000.0)
    macs = float(n_sig) * nS * n_mic
    tr_ach = macs / (tr_ms / 1000.0)
    kern = {"ism_kernel": ism_ms, "traj_kernel": tr_ms, "tail_kernel": tail_ms}
    dominant = max(kern, key=kern.get)
    roof_ism = {"bound": "alu", "achieved": ism_ach / 1e12, "peak": issue_peak / 1e12,
                "unit": "T FP32-lane-issue-slots/s", "frac": ism_ach / issue_peak, "traffic": None,
                "kernel": "ism_poly_kernel" if args.mode == "poly" else "ism_ws_kernel<0>",
                "basis": (f"{POLY_OPS_PER_IMAGE} lane-ops per in-range image + {fir_macs} MACs per output sample "
                          f"(rotated low-rank FIR, R13)" if args.mode == "poly" else
                          f"{ISSUE_SLOTS_PER_TAP} issue slots per in-window tap x {taps_launch:.4g} taps per launch")
                + f" (exact counts on {len(pairs)} sampled pairs)"}
    roof_tr = traj_roofline(n_sig, n_pts, n_mic, nS, tr_ms, pk, pk_kind)
    line = {
        "metric": TRAJ_METRIC, "value": value, "unit": "trajectories/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": sc.name, "points": n_pts, "mics": n_mic, "n_sig": n_sig, "L": nS, "nISM": nISM,
                   "room": [3, 4, 2.5], "T60": sc.T60, "fs": sc.fs, "nb_img": [int(v) for v in nb], "mode": args.mode,
                   "l2": "256 MB buffer written between timed steps (L2 126 MB)"},
        "kernel_ms": kern,
        "roofline": roof_ism if dominant.startswith("ism") else roof_tr,
        "traj_kernel": roof_tr,
        "ism_kernel": roof_ism,
        "e2e": {"value": e2e_value, "unit": "trajectories/s", "h2d_bytes_per_step": (h_src.numel() + h_rcv.numel() +
                h_sig.numel()) * 4, "d2h_bytes_per_step": h_out[0].numel() * 4, "steps": e2e_steps},
        # ISM, tail (fused into the polyphase ISM kernel), trajectory filtering (tensor-core kernel + the ordered
        # sum of its K-share partials)
        "gpu_launches": ((1 if (args.mode == "poly" and round(0.010 * sc.fs) <= 1024) else 2) +
                         (2 if nS % 4 == 0 else 1)) * K,
        "clocks": clk.summary(),
        "lib": lib,
    }
    if not args.no_cpu_baseline and world == 1:
        import oracle
        oracle.use_native()
        cores = oracle.max_threads()
        nr, nm = traj_oracle_sample(sc, sig_h, cores, 15.0)
        per_traj, nr, nm, spent = traj_oracle_times(sc, sig_h, nr, nm)
        line["cpu_baseline"] = {"value": 1.0 / per_traj, "unit": "trajectories/s", "cores": cores, "kind": "oracle",
                                "sample": f"{nr} of the {sc.M} RIRs + filtering of {nm} of {n_mic} microphones, "
                                          f"scaled to one trajectory ({spent:.1f} s)"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_cfg5(args, P, torch, dev, rank, world, dist, local_dev, lib):
    """--workload cfg5 (BASELINE.json config 5): dataset generation, 100 000 random rooms LPT-sharded over the
    ranks (no collective on the path, every room keeps its global rir_index), one batch call per
    rank per step.  value = 100 000 rooms / (max over ranks of the step's device time): strong scaling."""
    from paper_1810_11359_b200 import shard
    rb = W.cfg5(100_000)
    rooms, costs, ns, lattice = [], [], [], 0.0
    for i in range(rb.n):
        beta, _ = P.beta_sabine(rb.room[i], rb.T60[i])
        nb = P.t2n(rb.Tdiff[i], rb.room[i])
        n_i = P.nsamples(rb.Tmax[i], rb.fs)
        lattice += float(np.prod(nb.astype(np.float64)))
        rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i], nb_img=nb,
                          Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], rir_index=i, n=n_i))
        costs.append(shard.room_cost(rb.room[i], rb.Tdiff[i], rb.Tmax[i], rb.fs))
        ns.append(n_i)
    plan = shard.lpt_plan(costs, world)
    idx, mine, tot = shard.batch_shard(rooms, costs, world, rank)
    arr = P.room_array(mine)
    out = torch.empty((tot,), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        P.simulate_rir_batch(arr, rb.fs, out, seed=rb.seed, mode=args.mode, stream=stream,
                             ev_ism=ev[0] if ev else None, ev_tail=ev[1] if ev else None)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    K = args.steps
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    kev = [((RawEvent(), RawEvent()), (RawEvent(), RawEvent())) for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_dev) as clk:
        for i in range(K):
            flush.zero_()
            ev_s[i].record(stream)
            step(kev[i])
            ev_e[i].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev_s, ev_e)]
    dev_ms = [k[0][0].elapsed_ms(k[1][1]) for k in kev]
    if os.environ.get("GPURIR_BENCH_DEBUG"):
        print("cfg5 step ms", " ".join(f"{x:.1f}" for x in step_ms), "device ms", " ".join(f"{x:.1f}" for x in dev_ms),
              file=sys.stderr, flush=True)
    red_dev = dev if args.dist_backend == "nccl" else "cpu"
    tot_t = torch.tensor([sum(step_ms), sum(dev_ms)], dtype=torch.float64, device=red_dev)
    if dist:
        dist.all_reduce(tot_t, op=dist.ReduceOp.MAX)
    total_ms, total_dev_ms = float(tot_t[0].item()), float(tot_t[1].item())
    value = rb.n * K / (total_ms / 1000.0)

    # e2e through the public API from host memory: the room list in, every RIR of this rank back into pinned
    # host memory (D2H inside the timed region)
    e2e_steps = max(2, min(args.e2e_steps, 3))
    h_out = torch.empty((tot,), dtype=torch.float32).pin_memory()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        step()
        h_out.copy_(out, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
    if dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = rb.n * e2e_steps / (float(e2e_t.item()) / 1000.0)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "RIRs/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": "cfg5_100k_random_rooms_T60_0.2-1.5_fs16k", "rooms": rb.n, "rooms_rank0": len(idx),
                   "plan": "LPT on estimated room cost (shard.lpt_plan)",
                   "imbalance": shard.plan_imbalance(costs, plan), "mode": args.mode, "fs": rb.fs,
                   "samples_total": int(sum(ns)), "samples_rank0": tot,
                   "l2": "256 MB buffer written between timed steps (L2 126 MB); step output 5.4 GB"},
        "device_ms_per_step": total_dev_ms / K,
        "image_contributions_per_s": lattice * K / (total_ms / 1000.0),
        "e2e": {"value": e2e_value, "unit": "RIRs/s", "h2d_bytes_per_step": len(idx) * 160,
                "d2h_bytes_per_step": tot * 4, "steps": e2e_steps,
                "call": "gpurir_simulate_rir_batch (host room list, job table staged + uploaded inside the call) + "
                        "D2H of every RIR of the rank into pinned host memory"},
        "gpu_launches": K * (1 if args.mode == "poly" else 2),
        "clocks": clk.summary(), "lib": lib,
    }
    if not args.no_cpu_baseline and world == 1:
        import oracle
        oracle.use_native()
        cores = oracle.max_threads()
        t = time.perf_counter()
        n_done, errs = 0, []
        starts = np.concatenate([[0], np.cumsum([r["n"] for r in (rooms[i] for i in idx)])])
        sample = list(range(0, len(idx), max(1, len(idx) // 2000)))
        for j in sample:  # rooms spread over the shard until ~15 s of oracle time
            i = idx[j]
            r = rooms[i]
            h = oracle.simulate_rir(r["room_sz"], r["beta"], np.asarray(r["pos_src"], np.float32)[None],
                                    np.asarray(r["pos_rcv"], np.float32)[None], r["nb_img"], r["Tdiff"], r["Tmax"],
                                    fs=rb.fs, seed=rb.seed, rir_index_base=i)[0, 0]
            g = out[int(starts[j]):int(starts[j]) + h.size].cpu().numpy().astype(np.float64)
            errs.append(float(np.abs(g - h).max() / max(np.abs(h).max(), 1e-300)))
            n_done += 1
            if time.perf_counter() - t > 15.0:
                break
        dt = time.perf_counter() - t
        line["cpu_baseline"] = {"value": n_done / dt, "unit": "RIRs/s", "cores": 1, "kind": "oracle",
                                "sample": f"{n_done} rooms spread over the workload, one oracle call each ({dt:.1f} s; "
                                          f"a single-RIR call runs on one thread)", "build": oracle.build_flags(),
                                "cpu_model": oracle.cpu_model(), "host_cores": cores}
        line["parity"] = {"max_err_over_peak": max(errs), "n": n_done, "tol": 1e-4, "ok": max(errs) <= 1e-4,
                          "what": "the timed step's RIRs of the sampled rooms vs the oracle (C20)"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
