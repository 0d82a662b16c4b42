"""CUDA path vs the CPU oracle, element by element on identical seeded inputs (-m gpu).

Tolerances (north_star): per RIR, max |h_gpu - h_oracle| <= tol * max |h_oracle| over all
samples, tail included (reading C20): fp32 1e-4, LUT 5e-3, fp16 2e-2.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from helpers import TOL, derive, rel_err, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_1810_11359_b200 as P
    from paper_1810_11359_b200 import build as B
    B.build()
    return P


# ---------------------------------------------------------------- a1: image parameters

@pytest.mark.parametrize("pattern,orv", [(0, None), (2, [0.0, 1.0, 0.0]), (3, [1.0, 1.0, 0.0]), (4, [0.3, -0.2, 0.9])])
def test_image_params_vs_oracle(P, oracle, pattern, orv):
    room = np.float32([3, 4, 2.5])
    beta = np.float32([-0.9, 0.8, -0.7, 0.95, 0.6, -0.85])
    src, rcv = np.float32([0.7, 1.3, 0.9]), np.float32([2.2, 3.1, 1.7])
    nb = [9, 8, 7]
    x, A = P.image_params(room, beta, src, rcv, nb, 16000.0, mic_pattern=pattern, orv=orv)
    ref = oracle.image_set(room, beta, src, rcv, nb, fs=16000.0, pattern=pattern, orv=orv)
    x = x.cpu().numpy()
    A = A.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(x - ref["x"])) < 1e-9 * np.max(ref["x"])
    assert np.max(np.abs(A - ref["A"])) < 2e-6 * np.max(np.abs(ref["A"]))


def test_image_params_degenerate(P):
    room = np.float32([3, 4, 2.5])
    with pytest.raises(P.GpurirError) as e:
        P.image_params(room, [0.5] * 6, [1, 1, 1], [1, 1, 1], [3, 3, 3], 16000.0)
    assert e.value.status == 2


# ---------------------------------------------------------------- golden + random scenes (a3)

GOLD = os.path.join(os.path.dirname(__file__), "golden", "survey_appendix_b.json")


@pytest.mark.parametrize("case", ["G1", "G2", "G3", "G4"])
@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
def test_goldens(P, oracle, case, mode):
    import torch
    g = json.load(open(GOLD))["cases"][case]
    T = g["nS"] / g["fs"]
    room, beta = np.float32(g["room"]), np.float32(g["beta"])
    orv = None if g["orv"] is None else np.float32([g["orv"]])
    h = P.simulate_rir(room, beta, torch.tensor([g["src"]], dtype=torch.float32).cuda(),
                       torch.tensor([g["rcv"]], dtype=torch.float32).cuda(), g["nb"], T, T, g["fs"],
                       orV_rcv=None if orv is None else torch.from_numpy(orv).cuda(), mic_pattern=g["pattern"],
                       mode=mode, sync=True).cpu().numpy().astype(np.float64)[0, 0]
    ref = oracle.simulate_rir(room, beta, [g["src"]], [g["rcv"]], g["nb"], T, T, fs=g["fs"], pattern=g["pattern"],
                              orV_rcv=orv)[0, 0]
    assert h.shape == ref.shape
    assert rel_err(h, ref)[0] <= TOL[mode]
    if mode == "fp32":
        assert int(np.argmax(np.abs(h))) == g["argmax"]
        assert abs(h[g["argmax"]] - g["h_argmax"]) <= 1e-4 * abs(g["h_argmax"])


@pytest.mark.parametrize("kernel", ["auto", "persistent"])
@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
def test_random_scenes(P, oracle, mode, kernel):
    """S:525 style: random rooms 2-8 m, T60 0.3-1.0, <=2 src x 3 rcv, all patterns, 16 and 48 kHz.
    kernel = persistent forces the warp-specialised kernel (split = -1) on these small calls."""
    rng = np.random.default_rng(525)
    worst = 0.0
    for i in range(30):
        fs = 16000.0 if i % 3 else 48000.0
        sc = W.random_small_scene(rng, fs=fs)
        beta, nb = derive(oracle, sc)
        g = run_gpu(P, sc, beta, nb, mode=mode, split=-1 if kernel == "persistent" else 0)
        r = run_oracle(oracle, sc, beta, nb)
        e = rel_err(g, r).max()
        worst = max(worst, e)
        assert e <= TOL[mode], (i, sc.room, sc.pattern, fs, e)
    print(f"random scenes {mode}: worst {worst:.3e}")


# ---------------------------------------------------------------- configs (BASELINE.json)

def test_cfg1_fp32(P, oracle):
    sc = W.cfg1()
    beta, nb = derive(oracle, sc)
    assert list(nb) == [73, 55, 87]
    g = run_gpu(P, sc, beta, nb)
    r = run_oracle(oracle, sc, beta, nb)
    assert g.shape == r.shape == (1, 1, 4800)
    assert rel_err(g, r)[0] <= TOL["fp32"]


@pytest.mark.parametrize("mode", ["lut", "fp16", "lut_tex", "poly"])
def test_cfg1_modes(P, oracle, mode):
    sc = W.cfg1()
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode=mode)
    r = run_oracle(oracle, sc, beta, nb)
    assert rel_err(g, r)[0] <= TOL[mode]


@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
@pytest.mark.parametrize("T60", [0.1, 0.2, 0.5, 0.9, 1.4, 2.0])
def test_cfg2_t60_sweep(P, oracle, T60, mode):
    """ISM to T60/4 + diffuse tail to T60 (tail RNG is bit-reproducible, so parity covers every sample), in
    every mode (north_star: fp32 and fp16 across all five configs).  The lone RIR's poly call is forced onto
    the persistent polyphase kernel too (split = -1) besides the default (cluster items for a lone RIR)."""
    sc = W.cfg2(T60)
    beta, nb = derive(oracle, sc)
    r = run_oracle(oracle, sc, beta, nb)
    g = run_gpu(P, sc, beta, nb, mode=mode)
    assert rel_err(g, r)[0] <= TOL[mode], T60
    if mode == "poly":
        g = run_gpu(P, sc, beta, nb, mode=mode, split=-1)
        assert rel_err(g, r)[0] <= TOL[mode], T60


@pytest.mark.parametrize("kernel", ["auto", "persistent"])
@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
def test_cfg3_subset(P, oracle, mode, kernel):
    """#RIR sweep room, cardioid with random orientations, diffuse variant; first 24 receivers."""
    sc = W.cfg3(24, "diffuse")
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode=mode, split=-1 if kernel == "persistent" else 0)
    r = run_oracle(oracle, sc, beta, nb)
    assert rel_err(g, r).max() <= TOL[mode]


@pytest.mark.parametrize("mode", ["poly", "fp32"])
def test_cfg3_full_size_sampled(P, oracle, mode):
    """M = 16384 in the bench launch configuration (poly: the bench's path, 256-thread CTAs, fixed plane
    stride; fp32: the direct kernel beside it); 6 sampled RIRs re-computed by the oracle."""
    sc = W.cfg3(16384, "diffuse")
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode=mode)
    assert np.all(np.isfinite(g))
    idx = [0, 1, 4097, 8191, 12345, 16383]
    for m in idx:  # each sampled RIR with its own global tail stream id
        rj = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[m:m + 1], nb, sc.Tdiff, sc.Tmax, fs=sc.fs,
                                 pattern=sc.pattern, orV_rcv=sc.orV_rcv[m:m + 1], seed=sc.seed, rir_index_base=m)
        assert rel_err(g[0, m], rj[0, 0])[0] <= TOL[mode], m


def test_cfg3_full_size_poly_vs_direct_all_rirs(P, oracle):
    """Every one of the bench's 16384 RIRs: the polyphase path (bench default) within the fp32 tolerance of each
    RIR's peak of the direct fp32 kernel (itself pinned to the oracle above) — a property that holds at any
    size, so it covers the outputs the sampled oracle comparison does not.  Compared on the device.  Measured:
    max 5.6e-5, 99.9 % of RIRs below 2.8e-5; on the worst RIR (5590) the difference is the direct kernel's own
    error (5.6e-5 vs the oracle, degree-3 window polynomial R5) while poly is 2.5e-6 from the oracle
    (tools/diag_poly_vs_direct.py)."""
    import torch
    sc = W.cfg3(16384, "diffuse")
    beta, nb = derive(oracle, sc)
    src = torch.from_numpy(np.ascontiguousarray(sc.pos_src)).cuda()
    rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
    ov = torch.from_numpy(np.ascontiguousarray(sc.orV_rcv)).cuda()
    kw = dict(c=sc.c, orV_rcv=ov, mic_pattern=sc.pattern, seed=sc.seed, sync=True)
    a = P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, mode="poly", **kw)[0]
    b = P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, mode="fp32", **kw)[0]
    err = ((a - b).abs().amax(dim=1) / b.abs().amax(dim=1)).cpu().numpy()
    assert np.all(np.isfinite(err)) and err.max() <= TOL["poly"], (err.max(), int(err.argmax()))


@pytest.mark.parametrize("pinned", [True, False])
def test_host_call_matches_device_call(P, oracle, pinned):
    """gpurir_simulate_rir_host (host buffers, copies inside, 3 receiver chunks of <= 2048 RIRs overlapping
    their D2H with the next chunk's kernels) returns exactly the RIRs of one device call in poly mode (the
    chunks keep their global RIR index for the tail), from pinned tensors and from pageable numpy arrays."""
    import torch
    sc = W.cfg3(5000, "diffuse")
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode="poly").astype(np.float32)
    if pinned:
        src, rcv, orv = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (sc.pos_src, sc.pos_rcv, sc.orV_rcv))
        out = torch.empty((1, 5000, ref.shape[2]), dtype=torch.float32).pin_memory()
    else:
        src, rcv, orv, out = sc.pos_src, sc.pos_rcv, sc.orV_rcv, None
    h = P.simulate_rir_host(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv,
                            mic_pattern=sc.pattern, mode="poly", seed=sc.seed, out=out)
    h = h.numpy() if isinstance(h, torch.Tensor) else h
    assert h.shape == ref.shape and np.array_equal(h, ref)


@pytest.mark.parametrize("M", [591, 592, 2600])
def test_fused_tail_threshold_bit_identical(P, oracle, M):
    """Shards of a call and the chunks of a host call (2600 = 2048 + 552) give the bits of one device call, the
    diffuse tail fused into the polyphase kernel or not: the fusion threshold GPURIR_FUSE_MIN_PER_SM is 0 (always
    fused); an A/B build with 4 puts 591 / 592 and the host call's chunks on either side of it.
    Sampled RIRs checked against the oracle."""
    sc = W.cfg3(M, "diffuse")
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode="poly").astype(np.float32)
    if M == 2600:
        got = P.simulate_rir_host(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c,
                                  orV_rcv=sc.orV_rcv, mic_pattern=sc.pattern, mode="poly", seed=sc.seed)
        assert got.shape == ref.shape and np.array_equal(got, ref)
    else:
        half = M // 2  # two calls below the threshold: tail_kernel, and the same bits as the whole call
        parts = [run_gpu(P, sc, beta, nb, mode="poly", rir_index_base=a, pos_rcv=sc.pos_rcv[a:b], orv=sc.orV_rcv[a:b])
                 for a, b in ((0, half), (half, M))]
        assert np.array_equal(ref, np.concatenate(parts, axis=1).astype(np.float32))
    for m in (0, M - 1):
        rj = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[m:m + 1], nb, sc.Tdiff, sc.Tmax, fs=sc.fs,
                                 pattern=sc.pattern, orV_rcv=sc.orV_rcv[m:m + 1], seed=sc.seed, rir_index_base=m)
        assert rel_err(ref[0, m], rj[0, 0])[0] <= TOL["poly"], m


def test_host_call_directional_source(P, oracle):
    """The host call with a directional (cardioid) source and receivers: equal to the device call (poly)."""
    import torch
    sc = W.cfg3(3000, "diffuse")
    beta, nb = derive(oracle, sc)
    ors = np.array([[0.6, -0.8, 0.0]], np.float32)
    ref = P.simulate_rir(sc.room, beta, torch.from_numpy(sc.pos_src).cuda(), torch.from_numpy(sc.pos_rcv).cuda(), nb,
                         sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=torch.from_numpy(sc.orV_rcv).cuda(),
                         mic_pattern=sc.pattern, mode="poly", seed=sc.seed, orV_src=torch.from_numpy(ors).cuda(),
                         spkr_pattern="cardioid", sync=True).cpu().numpy()
    h = P.simulate_rir_host(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c,
                            orV_rcv=sc.orV_rcv, mic_pattern=sc.pattern, mode="poly", seed=sc.seed, orV_src=ors,
                            spkr_pattern="cardioid")
    assert np.array_equal(h, ref)


def test_host_call_many_sources(P, oracle):
    """Chunks of whole sources (M_rcv small): every RIR, tail included, matches the oracle on its global index."""
    sc = W.cfg3(6, "diffuse")
    rng = np.random.default_rng(5)
    sc.pos_src = (rng.random((700, 3)) * np.array([2.4, 3.4, 1.9]) + 0.3).astype(np.float32)
    beta, nb = derive(oracle, sc)
    h = P.simulate_rir_host(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c,
                            orV_rcv=sc.orV_rcv, mic_pattern=sc.pattern, mode="poly", seed=sc.seed, rir_index_base=7)
    assert h.shape[:2] == (700, 6)
    for s in (0, 340, 341, 699):  # 2048 // 6 = 341 sources per chunk: both sides of the first boundary
        r = oracle.simulate_rir(sc.room, beta, sc.pos_src[s:s + 1], sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, fs=sc.fs,
                                pattern=sc.pattern, orV_rcv=sc.orV_rcv, seed=sc.seed, rir_index_base=7 + 6 * s)
        assert rel_err(h[s].astype(np.float64), r[0]).max() <= TOL["poly"], s


@pytest.mark.parametrize("kernel", ["auto", "persistent"])
@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
def test_cfg4_48k_array(P, oracle, mode, kernel):
    sc = W.cfg4("a")
    sc.pos_rcv = sc.pos_rcv[:8]
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode=mode, split=-1 if kernel == "persistent" else 0)
    r = run_oracle(oracle, sc, beta, nb)
    assert rel_err(g, r).max() <= TOL[mode]


# ---------------------------------------------------------------- edge cases

def _scene(**kw):
    base = dict(name="edge", room=np.float32([3, 4, 2.5]), T60=0.4, pos_src=np.float32([[1.0, 1.0, 1.0]]),
                pos_rcv=np.float32([[2.0, 3.0, 1.5]]), orV_rcv=None, pattern=0, Tdiff=0.03, Tmax=0.05, fs=16000.0,
                seed=99)
    base.update(kw)
    return W.Scene(**base)


@pytest.mark.parametrize("kw", [
    dict(Tdiff=0.0, Tmax=0.03),                      # tail only -> silent
    dict(Tdiff=0.05, Tmax=0.05),                     # ISM only
    dict(Tdiff=0.1, Tmax=0.05),                      # Tdiff > Tmax -> ISM to Tmax
    dict(Tdiff=0.0301, Tmax=0.0511),                 # ragged lengths (not multiples of the tile / of 4)
    dict(pos_src=np.float32([[1.0, 2.0, 1.25]]), pos_rcv=np.float32([[3.14375, 2.0, 1.25]]),
         room=np.float32([5, 4, 2.5])),             # direct path on an integer sample delay
    dict(pos_rcv=np.float32([[3.0, 3.0, 1.5]])),     # receiver on a wall
    dict(pos_src=np.float32([[1.0, 1.0, 1.0], [0.5, 3.5, 2.0]]), pos_rcv=np.float32([[2.0, 3.0, 1.5], [1.1, 0.2, 0.3],
                                                                                      [2.9, 3.9, 2.4]])),  # M_src > 1
    dict(T60=0.05, clamp=True),                      # infeasible T60 clamped -> beta = 0, direct path only
])
@pytest.mark.parametrize("mode,split", [("fp32", 0), ("fp32", -1), ("poly", -1), ("poly", 0)])
def test_edge_cases(P, oracle, kw, mode, split):
    """Edge cases through the cluster-split (auto) and persistent direct kernels and the polyphase kernel
    (persistent and cluster items)."""
    sc = _scene(**kw)
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode=mode, split=split)
    r = run_oracle(oracle, sc, beta, nb)
    assert g.shape == r.shape
    if np.max(np.abs(r)) == 0:
        assert np.max(np.abs(g)) == 0
    else:
        assert rel_err(g, r).max() <= TOL[mode]


def test_nb_img_one(P, oracle):
    sc = _scene(Tdiff=0.02, Tmax=0.02)
    beta, _ = derive(oracle, sc)
    g = run_gpu(P, sc, beta, [1, 1, 1])
    r = run_oracle(oracle, sc, beta, [1, 1, 1])
    assert rel_err(g, r)[0] <= TOL["fp32"]


def test_degenerate_and_invalid(P):
    import torch
    room = np.float32([3, 4, 2.5])
    s = torch.tensor([[1.0, 1.0, 1.0]], device="cuda")
    # every accumulation kernel flags d_n = 0 (the polyphase kernel per lattice column: persistent and cluster items)
    for mode, split in (("fp32", 0), ("fp32", -1), ("poly", -1), ("poly", 0), ("poly", 8)):
        with pytest.raises(P.GpurirError) as e:
            P.simulate_rir(room, [0.9] * 6, s, s.clone(), [3, 3, 3], 0.02, 0.02, 16000.0, mode=mode, split=split,
                           sync=True)
        assert e.value.status == 2
    with pytest.raises(P.GpurirError) as e:
        P.simulate_rir(room, [1.1] + [0.9] * 5, s, s + 0.5, [3, 3, 3], 0.02, 0.02, 16000.0)
    assert e.value.status == 1
    with pytest.raises(P.GpurirError) as e:
        P.simulate_rir(room, [0.9] * 6, s, s + 0.5, [3, 3, 3], 0.02, 0.02, 16000.0, mic_pattern="cardioid",
                       orV_rcv=torch.zeros((1, 3), device="cuda"), sync=True)
    assert e.value.status == 1
    assert P.device_status() == 0


# ---------------------------------------------------------------- determinism, sharding, batch

@pytest.mark.parametrize("split", [0, -1])
def test_run_to_run_deterministic(P, oracle, split):
    sc = W.cfg3(32, "diffuse")
    beta, nb = derive(oracle, sc)
    a = run_gpu(P, sc, beta, nb, split=split)
    b = run_gpu(P, sc, beta, nb, split=split)
    assert np.array_equal(a, b)


def test_persistent_matches_cluster_kernel(P, oracle):
    """The two ISM kernels evaluate the same records in the same bin order per tile (the persistent one
    windows them differently and the persistent one uses 512-sample tiles, so the fp32 delay offsets
    differ in rounding), so they agree to fp32 rounding of the delays."""
    sc = W.cfg3(64, "diffuse")
    beta, nb = derive(oracle, sc)
    a = run_gpu(P, sc, beta, nb, split=1)
    b = run_gpu(P, sc, beta, nb, split=-1)
    assert rel_err(b, a).max() <= 1e-4  # both are within ~1e-5 of the oracle (profiles/r01_parity.txt)


@pytest.mark.parametrize("split", [2, -1])
def test_shard_invariance(P, oracle, split):
    """§8(e): running the receivers in 4 shards with rir_index_base offsets reproduces the unsharded
    call bit for bit (fixed kernel choice so the per-tile summation order is identical)."""
    sc = W.cfg3(64, "diffuse")
    beta, nb = derive(oracle, sc)
    full = run_gpu(P, sc, beta, nb, split=split)
    parts = []
    for s in range(4):
        sl = slice(16 * s, 16 * (s + 1))
        parts.append(run_gpu(P, sc, beta, nb, split=split, rir_index_base=16 * s, pos_rcv=sc.pos_rcv[sl],
                             orv=sc.orV_rcv[sl]))
    assert np.array_equal(full, np.concatenate(parts, axis=1))


def test_split_factor_within_tolerance(P, oracle):
    sc = W.cfg1()
    beta, nb = derive(oracle, sc)
    r = run_oracle(oracle, sc, beta, nb)
    for split in (1, 2, 4, 8):
        g = run_gpu(P, sc, beta, nb, split=split)
        assert rel_err(g, r)[0] <= TOL["fp32"], split


def test_reciprocity_gpu(P, oracle):
    sc = W.cfg1()
    beta, nb = derive(oracle, sc)
    a = run_gpu(P, sc, beta, nb)
    sw = W.Scene("swap", sc.room, sc.T60, sc.pos_rcv, sc.pos_src, None, 0, sc.Tdiff, sc.Tmax, sc.fs)
    b = run_gpu(P, sw, beta, nb)
    assert rel_err(a, b)[0] <= 1e-5


def _batch(oracle, rb, idx, base_off=0, rir_index=None):
    """gpurir_room dicts of rooms idx of a workloads.RoomBatch (beta, nb_img from the oracle's helpers), packed
    into ragged rows from base_off; returns (rooms, row offsets, total samples)."""
    rooms, offs, off = [], [], base_off
    for k, i in enumerate(idx):
        beta, _ = oracle.beta_sabine(rb.room[i], rb.T60[i])
        nb = oracle.t2n(rb.Tdiff[i], rb.room[i])
        rooms.append(dict(room_sz=rb.room[i], beta=beta.astype(np.float32), pos_src=rb.pos_src[i],
                          pos_rcv=rb.pos_rcv[i], nb_img=nb, Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], out_offset=off,
                          rir_index=int(i if rir_index is None else rir_index[k])))
        offs.append(off)
        off += oracle.nsamples(rb.Tmax[i], rb.fs)
    return rooms, offs, off


def _oracle_room(oracle, rb, room, base):
    src = np.asarray(room["pos_src"], np.float32)[None]
    rcv = np.asarray(room["pos_rcv"], np.float32)[None]
    return oracle.simulate_rir(room["room_sz"], room["beta"], src, rcv, room["nb_img"], room["Tdiff"], room["Tmax"],
                               fs=rb.fs, seed=rb.seed, rir_index_base=base + room["rir_index"])[0, 0]


@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
def test_batch_rooms_vs_oracle(P, oracle, mode):
    """config 5 shape in every mode: independent rooms, ragged rows, tail streams rir_index_base + rir_index."""
    import torch
    rb = W.cfg5(12)
    rooms, offs, tot = _batch(oracle, rb, range(rb.n))
    out = torch.full((tot,), float("nan"), device="cuda")
    P.simulate_rir_batch(rooms, rb.fs, out, seed=rb.seed, rir_index_base=1000, sync=True, mode=mode)
    o = out.cpu().numpy().astype(np.float64)
    for i, room in enumerate(rooms):
        r = _oracle_room(oracle, rb, room, 1000)
        assert rel_err(o[offs[i]:offs[i] + r.size], r)[0] <= TOL[mode], i


def test_batch_room_equals_single_room_call(P, oracle):
    """Polyphase: a room's RIR in a batch is bit-identical to the same room simulated alone (end-aligned
    tiles and per-tile fixed point in both; the batch fuses the diffuse tail like the single-room call)."""
    import torch
    rb = W.cfg5(40)
    rooms, offs, tot = _batch(oracle, rb, range(rb.n))
    out = torch.empty((tot,), device="cuda")
    P.simulate_rir_batch(rooms, rb.fs, out, seed=rb.seed, rir_index_base=5, sync=True, mode="poly")
    o = out.cpu().numpy()
    for i in (0, 17, 39):
        rm = rooms[i]
        h = P.simulate_rir(rm["room_sz"], rm["beta"], torch.tensor([rm["pos_src"]], device="cuda"),
                           torch.tensor([rm["pos_rcv"]], device="cuda"), rm["nb_img"], rm["Tdiff"], rm["Tmax"], rb.fs,
                           mode="poly", split=-1, seed=rb.seed, rir_index_base=5 + i, sync=True).cpu().numpy()[0, 0]
        assert np.array_equal(o[offs[i]:offs[i] + h.size], h), i


@pytest.mark.parametrize("mode", ["poly", "fp32"])
def test_batch_lpt_shards_reproduce_unsharded(P, oracle, mode):
    """SURVEY §8(e) / P:167: an 8-way LPT shard of a 2000-room batch (rooms in LPT order, not contiguous), each
    shard one batch call with the rooms' global rir_index, reproduces the unsharded call — bit for bit in
    polyphase mode (a RIR's bits depend only on its own room), within the fp32 tolerance of each other in
    direct mode (shards may take the other direct kernel)."""
    import torch
    from paper_1810_11359_b200 import shard
    rb = W.cfg5(2000)
    rooms, offs, tot = _batch(oracle, rb, range(rb.n))
    full = torch.empty((tot,), device="cuda")
    P.simulate_rir_batch(rooms, rb.fs, full, seed=rb.seed, mode=mode)
    costs = [shard.room_cost(rb.room[i], rb.Tdiff[i], rb.Tmax[i], rb.fs) for i in range(rb.n)]
    plan = shard.lpt_plan(costs, 8)
    assert shard.plan_imbalance(costs, plan) < 1.01
    got = torch.full((tot,), float("nan"), device="cuda")
    for ranks in plan:
        idx = list(ranks)
        sub, soff, stot = _batch(oracle, rb, idx)
        buf = torch.empty((stot,), device="cuda")
        P.simulate_rir_batch(sub, rb.fs, buf, seed=rb.seed, mode=mode)
        for k, i in enumerate(idx):
            n = oracle.nsamples(rb.Tmax[i], rb.fs)
            got[offs[i]:offs[i] + n] = buf[soff[k]:soff[k] + n]
    torch.cuda.synchronize()
    if mode == "poly":
        assert torch.equal(got, full)
    else:
        f, g = full.cpu().numpy(), got.cpu().numpy()
        for i in range(0, rb.n, 97):
            n = oracle.nsamples(rb.Tmax[i], rb.fs)
            assert rel_err(g[offs[i]:offs[i] + n], f[offs[i]:offs[i] + n])[0] <= TOL["fp32"], i


def test_batch_full_size_cfg5_sampled(P, oracle):
    """config 5 at full size: 100 000 random rooms in ONE batch call (polyphase, the bench's path), 64 rooms
    sampled across the batch checked against the oracle, tail included."""
    import torch
    rb = W.cfg5(100_000)
    rooms, offs, tot = _batch(oracle, rb, range(rb.n))
    out = torch.empty((tot,), device="cuda")
    P.simulate_rir_batch(rooms, rb.fs, out, seed=rb.seed, sync=True, mode="poly")
    for i in np.linspace(0, rb.n - 1, 64).astype(int):
        r = _oracle_room(oracle, rb, rooms[i], 0)
        g = out[offs[i]:offs[i] + r.size].cpu().numpy().astype(np.float64)
        assert rel_err(g, r)[0] <= TOL["poly"], i
    del out
    torch.cuda.empty_cache()


def test_batch_stream_ordered_workspace_and_status(P, oracle):
    """The batch call is stream-ordered: two calls on two streams without synchronisation, one with a caller
    workspace of exactly gpurir_workspace_bytes(), both correct after the streams drain; a workspace one byte
    short is EINVAL; a degenerate room (source on the receiver) raises the CALLER's status word (opts.status),
    not the device's shared one."""
    import torch
    rb = W.cfg5(300)
    rooms, offs, tot = _batch(oracle, rb, range(rb.n))
    need = P.workspace_bytes(rooms, rb.fs, mode="poly")
    assert need > 0
    ws = torch.empty((need,), dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    a, b = torch.empty((tot,), device="cuda"), torch.empty((tot,), device="cuda")
    P.simulate_rir_batch(rooms, rb.fs, a, seed=rb.seed, mode="poly", stream=s1, workspace=ws)
    P.simulate_rir_batch(rooms, rb.fs, b, seed=rb.seed, mode="poly", stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    for i in (0, 299):
        r = _oracle_room(oracle, rb, rooms[i], 0)
        assert rel_err(a[offs[i]:offs[i] + r.size].cpu().numpy().astype(np.float64), r)[0] <= TOL["poly"]
    with pytest.raises(P.GpurirError) as e:
        P.simulate_rir_batch(rooms, rb.fs, a, mode="poly", workspace=ws[:need - 1])
    assert e.value.status == P._lib.EINVAL
    bad = [dict(rooms[0], pos_rcv=rooms[0]["pos_src"])]
    st = torch.zeros((1,), dtype=torch.int32, device="cuda")
    P.simulate_rir_batch(bad, rb.fs, a, mode="poly", split=-1, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) != 0 and P.device_status(reset=True) == 0
    st.zero_()
    with pytest.raises(P.GpurirError) as e:
        P.simulate_rir_batch(bad, rb.fs, a, mode="poly", split=-1, status=st, sync=True)
    assert e.value.status == P._lib.EDEGENERATE and int(st.item()) == 0


@pytest.mark.parametrize("mode", ["poly", "fp32"])
def test_misaligned_output_rows(P, oracle, mode):
    """an output view starting 4 bytes into an allocation (contiguous, not 16-B aligned) — the tail's
    float4 stores must fall back to scalar stores (fused polyphase tail and tail_kernel alike)."""
    import torch
    sc = W.cfg3(64, "diffuse")
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode=mode).astype(np.float32)
    nS = ref.shape[-1]
    buf = torch.empty((64 * nS + 1,), device="cuda")
    out = buf[1:]
    src = torch.from_numpy(sc.pos_src).cuda()
    rcv, orv = torch.from_numpy(sc.pos_rcv).cuda(), torch.from_numpy(sc.orV_rcv).cuda()
    P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=orv, mic_pattern=sc.pattern,
                   mode=mode, seed=sc.seed, out=out, sync=True)
    assert np.array_equal(out.cpu().numpy().reshape(ref.shape), ref)


def test_host_call_small_last_chunk_bit_identical(P, oracle):
    """a host call whose last chunk has 10 receivers (2058 = 2048 + 10; 30 polyphase work items,
    below the kernel's 32) still runs every chunk on the polyphase kernel: the bits of one device call."""
    sc = W.cfg3(2058, "diffuse")
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode="poly").astype(np.float32)
    got = P.simulate_rir_host(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c,
                              orV_rcv=sc.orV_rcv, mic_pattern=sc.pattern, mode="poly", seed=sc.seed)
    assert np.array_equal(got, ref)


# ---------------------------------------------------------------- NEXT row f1: trajectory filtering

TRAJ_TOL = 2e-5  # fp32 accumulation of up to L products per output sample (reading R8)


@pytest.mark.parametrize("n_sig,n_points,n_mics,L", [(5003, 7, 3, 1337), (4096, 1, 2, 4096), (777, 777, 1, 64),
                                                     (10007, 13, 4, 1), (2500, 3, 5, 5000),
                                                     (20000, 9, 2, 9000), (30011, 31, 1, 2049),
                                                     (16000, 100, 33, 1200)])
@pytest.mark.parametrize("split", [0, -1, 3])
def test_trajectory_vs_oracle(P, oracle, n_sig, n_points, n_mics, L, split):
    """split 0: automatic (the tcgen05 kernel when L % 4 == 0, else the CUDA-core kernel); -1: the CUDA-core
    kernel; 3: the tensor-core kernel with a K split of 3 (partials summed in split order).  33 mics: tiles
    whose 256 (block, mic) columns straddle blocks and a ragged last tile."""
    import torch
    rng = np.random.default_rng(n_sig + L)
    sig = rng.standard_normal(n_sig).astype(np.float32)
    rirs = (rng.standard_normal((n_points, n_mics, L)) * np.exp(-np.arange(L) / max(L / 4, 1))).astype(np.float32)
    sg, rg = torch.from_numpy(sig).cuda(), torch.from_numpy(rirs).cuda()
    g = P.simulate_trajectory(sg, rg, sync=True, split=split).cpu().numpy()
    r = oracle.simulate_trajectory(sig, rirs)
    assert g.shape == r.shape == (n_mics, n_sig + L - 1)
    assert np.max(np.abs(g - r)) <= TRAJ_TOL * np.max(np.abs(r))
    assert np.array_equal(g, P.simulate_trajectory(sg, rg, sync=True, split=split).cpu().numpy())  # deterministic


def test_trajectory_moving_source_with_oracle_rirs(P, oracle):
    """A source moving across a 3x4x2.5 room, 6 trajectory points x 4 mics, RIR banks from the oracle."""
    import torch
    room = np.float32([3, 4, 2.5])
    beta, _ = oracle.beta_sabine(room, 0.4)
    beta = beta.astype(np.float32)
    pts = np.float32([[0.5 + 0.35 * i, 1.0 + 0.2 * i, 1.2] for i in range(6)])
    mics = np.float32([[2.0, 2.5, 1.3], [2.1, 2.5, 1.3], [2.0, 2.6, 1.3], [2.1, 2.6, 1.3]])
    nb = oracle.t2n(0.06, room)
    rirs = oracle.simulate_rir(room, beta, pts, mics, nb, 0.06, 0.06).astype(np.float32)  # [6][4][960]
    sig = np.random.default_rng(3).standard_normal(16000).astype(np.float32)
    g = P.simulate_trajectory(torch.from_numpy(sig).cuda(), torch.from_numpy(rirs).cuda(), sync=True).cpu().numpy()
    r = oracle.simulate_trajectory(sig, rirs)
    assert np.max(np.abs(g - r)) <= TRAJ_TOL * np.max(np.abs(r))


@pytest.mark.parametrize("L", [50, 52])
def test_trajectory_impulse(P, L):
    """Unit impulses in the RIR bank reproduce the (delayed) signal: exactly on the CUDA-core kernel (L = 50),
    within the 3xTF32 split's 2^-22 per product on the tensor-core kernel (L = 52: tf32 keeps 11 of the 13 bits
    of the low part), and exact zeros elsewhere on both."""
    import torch
    sig = torch.randn(3001, device="cuda")
    rirs = torch.zeros((3, 2, L), device="cuda")
    rirs[:, 0, 0] = 1.0
    rirs[:, 1, 7] = 1.0
    out = P.simulate_trajectory(sig, rirs, sync=True)
    tol = 0.0 if L % 4 else 2.0 ** -21
    assert torch.max(torch.abs(out[0, :3001] - sig) / torch.abs(sig).clamp_min(1e-30)) <= tol
    assert torch.max(torch.abs(out[1, 7:3008] - sig) / torch.abs(sig).clamp_min(1e-30)) <= tol
    assert torch.all(out[0, 3001:] == 0) and torch.all(out[1, :7] == 0)


def test_trajectory_invalid(P):
    import torch
    with pytest.raises(P.GpurirError):
        P.simulate_trajectory(torch.randn(3, device="cuda"), torch.zeros((5, 1, 4), device="cuda"))


def test_trajectory_full_size_sampled_mics(P, oracle):
    """bench.py's trajectory launch (traj1: 1 s, 100 points, 32 mics, L = 11200) with seeded random banks;
    the oracle filters 2 of the 32 microphones in full."""
    import torch
    import workloads as W
    sc = W.traj1()
    sig = W.traj_signal(sc.meta["n_sig"])
    L = 11200
    rirs = (np.random.default_rng(12).standard_normal((len(sc.pos_src), len(sc.pos_rcv), L)) *
            np.exp(-np.arange(L) / 2000.0)).astype(np.float32)
    g = P.simulate_trajectory(torch.from_numpy(sig).cuda(), torch.from_numpy(rirs).cuda(), sync=True).cpu().numpy()
    gf = P.simulate_trajectory(torch.from_numpy(sig).cuda(), torch.from_numpy(rirs).cuda(), sync=True,
                               split=-1).cpu().numpy()  # the CUDA-core kernel
    assert np.max(np.abs(g - gf)) <= TRAJ_TOL * np.max(np.abs(gf))
    for m in (0, 17):
        r = oracle.simulate_trajectory(sig, rirs[:, m:m + 1])[0]
        assert np.max(np.abs(g[m] - r)) <= TRAJ_TOL * np.max(np.abs(r))


# ---------------------------------------------------------------- NEXT row f3: source directivity, weighted walls

@pytest.mark.parametrize("spkr,ors,mic,orv", [(2, [0.3, -0.5, 0.8], 0, None), (4, [1.0, 0.0, 0.0], 3, [0.0, 1.0, 0.0]),
                                              (1, [-0.2, 0.7, 0.1], 2, [0.3, -0.2, 0.9])])
def test_image_params_source_pattern(P, oracle, spkr, ors, mic, orv):
    room = np.float32([3, 4, 2.5])
    beta = np.float32([-0.9, 0.8, -0.7, 0.95, 0.6, -0.85])
    src, rcv = np.float32([0.7, 1.3, 0.9]), np.float32([2.2, 3.1, 1.7])
    nb = [9, 8, 7]
    x, A = P.image_params(room, beta, src, rcv, nb, 16000.0, mic_pattern=mic, orv=orv, spkr_pattern=spkr, ors=ors)
    ref = oracle.image_set(room, beta, src, rcv, nb, fs=16000.0, pattern=mic, orv=orv, spkr_pattern=spkr, ors=ors)
    A = A.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(A - ref["A"])) < 2e-6 * np.max(np.abs(ref["A"]))


def _dir_scene(rng, fs, Ms, Mr, T):
    sc = W.random_small_scene(rng, fs=fs, max_src=Ms, max_rcv=Mr, T=T)
    spkr = int(rng.integers(1, 5))
    v = rng.standard_normal((sc.pos_src.shape[0], 3))
    ors = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(np.float32)
    return sc, spkr, ors


def _run_dir(P, sc, beta, nb, spkr, ors, mode="fp32", split=0):
    import torch
    ov = torch.from_numpy(sc.orV_rcv).cuda() if sc.orV_rcv is not None else None
    h = P.simulate_rir(sc.room, beta, torch.from_numpy(sc.pos_src).cuda(), torch.from_numpy(sc.pos_rcv).cuda(), nb,
                       sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, orV_rcv=ov, mic_pattern=sc.pattern, mode=mode, seed=sc.seed,
                       split=split, sync=True, orV_src=torch.from_numpy(ors).cuda(), spkr_pattern=spkr)
    return h.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("kernel", ["auto", "persistent"])
@pytest.mark.parametrize("mode", ["fp32", "lut", "fp16", "lut_tex", "poly"])
def test_source_directivity_random_scenes(P, oracle, mode, kernel):
    """f3 (reading R10): random rooms, all source and receiver patterns, 16 / 48 kHz, both ISM kernels."""
    rng = np.random.default_rng(3310)
    for i in range(12):
        sc, spkr, ors = _dir_scene(rng, 16000.0 if i % 3 else 48000.0, 2, 3, None)
        beta, nb = derive(oracle, sc)
        g = _run_dir(P, sc, beta, nb, spkr, ors, mode=mode, split=-1 if kernel == "persistent" else 0)
        r = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, fs=sc.fs, c=sc.c,
                                pattern=sc.pattern, orV_rcv=sc.orV_rcv, seed=sc.seed, spkr_pattern=spkr, orV_src=ors)
        assert rel_err(g, r).max() <= TOL[mode], (i, spkr, sc.pattern)


def test_source_directivity_with_tail(P, oracle):
    """Directional source + diffuse tail: the envelope is estimated from the directional ISM part."""
    rng = np.random.default_rng(77)
    sc, spkr, ors = _dir_scene(rng, 16000.0, 1, 4, 0.05)
    sc.Tmax = 0.2
    beta, nb = derive(oracle, sc)
    g = _run_dir(P, sc, beta, nb, spkr, ors)
    r = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv, nb, sc.Tdiff, sc.Tmax, fs=sc.fs, c=sc.c,
                            pattern=sc.pattern, orV_rcv=sc.orV_rcv, seed=sc.seed, spkr_pattern=spkr, orV_src=ors)
    assert rel_err(g, r).max() <= TOL["fp32"]


@pytest.mark.parametrize("split", [0, -1])
def test_omni_source_dir_entry_bit_identical(P, oracle, split):
    """gpurir_simulate_rir == gpurir_simulate_rir_dir with an omni source (g_s = 1 exactly)."""
    sc = W.cfg3(16, "diffuse")
    beta, nb = derive(oracle, sc)
    a = run_gpu(P, sc, beta, nb, split=split)
    b = _run_dir(P, sc, beta, nb, 0, np.float32([[0.0, 0.0, 1.0]]), split=split)
    assert np.array_equal(a, b)


def test_directional_reciprocity_gpu(P, oracle):
    sc = W.cfg1()
    beta, nb = derive(oracle, sc)
    oa, ob = np.float32([[0.3, -0.5, 0.8]]), np.float32([[-0.6, 0.2, 0.4]])
    s1 = W.Scene("d", sc.room, sc.T60, sc.pos_src, sc.pos_rcv, ob, 3, sc.Tdiff, sc.Tmax, sc.fs)
    s2 = W.Scene("d", sc.room, sc.T60, sc.pos_rcv, sc.pos_src, oa, 2, sc.Tdiff, sc.Tmax, sc.fs)
    a = _run_dir(P, s1, beta, nb, 2, oa)
    b = _run_dir(P, s2, beta, nb, 3, ob)
    assert rel_err(a, b)[0] <= 1e-5


def test_batch_directional_weighted_rooms(P, oracle):
    """Batch API with per-room source patterns and non-uniform wall weights (f3) vs the oracle."""
    import torch
    rb = W.cfg5(10)
    rng = np.random.default_rng(5150)
    rooms, refs, off = [], [], 0
    for i in range(rb.n):
        w = rng.uniform(0.3, 1.0, 6)
        beta, _ = oracle.beta_sabine_weighted(rb.room[i], rb.T60[i], w, clamp=True)
        beta = beta.astype(np.float32)
        nb = oracle.t2n(rb.Tdiff[i], rb.room[i])
        nS = oracle.nsamples(rb.Tmax[i], rb.fs)
        spkr = i % 5
        v = rng.standard_normal(3)
        ors = (v / np.linalg.norm(v)).astype(np.float32)
        rooms.append(dict(room_sz=rb.room[i], beta=beta, pos_src=rb.pos_src[i], pos_rcv=rb.pos_rcv[i], nb_img=nb,
                          Tdiff=rb.Tdiff[i], Tmax=rb.Tmax[i], out_offset=off, orV_src=ors, spkr_pattern=spkr))
        refs.append(oracle.simulate_rir(rb.room[i], beta, rb.pos_src[i:i + 1], rb.pos_rcv[i:i + 1], nb, rb.Tdiff[i],
                                        rb.Tmax[i], fs=rb.fs, seed=rb.seed, rir_index_base=i, spkr_pattern=spkr,
                                        orV_src=ors[None] if spkr else None)[0, 0])
        off += nS
    out = torch.full((off,), float("nan"), device="cuda")
    P.simulate_rir_batch(rooms, rb.fs, out, seed=rb.seed, sync=True)
    o = out.cpu().numpy().astype(np.float64)
    off = 0
    for i, r in enumerate(refs):
        g = o[off:off + r.size]
        off += r.size
        assert rel_err(g, r)[0] <= TOL["fp32"], i


# ---------------------------------------------------------------- polyphase mode (reading R11)

def test_poly_deterministic_and_shard_invariant(P, oracle):
    """Integer fixed-point aggregation: bitwise identical run to run and across receiver shards."""
    sc = W.cfg3(64, "diffuse")
    beta, nb = derive(oracle, sc)
    a = run_gpu(P, sc, beta, nb, mode="poly")
    b = run_gpu(P, sc, beta, nb, mode="poly")
    assert np.array_equal(a, b)
    parts = [run_gpu(P, sc, beta, nb, mode="poly", rir_index_base=16 * s, pos_rcv=sc.pos_rcv[16 * s:16 * (s + 1)],
                     orv=sc.orV_rcv[16 * s:16 * (s + 1)]) for s in range(4)]
    assert np.array_equal(a, np.concatenate(parts, axis=1))


@pytest.mark.parametrize("split", [-1, -2])
def test_poly_long_rir_per_tile_scale(P, oracle, split):
    """Full ISM to 0.7 s (config 3 (ii)): the per-tile fixed point keeps every tile single-word (split -1; the
    late tiles' scale follows their closest image) and the two-word scheme forced on every tile (split -2,
    the test hook) must agree with the oracle too; parity at the fp32 tolerance on 2 receivers."""
    sc = W.cfg3(2, "full")
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode="poly", split=split)  # 22 work items: forced onto the polyphase kernel
    r = run_oracle(oracle, sc, beta, nb)
    assert rel_err(g, r).max() <= TOL["poly"]


@pytest.mark.parametrize("fs", [16000.0, 48000.0])
def test_poly_rigid_centred_cube(P, oracle, fs):
    """The fixed point's worst case: rigid walls (beta = 1: every image at full amplitude, all of one sign)
    in a cube with the source at its centre and receivers on its symmetry axes, where the image lattice
    stacks up to r3(n) images on one delay (tests/test_poly_headroom.py).  Polyphase vs oracle at the fp32
    tolerance, plus the other sign pattern (beta = -1)."""
    room = np.array([2.0, 2.0, 2.0], np.float32)
    src = np.array([[1.0, 1.0, 1.0]], np.float32)
    rcv = np.array([[1.0, 1.0, 1.5], [1.0, 1.5, 1.5], [0.5, 1.0, 1.0], [1.25, 1.25, 1.25]], np.float32)
    T = 0.05
    nb = oracle.t2n(T, room, 343.0)
    for b in (1.0, -1.0):
        beta = np.full(6, b, np.float32)
        import torch
        g = P.simulate_rir(room, beta, torch.from_numpy(src).cuda(), torch.from_numpy(rcv).cuda(), nb, T, T, fs,
                           mode="poly", split=-1, sync=True).cpu().numpy().astype(np.float64)
        r = oracle.simulate_rir(room, beta, src, rcv, nb, T, T, fs=fs)
        assert rel_err(g, r).max() <= TOL["poly"], (b, rel_err(g, r).max())


@pytest.mark.parametrize("fs", [8000.0, 22050.0, 44100.0, 96000.0])
def test_poly_sampling_rates(P, oracle, fs):
    """Integer and fractional half-windows H = Tw fs / 2 (16, 44.1, 88.2, 192 taps-half), zero-padded tap
    groups; random scenes against the oracle."""
    rng = np.random.default_rng(int(fs))
    for i in range(3):
        sc = W.random_small_scene(rng, fs=fs, T=0.03)
        beta, nb = derive(oracle, sc)
        g = run_gpu(P, sc, beta, nb, mode="poly", split=-1)  # small call: forced onto the polyphase kernel
        r = run_oracle(oracle, sc, beta, nb)
        assert rel_err(g, r).max() <= TOL["poly"], (fs, i)


def test_poly_matches_direct_kernel(P, oracle):
    """The two fp32 implementations of Eq. 5-6 (direct taps, polyphase) agree far inside the tolerance."""
    sc = W.cfg3(32, "diffuse")
    beta, nb = derive(oracle, sc)
    a = run_gpu(P, sc, beta, nb, mode="fp32")
    b = run_gpu(P, sc, beta, nb, mode="poly")
    assert rel_err(b, a).max() <= 5e-5


def test_poly_small_calls_cluster_kernel(P, oracle):
    """A lone RIR (config 1: 5 tiles) runs the polyphase kernel with each tile's columns split over a cluster of
    S CTAs (auto S = 16; forced 4 and 8 through opts.split), whose summed integer planes and per-output FIR
    reproduce the persistent kernel (split = -1) bit for bit; the oracle at the fp32 tolerance."""
    sc = W.cfg1()
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode="poly", split=-1)
    for split in (0, 4, 8, 16):
        assert np.array_equal(run_gpu(P, sc, beta, nb, mode="poly", split=split), ref), split
    assert not np.array_equal(run_gpu(P, sc, beta, nb, mode="fp32"), ref)
    assert rel_err(ref, run_oracle(oracle, sc, beta, nb))[0] <= TOL["poly"]


@pytest.mark.parametrize("case", ["cfg2_2.0", "cfg4a", "cfg3_16", "two_word_48k"])
def test_poly_cluster_matches_persistent(P, oracle, case):
    """Cluster items (small calls) and persistent items give the same bits: a tail-fused lone RIR (config 2,
    T60 = 2 s), the 48 kHz array (config 4 (a): 192 taps, runtime plane stride), 16 cardioid receivers, and a
    2 m cube at 48 kHz to 0.8 s whose late tiles take the two-word format (N >= 2^12)."""
    import torch
    if case == "two_word_48k":
        room = np.array([2.0, 2.0, 2.0], np.float32)
        src = torch.tensor([[0.7, 1.1, 0.9]], device="cuda")
        rcv = torch.tensor([[1.3, 0.6, 1.45]], device="cuda")
        T = 0.8
        nb = oracle.t2n(T, room, 343.0)
        beta = np.full(6, -0.95, np.float32)
        a, b, c = (P.simulate_rir(room, beta, src, rcv, nb, T, T, 48000.0, mode="poly", split=sp, sync=True).cpu().numpy()
                   for sp in (-1, 8, 0))  # 0: heavy tiles split into parts merged in global memory (two words)
        assert np.array_equal(a, b) and np.array_equal(a, c)
        return
    sc = {"cfg2_2.0": lambda: W.cfg2(2.0), "cfg4a": lambda: W.cfg4("a"), "cfg3_16": lambda: W.cfg3(16, "diffuse")}[case]()
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode="poly", split=-1)
    for split in (0, 4, 16):
        assert np.array_equal(run_gpu(P, sc, beta, nb, mode="poly", split=split), ref), split


@pytest.mark.parametrize("M", [16, 90])
def test_poly_split_plan_persistent_bit_identical(P, oracle, M):
    """Calls of at most two work items per SM split their heavy tiles' output ranges over the free CTA slots (one
    queue entry per part, 1024- or 512-thread persistent CTAs): 16 receivers (48 items) and 90 receivers (270
    items, item indices past 8 bits in the plan map) give the bits of the unsplit persistent call (split = -1),
    and the oracle at the fp32 tolerance."""
    sc = W.cfg3(M, "diffuse")
    beta, nb = derive(oracle, sc)
    ref = run_gpu(P, sc, beta, nb, mode="poly", split=-1)
    assert np.array_equal(run_gpu(P, sc, beta, nb, mode="poly"), ref)
    for m in (0, M - 1):
        r = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[m:m + 1], nb, sc.Tdiff, sc.Tmax, fs=sc.fs,
                                pattern=sc.pattern, orV_rcv=sc.orV_rcv[m:m + 1], seed=sc.seed, rir_index_base=m)
        assert rel_err(ref[:, m], r[:, 0]).max() <= TOL["poly"], m


def test_poly_parts_scratch_self_cleaning(P, oracle):
    """Small calls split their heavy tiles into parts whose integer planes meet in a global scratch slot that
    the last part zeroes again: back-to-back calls of different sizes and sampling rates on one stream (which
    reuse the ring's slots) reproduce their first results bit for bit."""
    cases = [W.cfg1(), W.cfg2(2.0), W.cfg4("a"), W.cfg2(0.7)]
    derived = [derive(oracle, sc) for sc in cases]
    first = [run_gpu(P, sc, b, n, mode="poly") for sc, (b, n) in zip(cases, derived)]
    for _ in range(3):
        for sc, (b, n), f in zip(cases, derived, first):
            assert np.array_equal(run_gpu(P, sc, b, n, mode="poly"), f), sc.name
    assert rel_err(first[0], run_oracle(oracle, cases[0], *derived[0]))[0] <= TOL["poly"]


@pytest.mark.parametrize("mode", ["poly", "fp32"])
def test_small_call_cuda_graph_replay(P, oracle, mode):
    """The call is stream-ordered and capturable: a lone-RIR call (config 1, and config 2 with its diffuse
    tail) captured into a CUDA graph and replayed gives the eager call's bits (the small-call latency path)."""
    import torch
    for sc in (W.cfg1(), W.cfg2(0.7)):
        beta, nb = derive(oracle, sc)
        src = torch.from_numpy(sc.pos_src).cuda()
        rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
        out = torch.empty((1, 1, P.nsamples(sc.Tmax, sc.fs)), device="cuda")
        call = lambda: P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, mode=mode,
                                      seed=sc.seed, out=out)
        call()
        torch.cuda.synchronize()
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            call()  # warm-up on the capture stream
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            call()
        for _ in range(3):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, ref), sc.name
        # several calls in one graph (how small calls amortise the graph launch): the scratch ring's slots are
        # taken in turn inside the capture; every call writes the same bits
        outs = [torch.empty_like(out) for _ in range(6)]
        g6 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g6):
            for o in outs:
                P.simulate_rir(sc.room, beta, src, rcv, nb, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c, mode=mode,
                               seed=sc.seed, out=o)
        for o in outs:
            o.zero_()
        g6.replay()
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o, ref), sc.name
        assert P.device_status() == 0


def test_trajectory_cuda_graph_replay(P):
    """The trajectory filter (tensor-core kernel with K shares and the ordered partial sum; CUDA-core kernel) is
    capturable after one eager call of its size: graph replays give the eager bits."""
    import torch
    g0 = torch.Generator(device="cuda").manual_seed(7)
    sig = torch.randn(6000, device="cuda", generator=g0)
    for shape, split in (((12, 32, 2000), 0), ((12, 32, 2001), 0), ((12, 32, 2000), -1)):
        rirs = torch.randn(shape, device="cuda", generator=g0)
        out = torch.empty((shape[1], 6000 + shape[2] - 1), device="cuda")
        call = lambda: P.simulate_trajectory(sig, rirs, out=out, split=split)
        call()
        torch.cuda.synchronize()
        ref = out.clone()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            call()
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            call()
        for _ in range(2):
            out.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, ref), (shape, split)


def test_concurrent_calls_on_many_streams(P, oracle):
    """Calls in flight on more streams than the library's scratch slots (4 for small polyphase calls' exchange,
    2 for the trajectory filter's partials): slot reuse is ordered by events, so every call equals its serial result."""
    import torch
    cases = [W.cfg1(), W.cfg2(2.0), W.cfg2(0.7), W.cfg1()]
    ref = []
    for sc in cases:
        b, n = derive(oracle, sc)
        ref.append(run_gpu(P, sc, b, n, mode="poly"))
    g = torch.Generator(device="cuda").manual_seed(5)
    sig = torch.randn(5000, device="cuda", generator=g)
    rirs = torch.randn((10, 8, 1200), device="cuda", generator=g)
    tref = P.simulate_trajectory(sig, rirs, sync=True).clone()
    streams = [torch.cuda.Stream() for _ in range(8)]
    outs, touts = [], []
    for rep in range(2):
        for i, st in enumerate(streams):
            sc = cases[i % len(cases)]
            b, n = derive(oracle, sc)
            with torch.cuda.stream(st):
                src = torch.from_numpy(sc.pos_src).cuda()
                rcv = torch.from_numpy(np.ascontiguousarray(sc.pos_rcv)).cuda()
                outs.append((i % len(cases), P.simulate_rir(sc.room, b, src, rcv, n, sc.Tdiff, sc.Tmax, sc.fs, c=sc.c,
                                                             mode="poly", seed=sc.seed, stream=st)))
                touts.append(P.simulate_trajectory(sig, rirs, stream=st))
    torch.cuda.synchronize()
    for k, h in outs:
        assert np.array_equal(h.cpu().numpy().astype(np.float64), ref[k])
    for y in touts:
        assert torch.equal(y, tref)
    assert P.device_status() == 0


def test_poly_cta_shapes_bit_identical(P, oracle):
    """A large call (256-thread CTAs) and its 8 shards (512-thread CTAs, too few work items for the small
    shape) give bit-identical RIRs: the aggregation is exact and each output's FIR arithmetic is fixed.  Both
    fuse the diffuse tail into the polyphase kernel (tiles end-aligned for every single-room call)."""
    sc = W.cfg3(1024, "diffuse")
    beta, nb = derive(oracle, sc)
    full = run_gpu(P, sc, beta, nb, mode="poly")
    parts = [run_gpu(P, sc, beta, nb, mode="poly", rir_index_base=128 * s, pos_rcv=sc.pos_rcv[128 * s:128 * (s + 1)],
                     orv=sc.orV_rcv[128 * s:128 * (s + 1)]) for s in range(8)]
    assert np.array_equal(full, np.concatenate(parts, axis=1))
    idx = [0, 511, 1023]
    for m in idx:
        rj = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[m:m + 1], nb, sc.Tdiff, sc.Tmax, fs=sc.fs,
                                 pattern=sc.pattern, orV_rcv=sc.orV_rcv[m:m + 1], seed=sc.seed, rir_index_base=m)
        assert rel_err(full[0, m], rj[0, 0])[0] <= TOL["poly"], m


def test_poly_count_guard_redo(P, oracle):
    """The polyphase overflow guard (poly_add): with the test hook split = -3 every tile's first pass has a
    count capacity of 4 images per sample position, so the guard fires on nearly every tile; a call whose
    512-thread CTAs hold the fine plane (64 receivers) redoes those tiles in the two-word format and must match
    the oracle at the fp32 tolerance, and its shards the whole call bit for bit (the format depends only on the
    tile's own images)."""
    sc = W.cfg3(64, "diffuse")
    beta, nb = derive(oracle, sc)
    g = run_gpu(P, sc, beta, nb, mode="poly", split=-3)
    for m in (0, 32, 63):  # each RIR keeps its global index (tail stream, reading C16)
        r = oracle.simulate_rir(sc.room, beta, sc.pos_src, sc.pos_rcv[m:m + 1], nb, sc.Tdiff, sc.Tmax, fs=sc.fs,
                                pattern=sc.pattern, orV_rcv=sc.orV_rcv[m:m + 1], seed=sc.seed, rir_index_base=m)
        assert rel_err(g[:, m], r[:, 0]).max() <= TOL["poly"], m
    part = run_gpu(P, sc, beta, nb, mode="poly", split=-3, rir_index_base=16, pos_rcv=sc.pos_rcv[16:48],
                   orv=sc.orV_rcv[16:48])
    assert np.array_equal(g[:, 16:48], part)


def test_poly_count_guard_capacity_status(P, oracle):
    """Where the redo has no room — 256-thread CTAs without the fine plane (1024 receivers, split = -3), or a
    two-word tile that fires (split = -5) — the call must fail loudly with GPURIR_ECAPACITY, never return a
    wrapped sum as a result; the status word is cleared afterwards."""
    beta = None
    for split, M in ((-3, 1024), (-5, 64)):
        sc = W.cfg3(M, "diffuse")
        beta, nb = derive(oracle, sc)
        with pytest.raises(P.GpurirError) as ei:
            run_gpu(P, sc, beta, nb, mode="poly", split=split)
        assert ei.value.status == P._lib.ECAPACITY, split
    assert P.device_status(reset=True) == 0


@pytest.mark.parametrize("fs,T", [(16000.0, 0.6), (48000.0, 0.3)])
def test_poly_worst_geometry_found(P, oracle, fs, T):
    """The geometry tests/test_poly_headroom.py's brute force found closest to the single-word capacity (35 %
    of it at 48 kHz): a 2 m cube, source at the centre, receiver 1 mm above it, rigid walls (beta = +-1: every
    image at full amplitude).  Polyphase (default path, no hooks) vs the oracle at the fp32 tolerance."""
    import torch
    room = np.array([2.0, 2.0, 2.0], np.float32)
    src = np.array([[1.0, 1.0, 1.0]], np.float32)
    rcv = np.array([[1.0, 1.0, 1.0 + 2.0 ** -10], [1.0, 1.0, 1.5]], np.float32)
    nb = oracle.t2n(T, room, 343.0)
    for b in (1.0, -1.0):
        beta = np.full(6, b, np.float32)
        g = P.simulate_rir(room, beta, torch.from_numpy(src).cuda(), torch.from_numpy(rcv).cuda(), nb, T, T, fs,
                           mode="poly", split=-1, sync=True).cpu().numpy().astype(np.float64)
        r = oracle.simulate_rir(room, beta, src, rcv, nb, T, T, fs=fs)
        assert rel_err(g, r).max() <= TOL["poly"], (b, rel_err(g, r).max())


@pytest.fixture(scope="module")
def curand_lib(tmp_path_factory):
    import ctypes
    import subprocess
    d = tmp_path_factory.mktemp("curand")
    so = str(d / "libcurand_stream.so")
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "curand_stream.cu")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                    "-Xcompiler", "-fPIC", "-o", so, src], check=True)
    L = ctypes.CDLL(so)
    L.curand_words.restype = ctypes.c_int
    L.curand_words.argtypes = [ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int,
                               ctypes.c_void_p]
    return L


@pytest.mark.parametrize("seed,r,k0", [(0, 0, 0), (0x5EED0003, 5, 8400), (0xFFFFFFFF12345678, 2**33 + 7, 2**32 - 6),
                                       (12345, 99999, 1)])
def test_tail_rng_is_curand_philox_stream(oracle, curand_lib, seed, r, k0):
    """The library special case of SURVEY §8(c)'s RNG row: the oracle's uniform u(seed, r, k) = (2 (w >> 9) + 1)
    2^-24 takes w = the k-th word of cuRAND's device API after curand_init(seed, subsequence = r, offset = 0)
    — pinning the counter layout (k >> 2 in the low, r in the high counter words), the key and the word order
    (x, y, z, w) against an implementation that is not ours.  Offsets k0 straddle a 2^32 counter carry."""
    import torch
    n = 64
    buf = torch.zeros((n,), dtype=torch.int32, device="cuda")
    assert curand_lib.curand_words(seed, r, k0, n, buf.data_ptr()) == 0
    w = buf.cpu().numpy().view(np.uint32).astype(np.uint64)
    u_curand = (2.0 * (w >> np.uint64(9)).astype(np.float64) + 1.0) / 16777216.0
    u_oracle = np.array([oracle.uniform(seed, r, k0 + i) for i in range(n)])
    assert np.array_equal(u_curand, u_oracle)


def test_cfg5_two_ranks_through_the_library(P, tmp_path):
    """SURVEY §8(e) through the library, not the oracle: config-5 rooms LPT-sharded over 2 ranks (two processes
    on cuda:0, torch.distributed gloo, one batch call per rank) and gathered to rank 0 equal the 1-rank call
    bit for bit (polyphase; every room keeps its global rir_index)."""
    import socket
    import subprocess
    import sys
    import torch
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import shard_worker
    rb, rooms, costs, ns = shard_worker.rooms_of(P, W, 600)
    one = [dict(r, out_offset=int(sum(ns[:i]))) for i, r in enumerate(rooms)]
    for r in one:
        r.pop("n")
    ref = torch.empty((int(sum(ns)),), device="cuda")
    P.simulate_rir_batch(one, rb.fs, ref, seed=rb.seed, mode="poly", sync=True)
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    out = str(tmp_path / "two_ranks.npy")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                                  "shard_worker.py"), "--out", out]
    subprocess.run(cmd, check=True, timeout=600)
    got = np.load(out)
    assert np.array_equal(got, ref.cpu().numpy())
