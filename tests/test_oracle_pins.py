"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a closed form of the paper's
equations, a value printed in SPEC.md / SURVEY.md (tests/golden/), an
independent algorithm (mirror BFS, ray unfolding, numpy's sinc), an invariant
(reciprocity, completeness, dense == support-restricted), or a statistical law.
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- helpers (A17-A19, Eq. 7)

def test_spec_helper_examples(oracle):
    g = _load("spec_examples.json")
    for e in g["sabine"]:
        T = oracle.sabine_t60(e["room"], [e["beta_abs"]] * 6)
        assert abs(T - e["T60"]) <= e["tol"], e
        assert oracle.sabine_t60(e["room"], [-e["beta_abs"]] * 6) == T  # sign invariance
    e = g["beta_from_t60"]
    b, cl = oracle.beta_sabine(e["room"], e["T60"])
    assert not cl and np.all(b < 0) and abs(abs(b[0]) - e["beta_abs"]) < e["tol"]
    e = g["beta_infeasible"]
    with pytest.raises(oracle.OracleError) as ei:
        oracle.beta_sabine(e["room"], e["T60"])
    assert ei.value.status == 3
    b, cl = oracle.beta_sabine(e["room"], e["T60"], clamp=True)
    assert cl and np.all(b == 0)
    for e in g["att2t"]:
        assert oracle.att2t(e["att"], e["T60"]) == pytest.approx(e["t"], abs=1e-15)
    e = g["t2n"]
    assert oracle.t2n(e["t"], [e["L"]] * 3)[0] == e["N"]
    # S:356 claims t -> 0+ gives (3,3,3), but its own rule gives 2(ceil(0+)+1)+1 = 5: the rule wins
    # (reading R-t2n).
    assert list(oracle.t2n(1e-9, [3, 4, 2.5])) == [5, 5, 5]


def test_sabine_round_trip(oracle):
    rng = np.random.default_rng(0)
    for _ in range(1000):
        room = rng.uniform(2, 10, 3)
        V, S = np.prod(room), 2 * (room[0] * room[1] + room[0] * room[2] + room[1] * room[2])
        Tmin = 0.161 * V / S
        T = rng.uniform(Tmin * 1.01, 3.0)
        b, _ = oracle.beta_sabine(room, T, sign=int(rng.choice([-1, 1])))
        assert abs(oracle.sabine_t60(room, b) - T) / T < 1e-9


def test_t2n_monotone(oracle):
    room = [3.0, 4.0, 2.5]
    prev = oracle.t2n(0.01, room)
    for T in np.linspace(0.02, 2.0, 60):
        cur = oracle.t2n(T, room)
        assert np.all(cur >= prev) and np.all(cur % 2 == 1)
        prev = cur


# ---------------------------------------------------------------- Eq. 1, crossing rule

def test_spec_geometry_examples(oracle):
    g = _load("spec_examples.json")
    for e in g["image_position"]:
        assert oracle.image_coord(e["n"], e["L"], e["s"]) == e["x"]
    for e in g["wall_crossings"]:
        assert list(oracle.wall_crossings(e["n"])) == e["c"]


def test_wall_crossings_vs_ray_unfolding(oracle):
    """P:109 prose ("each wall crossed"): count the unfolded boundary planes x = jL the straight
    path from image cell n to the receiver cell 0 crosses; plane j is wall 0 (j even) or wall 1 (j odd)."""
    for n in range(-50, 51):
        js = range(1, n + 1) if n > 0 else range(n + 1, 1)
        c0 = sum(1 for j in js if j % 2 == 0)
        c1 = sum(1 for j in js if j % 2 != 0)
        assert oracle.wall_crossings(n) == (c0, c1), n


def _mirror_bfs(room, beta, src, order):
    """Independent image generator: breadth-first mirror reflections of the source across the six
    faces of each image room (SURVEY §8(c) pin "image set = brute-force mirror enumeration").
    Returns {n: (position, beta product)} with n the image-room index per axis.  An image room is
    first reached by a shortest reflection sequence (the straight-line path of the image); longer
    sequences that revisit a room (reflecting back across a plane) are not physical paths and are
    ignored, while all shortest sequences to a room must agree."""
    L = np.asarray(room, float)
    start = (tuple(np.asarray(src, float)), (0, 0, 0), (False, False, False), 1.0)
    seen = {(0, 0, 0): (np.asarray(src, float), 1.0, 0, (False, False, False))}
    frontier = [start]
    for depth in range(1, order + 1):
        nxt = []
        for pos, cell, flipped, bprod in frontier:
            for ax in range(3):
                for side in (0, 1):  # 0 = low face of the image room, 1 = high face
                    lo = cell[ax] * L[ax]
                    plane = lo if side == 0 else lo + L[ax]
                    newpos = list(pos)
                    newpos[ax] = 2 * plane - pos[ax]
                    newcell = list(cell)
                    newcell[ax] += -1 if side == 0 else 1
                    # physical wall behind this face: low face is wall 0 unless the image room is flipped
                    wall = side if not flipped[ax] else 1 - side
                    nb = bprod * beta[2 * ax + wall]
                    nf = list(flipped)
                    nf[ax] = not nf[ax]
                    key = tuple(newcell)
                    if key in seen:
                        assert np.allclose(seen[key][0], newpos)
                        if seen[key][2] == depth:
                            assert abs(seen[key][1] - nb) < 1e-12
                        continue
                    seen[key] = (np.asarray(newpos), nb, depth, tuple(nf))
                    nxt.append((tuple(newpos), key, tuple(nf), nb))
        frontier = nxt
    return seen


@pytest.mark.parametrize("nb", [(3, 4, 5), (5, 5, 5), (6, 3, 7)])
def test_image_set_vs_mirror_bfs(oracle, nb):
    room = [3.0, 4.0, 2.5]
    beta = [-0.9, 0.8, -0.7, 0.95, 0.6, -0.85]
    src, rcv = [0.7, 1.3, 0.9], [2.2, 3.1, 1.7]
    fs, c = 16000.0, 343.0
    imgs = oracle.image_set(room, beta, src, rcv, nb, fs=fs, c=c)
    order = sum(int(math.ceil(N / 2)) for N in nb) + 3
    bfs = _mirror_bfs(room, beta, src, order)
    assert len(imgs["x"]) == int(np.prod(nb))
    for n, x, bn in zip(imgs["n"], imgs["x"], imgs["beta"]):
        pos, bprod = bfs[tuple(int(v) for v in n)][:2]
        d = np.linalg.norm(pos - np.asarray(rcv))
        assert abs(x - d / c * fs) < 1e-9
        assert abs(bn - bprod) < 1e-12


@pytest.mark.parametrize("spkr,mic", [(2, 0), (4, 3), (1, 2)])
def test_source_directivity_vs_mirror_bfs(oracle, spkr, mic):
    """f3 (reading R10): every image source carries the source orientation mirrored by the reflections that
    produced it (tracked independently by the BFS as flipped axes) and radiates along p_r - p_n, so
    A_n = beta_n g_r g_s / (4 pi d_n) with g_s = a_s + (1 - a_s) cos(theta_s)."""
    room = [3.0, 4.0, 2.5]
    beta = [-0.9, 0.8, -0.7, 0.95, 0.6, -0.85]
    src, rcv = [0.7, 1.3, 0.9], [2.2, 3.1, 1.7]
    os_, orv = np.array([0.3, -0.5, 0.8]), np.array([-0.6, 0.2, 0.4])
    nb = (5, 4, 5)
    a = {0: 1.0, 1: 0.75, 2: 0.5, 3: 0.25, 4: 0.0}
    imgs = oracle.image_set(room, beta, src, rcv, nb, pattern=mic, orv=orv, spkr_pattern=spkr, ors=os_)
    bfs = _mirror_bfs(room, beta, src, sum(int(math.ceil(N / 2)) for N in nb) + 3)
    us, ur = os_ / np.linalg.norm(os_), orv / np.linalg.norm(orv)
    for n, A in zip(imgs["n"], imgs["A"]):
        pos, bprod, _, flipped = bfs[tuple(int(v) for v in n)]
        o_img = np.where(flipped, -us, us)  # the orientation reflected with the source
        d = np.linalg.norm(pos - np.asarray(rcv))
        gs = a[spkr] + (1 - a[spkr]) * np.dot(o_img, np.asarray(rcv) - pos) / d
        gr = a[mic] + (1 - a[mic]) * np.dot(ur, pos - np.asarray(rcv)) / d
        assert abs(A - bprod * gs * gr / (4 * math.pi * d)) < 1e-13


def test_source_directivity_reflection_point(oracle):
    """f3: a first-order reflection off wall x0 leaves the source toward the specular point on x = 0, found
    by intersecting the receiver -> image line with the wall plane (no image arithmetic involved)."""
    room, src, rcv = [5.0, 4.0, 3.0], np.array([1.5, 1.2, 1.0]), np.array([3.5, 2.9, 1.8])
    beta = [1.0, 0.0, 0.0, 0.0, 0.0, 0.0]  # only the direct path and the x0 reflection survive
    o = np.array([-1.0, 0.2, 0.1])
    im = oracle.image_set(room, beta, src, rcv, [3, 1, 1], spkr_pattern=2, ors=o)
    uo = o / np.linalg.norm(o)
    mirror = np.array([-src[0], src[1], src[2]])
    t = rcv[0] / (rcv[0] - mirror[0])                  # receiver -> image line meets x = 0
    q = rcv + t * (mirror - rcv)
    dep = (q - src) / np.linalg.norm(q - src)
    d = np.linalg.norm(rcv - mirror)
    want = {(-1, 0, 0): (0.5 + 0.5 * np.dot(uo, dep)) / (4 * math.pi * d),
            (0, 0, 0): (0.5 + 0.5 * np.dot(uo, (rcv - src) / np.linalg.norm(rcv - src)))
            / (4 * math.pi * np.linalg.norm(rcv - src)),
            (1, 0, 0): 0.0}
    for n, A in zip(im["n"], im["A"]):
        assert A == pytest.approx(want[tuple(int(v) for v in n)], abs=1e-15)


def test_source_pattern_special_cases(oracle):
    """f3, beta = 0: direct path only, g_s from the angle between the source axis and r - s (cardioid
    1 toward / 0 away, bidirectional 0 broadside, hypercardioid a = 0.25 broadside)."""
    room, src, rcv = [10.0, 10.0, 10.0], [2.0, 5.0, 5.0], [5.0, 5.0, 5.0]
    cases = [(2, [1, 0, 0], 1.0), (2, [-1, 0, 0], 0.0), (4, [0, 0, 1], 0.0), (3, [0, 1, 0], 0.25),
             (1, [-1, 0, 0], 0.5)]
    for pat, o, g in cases:
        im = oracle.image_set(room, [0.0] * 6, src, rcv, [1, 1, 1], spkr_pattern=pat, ors=o)
        assert im["A"][0] == pytest.approx(g / (4 * math.pi * 3.0), abs=1e-15)


def test_directional_reciprocity(oracle):
    """f3: swapping source and receiver together with their patterns and orientations gives an identical
    RIR (odd N, non-uniform walls): the arrival direction of one is the departure direction of the other."""
    room = [3.0, 4.0, 2.5]
    beta = np.array([-0.9, 0.8, -0.7, 0.95, 0.6, -0.85])
    nb = oracle.t2n(0.05, room)
    s, r = [1.2, 1.5, 1.1], [2.1, 2.9, 1.4]
    oa, ob = [0.3, -0.5, 0.8], [-0.6, 0.2, 0.4]
    h1 = oracle.simulate_rir(room, beta, [s], [r], nb, 0.05, 0.05, pattern=3, orV_rcv=[ob], spkr_pattern=2,
                             orV_src=[oa])
    h2 = oracle.simulate_rir(room, beta, [r], [s], nb, 0.05, 0.05, pattern=2, orV_rcv=[oa], spkr_pattern=3,
                             orV_src=[ob])
    h0 = oracle.simulate_rir(room, beta, [s], [r], nb, 0.05, 0.05)
    assert np.max(np.abs(h1 - h2)) < 1e-12 * np.max(np.abs(h1))
    assert np.max(np.abs(h1 - h0)) > 1e-2 * np.max(np.abs(h0))  # the patterns do change the RIR


def test_weighted_beta_sabine(oracle):
    """f3 (reading R9): non-uniform absorption weights meet Sabine's T60 exactly (Eq. 7), keep the
    absorption ratios alpha_i / alpha_j = w_i / w_j, reduce to the uniform helper for equal weights, and
    report infeasibility when a wall would need alpha > 1."""
    rng = np.random.default_rng(9)
    for _ in range(200):
        room = rng.uniform(2, 10, 3)
        w = rng.uniform(0.1, 1.0, 6)
        T = rng.uniform(0.5, 3.0)
        try:
            b, _ = oracle.beta_sabine_weighted(room, T, w)
        except oracle.OracleError as e:
            assert e.status == 3
            continue
        assert abs(oracle.sabine_t60(room, b) - T) / T < 1e-12
        al = 1 - b ** 2
        assert np.allclose(al / al[0], w / w[0], rtol=1e-12)
        assert np.all(b <= 0)
    room = [3.0, 4.0, 2.5]
    bu, _ = oracle.beta_sabine(room, 0.7)
    bw, _ = oracle.beta_sabine_weighted(room, 0.7, [2.0] * 6)
    assert np.allclose(bu, bw, rtol=0, atol=1e-15)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.beta_sabine_weighted(room, 0.2, [1, 1, 1, 1, 1, 20])
    assert ei.value.status == 3
    b, cl = oracle.beta_sabine_weighted(room, 0.2, [1, 1, 1, 1, 1, 20], clamp=True)
    assert cl and np.all(b == 0)
    bz, _ = oracle.beta_sabine_weighted(room, 0.7, [1, 1, 0, 0, 1, 1])  # y walls reflect perfectly
    assert bz[2] == -1.0 and bz[3] == -1.0


def test_image_amp_example(oracle):
    """S:90 (Eqs. 2-4): n = 0, beta = 1, src (1,1,1), rcv (2,1,1) -> tau = 1/343 s, A = 1/(4 pi)."""
    im = oracle.image_set([3, 4, 2.5], [1.0] * 6, [1, 1, 1], [2, 1, 1], [1, 1, 1], fs=16000.0, c=343.0)
    assert im["x"][0] == pytest.approx(16000.0 / 343.0, rel=1e-15)
    assert im["A"][0] == pytest.approx(1.0 / (4 * math.pi), rel=1e-15)


def test_polar_pattern_special_cases(oracle):
    """A16 / S:99-101: cardioid null at 180 deg, hypercardioid 0.25 at 90 deg, bidirectional 0 at 90 deg."""
    room, src, rcv = [10.0, 10.0, 10.0], [2.0, 5.0, 5.0], [5.0, 5.0, 5.0]
    # direct path arrives from -x (image - receiver = (-3, 0, 0))
    cases = [(2, [1, 0, 0], 0.0), (2, [-1, 0, 0], 1.0), (3, [0, 1, 0], 0.25), (4, [0, 0, 1], 0.0), (1, [1, 0, 0], 0.5)]
    for pat, o, g in cases:
        im = oracle.image_set(room, [0.0] * 6, src, rcv, [1, 1, 1], pattern=pat, orv=o)
        assert im["A"][0] == pytest.approx(g / (4 * math.pi * 3.0), abs=1e-15)


# ---------------------------------------------------------------- Eq. 6 and the RIR sum

def _eq6_numpy(u, H):
    """Eq. 6 in samples via numpy's normalised sinc (sin(pi u)/(pi u)), independent of the oracle."""
    u = np.asarray(u, float)
    w = 0.5 * (1 + np.cos(np.pi * u / H))
    return np.where(np.abs(u) < H, w * np.sinc(u), 0.0)


def test_windowed_sinc_closed_forms(oracle):
    g = _load("spec_examples.json")["windowed_sinc_half_sample_16k"]
    v = oracle.windowed_sinc(0.5 / 16000, 4e-3, 8000.0)
    assert abs(v - g["value"]) < g["tol"]
    assert v == pytest.approx(0.5 * (1 + math.cos(math.pi / 64)) * 2 / math.pi, rel=1e-14)
    assert oracle.windowed_sinc(0.0) == 1.0
    assert oracle.windowed_sinc(2e-3) == 0.0 and oracle.windowed_sinc(-2e-3) == 0.0
    for t in np.random.default_rng(1).uniform(-2.2e-3, 2.2e-3, 200):
        assert oracle.windowed_sinc(t) == pytest.approx(float(_eq6_numpy(t * 16000, 32.0)), abs=1e-14)


def test_direct_path_beta0(oracle):
    """north_star pin: beta = 0 leaves only the direct path, amplitude 1/(4 pi d) at delay d/c."""
    room, src, rcv = [3.0, 4.0, 2.5], [1.0, 1.0, 1.0], [2.0, 3.0, 1.5]
    fs, c = 16000.0, 343.0
    im = oracle.image_set(room, [0.0] * 6, src, rcv, [9, 9, 9], fs=fs, c=c)
    nz = np.nonzero(im["A"])[0]
    assert len(nz) == 1 and tuple(im["n"][nz[0]]) == (0, 0, 0)
    d = math.sqrt(1 + 4 + 0.25)
    assert im["A"][nz[0]] == pytest.approx(1 / (4 * math.pi * d), rel=1e-14)
    h = oracle.simulate_rir(room, [0.0] * 6, [src], [rcv], [9, 9, 9], 0.02, 0.02, fs=fs, c=c)[0, 0]
    k = np.arange(h.size)
    ref = _eq6_numpy(k - d / c * fs, 32.0) / (4 * math.pi * d)
    assert np.max(np.abs(h - ref)) < 1e-15


@pytest.mark.parametrize("xs, expect", [(100.0, {100: 1.0}), (100.5, {100: 0.6362363541693464, 101: 0.6362363541693464})])
def test_single_image_render(oracle, xs, expect):
    """one image at tau = 100/fs -> h[100] = A, 0 elsewhere; at 100.5/fs -> h[100] = h[101] = 0.63624 A."""
    fs, c = 16000.0, 343.0
    d = xs * c / fs
    src, rcv = [1.0, 2.0, 1.25], [1.0 + d, 2.0, 1.25]
    h = oracle.simulate_rir([5.0, 4.0, 2.5], [0.0] * 6, [src], [rcv], [3, 3, 3], 0.02, 0.02, fs=fs, c=c)[0, 0]
    A = 1 / (4 * math.pi * d)
    for k, v in expect.items():
        assert h[k] == pytest.approx(A * v, rel=1e-12)
    if xs == int(xs):  # integer delay: every other sample sits on a sinc zero
        for k in range(h.size):
            if k not in expect:
                assert abs(h[k]) < 1e-12 * A, k
    ref = _eq6_numpy(np.arange(h.size) - xs, 32.0) * A
    assert np.max(np.abs(h - ref)) < 1e-12 * A


def test_dense_equals_support(oracle):
    """P:208's dense formulation (every sample of every image) equals the support-restricted loop."""
    room, beta = [3.0, 4.0, 2.5], [-0.9, 0.8, -0.7, 0.95, 0.6, -0.85]
    for fs in (16000.0, 48000.0):
        a = oracle.simulate_rir(room, beta, [[0.7, 1.3, 0.9]], [[2.2, 3.1, 1.7], [1.1, 0.4, 2.0]], [5, 6, 5], 0.03,
                                0.03, fs=fs, dense=False)
        b = oracle.simulate_rir(room, beta, [[0.7, 1.3, 0.9]], [[2.2, 3.1, 1.7], [1.1, 0.4, 2.0]], [5, 6, 5], 0.03,
                                0.03, fs=fs, dense=True)
        assert np.max(np.abs(a - b)) < 1e-14 * np.max(np.abs(a))


def test_reciprocity(oracle):
    """north_star pin: swapping source and receiver (omni, odd N) gives an identical RIR."""
    room = [3.0, 4.0, 2.5]
    beta, _ = oracle.beta_sabine(room, 0.3)
    nb = oracle.t2n(0.1, room)
    s, r = [1.2, 1.5, 1.1], [2.1, 2.9, 1.4]
    h1 = oracle.simulate_rir(room, beta, [s], [r], nb, 0.1, 0.1)
    h2 = oracle.simulate_rir(room, beta, [r], [s], nb, 0.1, 0.1)
    assert np.max(np.abs(h1 - h2)) < 1e-12 * np.max(np.abs(h1))


def test_lattice_completeness(oracle):
    """C6: the t2n grid already holds every image reaching T; enlarging N by 4 per axis changes nothing."""
    room = [3.0, 4.0, 2.5]
    beta, _ = oracle.beta_sabine(room, 0.5)
    for T in (0.05, 0.08):
        nb = oracle.t2n(T, room)
        a = oracle.simulate_rir(room, beta, [[0.4, 3.5, 2.2]], [[2.7, 0.3, 0.2]], nb, T, T)
        b = oracle.simulate_rir(room, beta, [[0.4, 3.5, 2.2]], [[2.7, 0.3, 0.2]], nb + 4, T, T)
        assert np.max(np.abs(a - b)) == 0.0


@pytest.mark.parametrize("case", ["G1", "G2", "G3", "G4"])
def test_cross_implementation_goldens(oracle, case):
    g = _load("survey_appendix_b.json")["cases"][case]
    T = g["nS"] / g["fs"]
    h = oracle.simulate_rir(g["room"], g["beta"], [g["src"]], [g["rcv"]], g["nb"], T, T, fs=g["fs"],
                            pattern=g["pattern"], orV_rcv=None if g["orv"] is None else [g["orv"]])[0, 0]
    assert h.size == g["nS"]
    assert int(np.argmax(np.abs(h))) == g["argmax"]
    assert h[g["argmax"]] == pytest.approx(g["h_argmax"], rel=1e-9)
    assert h.sum() == pytest.approx(g["sum"], rel=1e-9, abs=1e-15)
    assert (h * h).sum() == pytest.approx(g["sum2"], rel=1e-9)
    for k, v in g["spot"].items():
        assert h[int(k)] == pytest.approx(v, rel=1e-8, abs=1e-15)


# ---------------------------------------------------------------- Eq. 7-8 decay, tail

def _edc_db(h):
    e = np.cumsum((h[::-1] ** 2))[::-1]
    return 10 * np.log10(e / e[0])


def _fit_t60(h, fs, hi_db, lo_db):
    edc = _edc_db(h)
    idx = np.nonzero((edc <= hi_db) & (edc >= lo_db))[0]
    t = idx / fs
    slope = np.polyfit(t, edc[idx], 1)[0]
    return -60.0 / slope


def test_energy_decay_ism_only_vs_sabine(oracle):
    """north_star pin: ISM-only energy-decay slope matches Sabine T60 within 10% (negative beta, SURVEY A-7)."""
    room = [3.0, 4.0, 2.5]
    beta, _ = oracle.beta_sabine(room, 0.3)
    nb = oracle.t2n(0.3, room)
    h = oracle.simulate_rir(room, beta, [[1.2, 1.5, 1.1]], [[2.1, 2.9, 1.4]], nb, 0.3, 0.3)[0, 0]
    T20 = _fit_t60(h, 16000.0, -5.0, -25.0)
    assert abs(T20 / 0.3 - 1) < 0.10, T20


def test_full_pipeline_decay_vs_sabine(oracle):
    """Eqs. 7-8 + P:160: ISM to T60/4 plus logistic tail to T60; EDC slope within 10% of Sabine."""
    room = [6.0, 4.0, 3.0]
    for T60 in (0.3, 0.7):
        beta, _ = oracle.beta_sabine(room, T60)
        nb = oracle.t2n(T60 / 4, room)
        h = oracle.simulate_rir(room, beta, [[2.0, 1.5, 1.2]], [[4.1, 2.9, 1.6]], nb, T60 / 4, T60, seed=7)[0, 0]
        T30 = _fit_t60(h, 16000.0, -5.0, -35.0)
        assert abs(T30 / T60 - 1) < 0.10, (T60, T30)


def test_tail_envelope_slope(oracle):
    """the tail envelope decays at -60/T60 dB/s (block-energy regression, 8 independent channels)."""
    room, T60, fs = [6.0, 4.0, 3.0], 0.7, 16000.0
    beta, _ = oracle.beta_sabine(room, T60)
    nb = oracle.t2n(T60 / 4, room)
    rcv = [[4.1, 2.9, 1.6]] * 8
    h = oracle.simulate_rir(room, beta, [[2.0, 1.5, 1.2]], rcv, nb, T60 / 4, T60, seed=11)[0]
    nISM = oracle.nsamples(T60 / 4, fs)
    tail = h[:, nISM:]
    B = 160
    nb_ = tail.shape[1] // B
    e = (tail[:, : nb_ * B] ** 2).reshape(8, nb_, B).mean(axis=(0, 2))
    t = (nISM + B * np.arange(nb_) + B / 2) / fs
    slope = np.polyfit(t, 10 * np.log10(e), 1)[0]
    assert abs(slope / (-60.0 / T60) - 1) < 0.05, slope
    # channels are independent draws
    cc = np.corrcoef(tail[0], tail[1])[0, 1]
    assert abs(cc) < 0.05


def test_tail_silent_when_no_early_part(oracle):
    """S:293 / §8(b): Tdiff = 0 leaves the estimation window empty -> A_env = 0 -> silent tail."""
    h = oracle.simulate_rir([3, 4, 2.5], [-0.9] * 6, [[1, 1, 1]], [[2, 3, 1.5]], [5, 5, 5], 0.0, 0.05)
    assert np.all(h == 0.0)


def test_tail_power_continuity(oracle):
    """C15 exact averaging: expected tail power just after Tdiff equals the ISM power just before it
    (ratio of mean h^2 over 10 ms on each side ~ exp(-kappa * 10 ms), SURVEY A-10)."""
    room, T60, fs = [6.0, 4.0, 3.0], 1.0, 16000.0
    beta, _ = oracle.beta_sabine(room, T60)
    nb = oracle.t2n(T60 / 4, room)
    h = oracle.simulate_rir(room, beta, [[2.0, 1.5, 1.2]], [[4.1, 2.9, 1.6]] * 16, nb, T60 / 4, T60, seed=3)[0]
    n = oracle.nsamples(T60 / 4, fs)
    before = np.mean(h[0, n - 160:n] ** 2)
    after = np.mean(h[:, n:n + 160] ** 2)
    expect = math.exp(-6 * math.log(10) / T60 * 0.010)
    assert abs(after / before / expect - 1) < 0.15


# ---------------------------------------------------------------- RNG (C16)

def test_philox_known_answers(oracle):
    """Random123 Philox4x32-10 KAT vectors (the generator behind cuRAND's curand_init/curand)."""
    kat = [([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
           ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
           ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
            [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]
    for ctr, key, out in kat:
        assert oracle.philox4x32_10(ctr, key).tolist() == out


def test_uniform_open_interval(oracle):
    for k in range(0, 4000, 7):
        u = oracle.uniform(0x5EED0003, 12345, k)
        assert 0.0 < u < 1.0
        m = u * 2 ** 24
        assert m == int(m) and int(m) % 2 == 1


def test_uniform_is_curand_device_stream(oracle):
    """The counter / key / word layout of oracle_uniform (reading C16) against cuRAND itself: P:223 draws the
    tail noise with cuRAND, and tests/golden/curand_philox4x32_10.txt holds words of cuRAND's device-API stream
    (curand_init(seed, subsequence = r, offset = k0), then curand()) written on a B200 box by
    tools/gen_curand_golden.py, which calls only cuRAND.  A swapped (k, r) counter, a reversed word order or a
    wrong key half fails here; offsets straddle a 2^32 counter carry (r = 2^33 + 7, k near 2^32)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "curand_philox4x32_10.txt")
    rows = [tuple(int(v) for v in line.split()) for line in open(path) if line.strip() and not line.startswith("#")]
    assert len(rows) >= 60
    for seed, r, k, w in rows:
        assert oracle.uniform(seed, r, k) == (2.0 * (w >> 9) + 1.0) / 16777216.0, (seed, r, k)


def test_logistic_moments(oracle):
    """1e6 unit-variance logistic draws: mean within +-0.005, variance 1 +- 0.05."""
    x = oracle.logistic_stream(0x5EED0002, 9, 0, 10 ** 6)
    assert abs(x.mean()) < 0.005
    assert abs(x.var() - 1.0) < 0.05


# ---------------------------------------------------------------- Eq. 9 LUT, Eqs. 10-11 polynomials

def test_lut_pins(oracle):
    for fs, n_expect in ((16000.0, 1025), (48000.0, 3073)):
        lut, half = oracle.lut_build(4e-3, fs, 16)
        assert lut.size == n_expect
        assert lut[half] == 1.0 and lut[0] == 0.0 and lut[-1] == 0.0
        assert np.allclose(lut, lut[::-1], atol=1e-15)
        mult = np.arange(-half, half + 1) % 16 == 0
        mult[half] = False
        assert np.max(np.abs(lut[mult])) < 1e-15  # sinc zeros at whole samples
        H = 4e-3 * fs / 2
        t = np.random.default_rng(2).uniform(-H, H, 20000) / fs
        err = max(abs(oracle.lut_lookup(lut, half, 16, fs, ti) - float(_eq6_numpy(ti * fs, H))) for ti in t)
        assert err <= 2e-3  # S:189; SURVEY A-8 measured 1.60e-3


def test_sin_cos_polynomials(oracle):
    g = _load("spec_examples.json")["sin_pi_poly"]
    assert oracle.sin_pi_poly(g[0]["x"]) == g[0]["value"]
    assert abs(oracle.sin_pi_poly(g[1]["x"]) - g[1]["value"]) < g[1]["tol"]
    xs = np.linspace(-0.5, 0.5, 100001)
    es = max(abs(oracle.sin_pi_poly(x) - math.sin(math.pi * x)) for x in xs[::10])
    ec = max(abs(oracle.cos_pi_poly(x) - math.cos(math.pi * x)) for x in xs[::10])
    assert es < 3e-4 and ec < 1e-4  # SURVEY A-2: 2.82e-4 and 9.21e-5
    for x in np.linspace(-4, 4, 801):
        s = oracle.sin_pi_poly(x)
        assert s == -oracle.sin_pi_poly(-x)
        if abs(math.sin(math.pi * x)) > 1e-3:
            assert np.sign(s) == np.sign(math.sin(math.pi * x))
    # printed coefficients are exactly representable in fp16
    for c in (2.326171875, -5.14453125, 3.140625, -1.2294921875, 4.04296875, -4.93359375):
        assert float(np.float16(c)) == c


# ---------------------------------------------------------------- NEXT f1: trajectory filtering

def test_trajectory_single_point_equals_numpy_convolve(oracle):
    """One trajectory point: plain filtering, pinned by numpy's convolution (library routine)."""
    rng = np.random.default_rng(8)
    sig = rng.standard_normal(1001)
    rirs = rng.standard_normal((1, 3, 257))
    out = oracle.simulate_trajectory(sig, rirs)
    for m in range(3):
        assert np.allclose(out[m], np.convolve(sig, rirs[0, m]), rtol=0, atol=1e-11)


def test_trajectory_impulses_and_segments(oracle):
    """S:396-397 impulse RIRs give identity / delay; S:406 identical RIRs on every point = single point;
    S:407 scaled impulse scales the output; segment p uses point p's bank (remainder to the last)."""
    rng = np.random.default_rng(9)
    sig = rng.standard_normal(103)
    L = 9
    rir = np.zeros((1, 2, L)); rir[0, 0, 0] = 1.0; rir[0, 1, 4] = 0.5
    out = oracle.simulate_trajectory(sig, rir)
    assert np.array_equal(out[0, :103], sig) and np.all(out[0, 103:] == 0)
    assert np.allclose(out[1, 4:107], 0.5 * sig, atol=0)
    same = np.repeat(rng.standard_normal((1, 2, L)), 5, axis=0)
    assert np.allclose(oracle.simulate_trajectory(sig, same), oracle.simulate_trajectory(sig, same[:1]), atol=1e-12)
    # 103 samples, 5 points: segments of 20, last one 23 samples; point p = delta at delay p
    rir5 = np.zeros((5, 1, L))
    for p in range(5):
        rir5[p, 0, p] = 1.0
    out5 = oracle.simulate_trajectory(sig, rir5)[0]
    ref = np.zeros(103 + L - 1)
    for j in range(103):
        ref[j + min(j // 20, 4)] += sig[j]
    assert np.array_equal(out5, ref)
