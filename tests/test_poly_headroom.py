"""Headroom of the polyphase kernel's single-word fixed point (reading R11) — host logic, CPU.

The kernel adds every image's channel values v = round(A T_d 2^s), |v| <= 2^bits, into one int32 word per
sample position, with bits = min(22, 30 - ceil(log2 N)) and N = 8 pi x_hi^2 / V_s + 24 x_hi / L_min + 16 from
the tile's largest delay x_hi, the room volume V_s and its shortest side L_min (all in samples).  N is an
ESTIMATE of the images sharing one sample: the number of lattice points on a sphere is not bounded by any
fixed multiple of its mean (for a cube with source and receiver at its centre it is r3(n), which grows like
sqrt(n) log log n), so correctness does not rest on it: every deposit also counts itself in the last channel's
low bits and a tile whose count reaches the capacity 2^(31 - bits) is redone wider (ism_poly_kernel.cu,
poly_add; the GPU tests force that path).  These tests measure how much of the capacity real geometries use —
i.e. how rarely the redo runs — by brute force (tests/headroom_count.c, every lattice image of Eq. 1 within
the delay) up to the LONGEST delay the single-word format covers (N < 2^12) in each room, at 16 and 48 kHz,
with bits taken for the smallest tile that can hold the sample (x_hi = j + 1, the least headroom).
"""
import math
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "headroom_count.c")


@pytest.fixture(scope="module")
def counter(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("headroom") / "headroom_count")
    subprocess.run(["gcc", "-O3", "-fopenmp", "-o", exe, SRC, "-lm"], check=True)
    return exe


def image_delay_counts(exe, L, s, r, fs, T, c=343.0):
    """Number of images (every lattice point of Eq. 1 within T c) per integer delay floor(d fs / c)."""
    out = subprocess.run([exe, *map(repr, map(float, L)), *map(repr, map(float, s)), *map(repr, map(float, r)),
                          repr(float(fs)), repr(float(T)), repr(float(c))], check=True, capture_output=True,
                         text=True).stdout
    a = np.array([[int(v) for v in line.split()] for line in out.splitlines() if line], dtype=np.int64)
    cnt = np.zeros(int(T * fs) + 2, dtype=np.int64)
    cnt[a[:, 0]] = a[:, 1]
    return cnt


def kernel_bits(x_hi, L, fs, c=343.0):
    """The kernel's tile rule (ism_poly_kernel.cu tile setup): bits of one channel value, or None (two words)."""
    Vs = float(np.prod(L)) * (fs / c) ** 3
    Lmin = min(L) * fs / c
    N = 8.0 * math.pi * x_hi * x_hi / Vs + 24.0 * x_hi / Lmin + 16.0
    lb = math.frexp(N)[1]  # N < 2^lb
    bits = min(22, 30 - lb)
    return None if bits < 18 else bits


def single_word_limit(L, fs, c=343.0):
    """The largest delay (samples) whose tiles are single-word: N(x) < 2^12."""
    Vs = float(np.prod(L)) * (fs / c) ** 3
    a, b = 8.0 * math.pi / Vs, 24.0 / (min(L) * fs / c)
    return (-b + math.sqrt(b * b + 4.0 * a * (4096.0 - 16.0))) / (2.0 * a)


C = 1.0 + 2.0 ** -10  # 1 mm off a 2 m cube's centre, exact in fp32
CASES = [
    ("paper room, commensurate positions", [3, 4, 2.5], [1, 1, 1.2], [2, 3, 1.3]),
    ("cube, source and receiver at the centre", [2, 2, 2], [1, 1, 1], [1, 1, 1]),
    ("cube, receiver 1 mm off the centre", [2, 2, 2], [1, 1, 1], [1, 1, C]),
    ("unit cube", [1, 1, 1], [0.5, 0.5, 0.5], [0.2, 0.7, 0.3]),
    ("unit cube, centred", [1, 1, 1], [0.5, 0.5, 0.5], [0.5, 0.5, 0.5 + 2.0 ** -12]),
    ("flat room", [0.3, 10, 10], [0.15, 2, 3], [0.1, 8, 7]),
    ("corridor", [20, 0.3, 2], [3, 0.1, 1], [15, 0.2, 1.5]),
    ("cfg3 room, generic positions", [3, 4, 2.5], [1.5, 1.0, 1.2], [2.31, 3.17, 1.43]),
    ("cfg3 room, 0.1 m grid positions", [3, 4, 2.5], [1.1, 1.3, 0.7], [2.4, 3.1, 1.6]),
    ("5 m cube, centred", [5, 5, 5], [2.5, 2.5, 2.5], [2.5, 2.5, 2.5 + 2.0 ** -8]),
    ("4 m cube, half-integer", [4, 4, 4], [2, 2, 2], [1, 1, 1]),
    ("2x3x4, axis-aligned", [2, 3, 4], [1, 1.5, 2], [1, 1.5, 2.5]),
]


def worst_fill(cnt, L, fs):
    """max over samples of count * 2^bits / 2^31 (the fraction of the count capacity used) and where."""
    worst, at = 0.0, None
    for j in np.nonzero(cnt)[0]:
        bits = kernel_bits(j + 1.0, L, fs)
        if bits is None:
            continue  # two-word tile: capacity 2^17
        f = cnt[j] * 2.0 ** bits / 2.0 ** 31
        if f > worst:
            worst, at = f, (int(j), int(cnt[j]), bits)
    return worst, at


@pytest.mark.parametrize("fs", [16000.0, 48000.0])
@pytest.mark.parametrize("name,L,s,r", CASES, ids=[c[0] for c in CASES])
def test_single_word_capacity_used(counter, name, L, s, r, fs):
    """Up to the longest single-word delay of each room (0.14-2.05 s), no sample position fills the count
    capacity 2^(31 - bits): the guard's redo never runs here.  Measured worst: 0.35 (2 m cube, receiver 1 mm off
    the centre, 48 kHz, at 0.215 s — the geometry of the GPU test; the same with source and receiver both at
    the centre), 0.35 (1 m centred cube, 48 kHz), 0.32 (5 m centred cube, 48 kHz)."""
    T = single_word_limit(L, fs) / fs
    cnt = image_delay_counts(counter, L, s, r, fs, T)
    worst, at = worst_fill(cnt, L, fs)
    assert 0.0 < worst < 0.5, (name, fs, worst, at)


def test_mean_density_is_a_mean(counter):
    """The count per sample averages to 4 pi x^2 / V_s (one image per room volume), for generic and for
    commensurate positions alike, while the commensurate ones exceed the mean several times on single samples
    (why the rule's density term alone would not bound a position)."""
    L, fs = [3, 4, 2.5], 16000.0
    cnt = image_delay_counts(counter, L, [1.5, 1.0, 1.2], [2.31, 3.17, 1.43], fs, 0.2)
    Vs = float(np.prod(L)) * (fs / 343.0) ** 3
    j = np.arange(1500, 3000)
    mean_pred = 4 * math.pi * (j + 0.5) ** 2 / Vs
    assert abs(cnt[j].sum() / mean_pred.sum() - 1.0) < 0.02
    sym = image_delay_counts(counter, L, [1, 1, 1.2], [2, 3, 1.3], fs, 0.2)
    assert abs(sym[j].sum() / mean_pred.sum() - 1.0) < 0.02
    assert (sym[j] / mean_pred).max() > 3 > (cnt[j] / mean_pred).max()
