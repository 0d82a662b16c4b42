"""Headroom of the polyphase kernel's single-word fixed point (reading R11) — host logic, CPU.

The kernel adds every image's channel values v = round(A T_d 2^s), |v| <= 2^bits, into one int32 word per
sample position, with bits = min(22, 30 - ceil(log2 N)) and N = 8 pi x_hi^2 / V_s + 24 x_hi / L_min + 16 from
the tile's largest delay x_hi, the room volume V_s and its shortest side L_min (all in samples).  The first
term is twice the MEAN number of images per sample; the lattice of images (Eq. 1) stacks many
images on one integer delay in symmetric or commensurate geometries (a cube with source and receiver at its
centre: r3(n) <= 24 sqrt(n) lattice points on |k|^2 = n), which the second term covers.  These tests count,
by brute force over the whole image lattice, the images whose delay floors to each sample j and check that
even at full amplitude they fit with a 2x margin: count_j * 2^bits < 2^30, with bits taken for the smallest
tile that can hold j (x_hi = j + 1, the least headroom).
"""
import math

import numpy as np
import pytest


def image_delay_counts(L, s, r, fs, T, c=343.0):
    """Number of images (every lattice point of Eq. 1 within T c) per integer delay floor(d fs / c)."""
    L, s, r = (np.asarray(v, dtype=np.float64) for v in (L, s, r))
    dmax = T * c
    axes = []
    for a in range(3):
        k = int(dmax / L[a]) + 3
        n = np.arange(-k, k + 1)
        # Eq. 1: x_n = n L + s for even n, (n + 1) L - s for odd n; minus the receiver
        axes.append(np.where(n % 2 == 0, n * L[a] + s[a], (n + 1) * L[a] - s[a]) - r[a])
    X, Y = np.meshgrid(axes[0], axes[1], indexing="ij")
    rho2 = (X * X + Y * Y).ravel()
    rho2 = rho2[rho2 < dmax * dmax]
    cnt = np.zeros(int(T * fs) + 2, dtype=np.int64)
    for z in axes[2]:
        d2 = rho2 + z * z
        d = np.sqrt(d2[d2 < dmax * dmax])
        np.add.at(cnt, np.floor(d * fs / c).astype(np.int64), 1)
    return cnt


def kernel_bits(x_hi, L, fs, c=343.0):
    """The kernel's tile rule (ism_poly_kernel.cu tile setup): bits of one channel value, or None (two words)."""
    Vs = float(np.prod(L)) * (fs / c) ** 3
    Lmin = min(L) * fs / c
    N = 8.0 * math.pi * x_hi * x_hi / Vs + 24.0 * x_hi / Lmin + 16.0
    lb = math.frexp(N)[1]  # N < 2^lb
    bits = min(22, 30 - lb)
    return None if bits < 16 else bits


CASES = [
    ("paper room, commensurate positions", [3, 4, 2.5], [1, 1, 1.2], [2, 3, 1.3]),
    ("cube, source and receiver at the centre", [2, 2, 2], [1, 1, 1], [1, 1, 1]),
    ("unit cube", [1, 1, 1], [0.5, 0.5, 0.5], [0.2, 0.7, 0.3]),
    ("flat room", [0.3, 10, 10], [0.15, 2, 3], [0.1, 8, 7]),
    ("corridor", [20, 0.3, 2], [3, 0.1, 1], [15, 0.2, 1.5]),
    ("cfg3 room, generic positions", [3, 4, 2.5], [1.5, 1.0, 1.2], [2.31, 3.17, 1.43]),
    ("cfg3 room, 0.1 m grid positions", [3, 4, 2.5], [1.1, 1.3, 0.7], [2.4, 3.1, 1.6]),
    ("5 m cube, centred", [5, 5, 5], [2.5, 2.5, 2.5], [2.5, 2.5, 2.5 + 1e-9]),
    ("4 m cube, half-integer", [4, 4, 4], [2, 2, 2], [1, 1, 1]),
    ("2x3x4, axis-aligned", [2, 3, 4], [1, 1.5, 2], [1, 1.5, 2.5]),
]


@pytest.mark.parametrize("fs", [16000.0, 48000.0])
@pytest.mark.parametrize("name,L,s,r", CASES, ids=[c[0] for c in CASES])
def test_single_word_sums_cannot_overflow(name, L, s, r, fs):
    T = 0.2 if np.prod(L) > 1.5 else 0.12
    cnt = image_delay_counts(L, s, r, fs, T)
    worst = 0.0
    for j in np.nonzero(cnt)[0]:
        bits = kernel_bits(j + 1.0, L, fs)
        if bits is None:
            continue  # two-word tile: 2^17 terms of headroom
        assert cnt[j] * 2.0 ** bits < 2.0 ** 30, (name, fs, int(j), int(cnt[j]), bits)
        worst = max(worst, cnt[j] * 2.0 ** bits / 2.0 ** 31)
    assert worst > 0.0


def test_mean_density_is_a_mean():
    """The count per sample averages to 4 pi x^2 / V_s (one image per room volume), for generic and for
    commensurate positions alike, while the commensurate ones exceed the mean several times on single samples
    (why the rule's density term alone would not bound a position)."""
    L, fs = [3, 4, 2.5], 16000.0
    cnt = image_delay_counts(L, [1.5, 1.0, 1.2], [2.31, 3.17, 1.43], fs, 0.2)
    Vs = float(np.prod(L)) * (fs / 343.0) ** 3
    j = np.arange(1500, 3000)
    mean_pred = 4 * math.pi * (j + 0.5) ** 2 / Vs
    assert abs(cnt[j].sum() / mean_pred.sum() - 1.0) < 0.02
    sym = image_delay_counts(L, [1, 1, 1.2], [2, 3, 1.3], fs, 0.2)
    assert abs(sym[j].sum() / mean_pred.sum() - 1.0) < 0.02
    assert (sym[j] / mean_pred).max() > 3 > (cnt[j] / mean_pred).max()
