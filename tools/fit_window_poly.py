"""Fit the Hann-window polynomial used by the fp32 accumulation kernel (product side, not oracle).

The kernel evaluates the Peterson window of Eq. 6,
    w(u) = 1/2 (1 + cos(pi u / H)) = cos^2(pi u / (2 H)),   |u| < H,  H = T_w fs / 2,
as w = (s' p(s'))^2 with v = u / H, s' = min(v^2 - 1, 0) in [-1, 0]: cos(pi/2 sqrt(1 - s)) has a simple
root at s = 1 - v^2 = 0, so c(s) = s q(s) and c^2 is exactly 0 for |v| >= 1 (the clamp also masks
out-of-window lanes).  p(s') = q(-s') so that p has coefficients b_i = (-1)^i a_i.

The fit is a Lawson-reweighted minimax of the window error |dw| ~ |2 c dc| weighted by the sinc envelope
env(v) = 1 / max(1, pi H_w v) that multiplies it in every tap (Eq. 6: w(u) sinc(u)), with H_w = 16 (8 kHz,
the smallest rate of interest; larger H only shrinks env away from v = 0).  So the error is pushed to the
window edges, where the sinc factor is small.  deg = degree of q (the kernel's DEG3 build uses deg = 2).

Prints the float32 coefficients b0..b_deg, max |dw| and max |dw| env over the window.
"""
import sys

import numpy as np

H_W = 16


def fit(deg=2, iters=200, weighted=True):
    n = 20000
    x = 0.5 - 0.5 * np.cos(np.pi * (np.arange(n) + 0.5) / n)  # s = 1 - v^2 in (0, 1), Chebyshev nodes
    v = np.sqrt(1 - x)
    cx = np.cos(np.pi / 2 * v)
    env = 1 / np.maximum(1, np.pi * H_W * v) if weighted else np.ones(n)
    A = np.vstack([x ** (i + 1) for i in range(deg + 1)]).T
    coef, *_ = np.linalg.lstsq(A * env[:, None], cx * env, rcond=None)
    for _ in range(iters):
        err = (A @ coef - cx) * 2 * cx * env
        wts = env * (np.sqrt(np.abs(err)) + 1e-15)
        coef, *_ = np.linalg.lstsq(A * wts[:, None], cx * wts, rcond=None)
    return coef


def check(b):
    v = np.linspace(-1, 1, 400001).astype(np.float32)
    sp = np.minimum(v ** 2 - np.float32(1), np.float32(0))
    p = np.float32(0)
    for bi in b[::-1]:
        p = p * sp + bi
    w = (p * sp).astype(np.float64) ** 2
    ref = np.cos(np.pi * v.astype(np.float64) / 2) ** 2
    env = 1 / np.maximum(1, np.pi * H_W * np.abs(v.astype(np.float64)))
    return float(np.max(np.abs(w - ref))), float(np.max(np.abs(w - ref) * env))


if __name__ == "__main__":
    deg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    a = fit(deg)
    b = np.array([(-1) ** i * a[i] for i in range(len(a))], dtype=np.float32)
    e, ee = check(b)
    print("b =", [float(x) for x in b])
    print(f"max |w err| = {e:.3e}   max |w err| env = {ee:.3e}")
