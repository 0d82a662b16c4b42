"""Fit the Hann-window polynomial used by the fp32 accumulation kernel (product side, not oracle).

The kernel evaluates the Peterson window of Eq. 6,
    w(u) = 1/2 (1 + cos(pi u / H)) = cos^2(pi u / (2 H)),   |u| < H,  H = T_w fs / 2,
as w = (s' p(s'))^2 with v = u / H, s' = min(v^2 - 1, 0) in [-1, 0]: cos(pi/2 sqrt(1 - s)) has a simple
root at s = 1 - v^2 = 0, so c(s) = s q(s) and c^2 is exactly 0 for |v| >= 1 (the clamp also masks
out-of-window lanes).  p(s') = q(-s') so that p has coefficients b_i = (-1)^i a_i.

Prints the float32 coefficients b0..b3 and the max |w| error over the window.
"""
import numpy as np


def fit(deg=3, iters=60):
    x = 0.5 - 0.5 * np.cos(np.pi * (np.arange(8000) + 0.5) / 8000)
    cx = np.cos(np.pi / 2 * np.sqrt(1 - x))
    A = np.vstack([x ** (i + 1) for i in range(deg + 1)]).T
    coef, *_ = np.linalg.lstsq(A, cx, rcond=None)
    for _ in range(iters):  # Lawson-style reweighting towards minimax
        err = A @ coef - cx
        wts = np.sqrt(np.abs(err)) + 1e-15
        coef, *_ = np.linalg.lstsq(A * wts[:, None], cx * wts, rcond=None)
    return coef


if __name__ == "__main__":
    a = fit()
    b = np.array([(-1) ** i * a[i] for i in range(len(a))], dtype=np.float32)
    v = np.linspace(-1, 1, 400001)
    sp = np.minimum(v.astype(np.float32) ** 2 - np.float32(1), np.float32(0))
    p = np.float32(0)
    for bi in b[::-1]:
        p = p * sp + bi
    w = (p * sp) ** 2
    ref = np.cos(np.pi * v / 2) ** 2
    print("b =", [float(x) for x in b])
    print("max |w err| =", float(np.max(np.abs(w - ref))))
