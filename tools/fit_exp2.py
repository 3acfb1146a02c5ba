"""Coefficients of the degree-3 polynomial for 2^f, f in [0, 1), used by
ex2_poly2 in csrc/sm100.cuh: p(f) = 1 + c1 f + c2 f^2 + c3 f^3 minimising the
max relative error (Lawson's iteratively reweighted least squares)."""
import struct

import numpy as np

f = np.linspace(0, 1, 20001)
t = 2.0 ** f
A = np.stack([f, f ** 2, f ** 3], 1) / t[:, None]
b = (t - 1) / t
w = np.ones_like(f)
for _ in range(200):
    W = np.sqrt(w)
    c, *_ = np.linalg.lstsq(A * W[:, None], b * W, rcond=None)
    e = np.abs(A @ c - b)
    w = w * e
    w /= w.sum()
p = 1 + c[0] * f + c[1] * f ** 2 + c[2] * f ** 3
hexf = lambda x: hex(struct.unpack("<I", struct.pack("<f", np.float32(x)))[0])
print("c1..c3 =", c, [hexf(x) for x in c], "max rel err", np.max(np.abs(p / t - 1)))
