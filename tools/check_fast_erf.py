#!/usr/bin/env python3
"""Exhaustive accuracy check of K1's fast erf (gate_tc.cu: gelu_fast2): the
rational p(x)/q(x) evaluated in fp32 with FMA (emulated through float64, where
a*b of two fp32 values is exact) and an exactly rounded reciprocal, over EVERY
fp32 x in [0, 4] (the function is odd; inputs are clamped to [-4, 4]).
Prints the max |error| against scipy's erf; the kernel's band uses
ERF_EPS = 1e-6, which must exceed this plus the rcp.approx error (<= 2^-22
relative).  Takes a few minutes on one core."""
import numpy as np
from scipy.special import erf

A = [-1.60960333262415e-02, -2.95459980854025e-03, -7.34990630326855e-04, -5.69250639462346e-05,
     -2.10102402082508e-06, 2.77068142495902e-08, -2.72614225801306e-10]
B = [-1.42647390514189e-02, -7.37332916720468e-03, -1.68282697438203e-03, -2.13374055278905e-04,
     -1.45660718464996e-05]


def fma32(x, y, z):
    return (x.astype(np.float64) * y.astype(np.float64) + z).astype(np.float32)


def main():
    a32 = [np.float32(c) for c in A]
    b32 = [np.float32(c) for c in B]
    hi = int(np.float32(4).view(np.uint32))
    step = 1 << 22
    worst = 0.0
    for s in range(0, hi + 1, step):
        x = np.arange(s, min(s + step, hi + 1), dtype=np.uint32).view(np.float32)
        x2 = (x * x).astype(np.float32)
        p = np.full_like(x, a32[6])
        for c in a32[5::-1]:
            p = fma32(p, x2, np.float64(c))
        p = (p * x).astype(np.float32)
        q = np.full_like(x, b32[4])
        for c in b32[3::-1]:
            q = fma32(q, x2, np.float64(c))
        e = (p * (np.float32(1) / q).astype(np.float32)).astype(np.float32)
        worst = max(worst, float(np.abs(e.astype(np.float64) - erf(x.astype(np.float64))).max()))
    print(f"max |fast_erf - erf| over all fp32 in [0, 4]: {worst:.3e}  (ERF_EPS = 1e-6)")
    assert worst + 2.0 ** -22 < 1e-6


if __name__ == "__main__":
    main()
