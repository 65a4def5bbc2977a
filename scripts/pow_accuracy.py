"""Accuracy of the real 2x2 symbol power (cfg5's leapfrog, C = 0.5, T = 1e6).

Compares, per frequency, three ways of raising the fp64 symbol
A(theta) = [[2 - 2C^2 + 2C^2 cos theta, -1], [1, 0]] to the T-th power against
the exact power of the same fp64 matrix (mpmath, 60 digits):

  matpow  right-to-left binary exponentiation of the matrix (the reference's
          pow_spectrum loop, proj/src/spectrum.cpp:66-82, and the CPU oracle)
  ch_pq   Cayley-Hamilton A^n = p A + q I, doubling (p, q)
  ch_ptr  Cayley-Hamilton tracked as (p_n, trace A^n, det^n): the GPU row-pair
          kernels' pow_real2_ch (fsx_kernels.cu)

numpy float64 without FMA, so the GPU's numbers are a little better still.
Usage: python scripts/pow_accuracy.py
"""
import mpmath
import numpy as np

C2 = 0.25
T = 10**6


def symbol(c):
    l0 = C2 * c
    l0 = l0 + (2 - 2 * C2)
    l0 = l0 + C2 * c
    one = np.ones_like(c)
    return l0, -one, one, np.zeros_like(c)


def matpow(l, T):
    l0, l1, l2, l3 = [x.copy() for x in l]
    a0, a1, a2, a3 = np.ones_like(l0), np.zeros_like(l0), np.zeros_like(l0), np.ones_like(l0)
    t = T
    while t:
        if t & 1:
            a0, a1, a2, a3 = a0 * l0 + a1 * l2, a0 * l1 + a1 * l3, a2 * l0 + a3 * l2, a2 * l1 + a3 * l3
        t >>= 1
        if t:
            pp, tr = l1 * l2, l0 + l3
            l0, l1, l2, l3 = l0 * l0 + pp, l1 * tr, l2 * tr, l3 * l3 + pp
    return a0, a1, a2, a3


def ch_pq(l, T):
    l0, l1, l2, l3 = l
    t, d = l0 + l3, l0 * l3 - l1 * l2
    p, q = np.ones_like(l0), np.zeros_like(l0)
    for b in bin(T)[3:]:
        p, q = p * (p * t + 2 * q), q * q - d * (p * p)
        if b == "1":
            p, q = p * t + q, -d * p
    return p * l0 + q, p * l1, p * l2, p * l3 + q


def ch_ptr(l, T):
    l0, l1, l2, l3 = l
    t, d = l0 + l3, l0 * l3 - l1 * l2
    p, tr, dn = np.ones_like(l0), t.copy(), d.copy()
    for b in bin(T)[3:]:
        p, tr, dn = p * tr, tr * tr - 2 * dn, dn * dn
        if b == "1":
            pn = (p * t + tr) * 0.5
            tr, p, dn = pn * t - 2 * d * p, pn, dn * d
    q = (tr - p * t) * 0.5
    return p * l0 + q, p * l1, p * l2, p * l3 + q


def exact(l0, T):
    mpmath.mp.dps = 60
    R = mpmath.matrix([[mpmath.mpf(float(l0)), -1], [1, 0]]) ** T
    return [float(R[0, 0]), float(R[0, 1]), float(R[1, 0]), float(R[1, 1])]


def main():
    for logn in (16, 20, 26):
        n = 1 << logn
        ks = np.unique(np.concatenate([np.arange(0, 64), np.geomspace(64, n // 2, 400).astype(np.int64)]))
        l = symbol(np.cos(2 * np.pi * ks / n))
        ex = np.array([exact(x, T) for x in l[0]]).T
        nrm = np.maximum(1.0, np.abs(ex).max(axis=0))
        for name, f in (("matpow", matpow), ("ch_pq", ch_pq), ("ch_ptr", ch_ptr)):
            e = np.abs(np.array(f(l, T)) - ex).max(axis=0) / nrm
            print(f"N=2^{logn} {name:7s} worst rel {e.max():.2e}  median {np.median(e):.2e}")


if __name__ == "__main__":
    main()
