"""Test-side helpers restating the reference's tests/oracles.hpp.

Independent of both the oracle's and the product's FFT/solver paths:
direct O(N^2) DFTs, dense DFT matrices, SplitMix64 ``Rng`` and the random
problem generators (proj/tests/oracles.hpp:24-166).  The generators draw in
the same order as the reference's so the parity cases are the same problems
the reference tests ran.
"""
from __future__ import annotations

import itertools

import numpy as np

MASK = (1 << 64) - 1


class Rng:
    """SplitMix64 (proj/tests/oracles.hpp:102-117, proj/src/problem.cpp:222-228)."""

    def __init__(self, seed: int):
        self.state = seed & MASK

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def symmetric(self) -> float:
        return 2.0 * self.uniform() - 1.0

    def range(self, lo: int, hi: int) -> int:  # inclusive
        return lo + self.next() % (hi - lo + 1)


class Kern:
    """Sorted offset -> m x m block map (proj/include/fftstencil/kernel.hpp:19-56)."""

    def __init__(self, rank: int, fields: int = 1):
        self.rank, self.fields = rank, fields
        self.taps: dict[tuple, np.ndarray] = {}

    def add(self, off, block):
        off = tuple(int(o) for o in off)
        b = np.array(block, dtype=np.float64).reshape(self.fields, self.fields)
        if off in self.taps:
            self.taps[off] = self.taps[off] + b
        else:
            self.taps[off] = b
        return self

    def arrays(self):
        keys = sorted(self.taps)
        off = np.array(keys, dtype=np.int64).reshape(len(keys), self.rank)
        blk = np.array([self.taps[k] for k in keys], dtype=np.float64).reshape(len(keys), self.fields, self.fields)
        return off, blk

    def max_reach(self):
        r = [0] * self.rank
        for off in self.taps:
            for a in range(self.rank):
                r[a] = max(r[a], abs(off[a]))
        return r


def kern_from(taps: dict, rank: int, fields: int = 1) -> Kern:
    k = Kern(rank, fields)
    for off, v in taps.items():
        k.add(off if isinstance(off, tuple) else (off,), v)
    return k


def random_kernel(rng: Rng, rank: int, sigma: int, fields: int = 1, target_norm: float = 0.9) -> Kern:
    """proj/tests/oracles.hpp:121-153 (C++17 sequencing: in
    ``shell[rng.next() % rank] = rng.next() % 2 ? s : -s`` the right side is
    drawn first)."""
    k = Kern(rank, fields)
    tap_count = rng.range(2, 6)
    shell = [rng.range(-sigma, sigma) for _ in range(rank)]
    sign = sigma if rng.next() % 2 else -sigma
    shell[rng.next() % rank] = sign
    offsets = [shell]
    for _ in range(1, tap_count):
        offsets.append([rng.range(-sigma, sigma) for _ in range(rank)])
    for off in offsets:
        block = [[rng.symmetric() for _ in range(fields)] for _ in range(fields)]
        k.add(off, block)
    row_sums = np.zeros(fields)
    for off in sorted(k.taps):
        row_sums += np.abs(k.taps[off]).sum(axis=1)
    norm = row_sums.max()
    scaled = Kern(rank, fields)
    for off in sorted(k.taps):
        scaled.add(off, k.taps[off] * (target_norm / norm))
    return scaled


def random_grid(rng: Rng, n_values: int) -> np.ndarray:
    return np.array([rng.symmetric() for _ in range(n_values)])


def random_complex_grid(rng: Rng, n_values: int) -> np.ndarray:
    out = np.empty(n_values, dtype=np.complex128)
    for i in range(n_values):
        re = rng.symmetric()
        im = rng.symmetric()
        out[i] = complex(re, im)
    return out


def direct_dft(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    """O(N^2) DFT with exact (j*k) mod n phase reduction (oracles.hpp:24-40)."""
    n = x.size
    j = np.arange(n)
    idx = np.outer(j, j) % n
    sign = 1.0 if inverse else -1.0
    w = np.exp(sign * 2j * np.pi * idx / n)
    out = w @ x
    return out / n if inverse else out


def direct_multi_dft(g: np.ndarray, dims, fields: int = 1, inverse: bool = False) -> np.ndarray:
    """Nested-sum d-D DFT per field (oracles.hpp:43-70), via per-axis dense DFT matrices."""
    a = np.asarray(g, dtype=np.complex128).reshape(tuple(dims) + (fields,))
    for ax, n in enumerate(dims):
        j = np.arange(n)
        sign = 1.0 if inverse else -1.0
        w = np.exp(sign * 2j * np.pi * (np.outer(j, j) % n) / n)
        a = np.moveaxis(np.tensordot(w, a, axes=([1], [ax])), 0, ax)
    if inverse:
        a = a / float(np.prod(dims))
    return a.reshape(-1)


def dense_dft_matrix(dims, fields: int = 1) -> np.ndarray:
    """(N m) x (N m) operator F (x) I_m (oracles.hpp:73-95)."""
    cells = list(itertools.product(*[range(n) for n in dims]))
    N = len(cells)
    F = np.zeros((N * fields, N * fields), dtype=np.complex128)
    for ic, i in enumerate(cells):
        for jc, j in enumerate(cells):
            frac = sum(((i[a] * j[a]) % dims[a]) / dims[a] for a in range(len(dims)))
            w = np.exp(-2j * np.pi * frac)
            for f in range(fields):
                F[ic * fields + f, jc * fields + f] = w
    return F


def dense_idft_matrix(dims, fields: int = 1) -> np.ndarray:
    return dense_dft_matrix(dims, fields).conj() / float(np.prod(dims))


def rotate_grid(a: np.ndarray, dims, fields: int, shift) -> np.ndarray:
    """out[i] = in[i - shift] per axis (proj/src/grid.cpp:17-35)."""
    x = np.asarray(a).reshape(tuple(dims) + (fields,))
    return np.roll(x, shift=tuple(shift), axis=tuple(range(len(dims)))).reshape(-1)


def heat1d(alpha: float) -> Kern:
    return kern_from({(-1,): alpha, (0,): 1 - 2 * alpha, (1,): alpha}, 1)


def appendix_kernel() -> Kern:
    return kern_from({(-1,): -2.0, (0,): 1.0, (1,): 3.0}, 1)
