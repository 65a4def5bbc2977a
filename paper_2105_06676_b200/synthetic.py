"""BASELINE.json configurations as seeded synthetic problems.

Inputs follow the reference's documented random init (SplitMix64, one draw
per value in storage order, U[0,1) = (x >> 11) * 2^-53, U[-1,1) = 2u - 1;
proj/src/problem.cpp:222-247).  Seeds 1-5 drive cfg1-cfg5's data; the
second stream (seed + 1000) draws cfg3's weights and cfg5's bump centres
(SURVEY.md section 8d).  No dataset is involved anywhere: the reference's
benchmarks are synthetic stencils.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .fftstencil import GridShape, StencilKernel

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, n: int, start: int = 0) -> np.ndarray:
    """SplitMix64 outputs start .. start+n-1 of the stream seeded with `seed`
    (counter based: output i uses state seed + (i+1) * gamma), vectorised;
    the same stream as the reference's sequential generator."""
    i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, n: int, start: int = 0) -> np.ndarray:
    return (splitmix64(seed, n, start) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uniform_sym(seed: int, n: int, start: int = 0) -> np.ndarray:
    return 2.0 * uniform01(seed, n, start) - 1.0


@dataclass
class Config:
    name: str
    description: str
    dims: list
    fields: int
    T: int
    taps: dict = field(default_factory=dict)  # offset tuple -> coefficient or m x m block
    init: str = "u01"
    seed: int = 1

    def shape(self) -> GridShape:
        return GridShape(self.dims, self.fields)

    def kernel(self) -> StencilKernel:
        k = StencilKernel(len(self.dims), self.fields)
        for off in sorted(self.taps):
            k.add_tap(off, self.taps[off])
        return k

    def cells(self) -> int:
        return int(np.prod(self.dims))

    def initial(self, start: int = 0, count: int | None = None) -> np.ndarray:
        """Values start .. start+count-1 of the initial grid (storage order)."""
        n = self.cells() * self.fields if count is None else count
        if self.init == "u01":
            return uniform01(self.seed, n, start)
        if self.init == "sym":
            return uniform_sym(self.seed, n, start)
        if self.init == "bumps":
            return leapfrog_bumps(self.dims[0], self.seed + 1000)[start:start + n]
        raise ValueError(self.init)

    def scaled(self, dims) -> "Config":
        """Same stencil family on a smaller grid (parity / CPU-baseline samples)."""
        return Config(self.name + "@" + "x".join(map(str, dims)), self.description, list(dims), self.fields,
                      self.T, dict(self.taps), self.init, self.seed)


def leapfrog_bumps(n: int, seed: int, K: int = 4, width: float = 64.0) -> np.ndarray:
    """cfg5 initial state (u^0, u^-1) = (g, g): K Gaussian bumps of width w at
    seeded centres, periodic distance, zero velocity (SURVEY.md section 8d:
    K = 4, w = 64 pinned here)."""
    centres = (uniform01(seed, K) * n).astype(np.int64)
    i = np.arange(n)
    g = np.zeros(n)
    for c in centres:
        d = np.abs(i - c)
        d = np.minimum(d, n - d)
        g += np.exp(-(d / width) ** 2)
    out = np.empty(2 * n)
    out[0::2] = g
    out[1::2] = g
    return out


def _box9_weights(seed: int):
    u = uniform01(seed, 9)
    u = u / u.sum()
    offs = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1)]  # sorted-offset order
    return {o: float(w) for o, w in zip(offs, u)}


def configs() -> dict:
    heat7 = {(0, 0, 0): 0.4}
    for a in range(3):
        for s in (-1, 1):
            o = [0, 0, 0]
            o[a] = s
            heat7[tuple(o)] = 0.1
    C2 = 0.5 ** 2
    leap = {(0,): np.array([[2 - 2 * C2, -1.0], [1.0, 0.0]]),
            (-1,): np.array([[C2, 0.0], [0.0, 0.0]]),
            (1,): np.array([[C2, 0.0], [0.0, 0.0]])}
    return {
        "cfg1": Config("cfg1", "1D periodic 3-point heat {-1:.25,0:.5,+1:.25}, N=2^20 fp64, T=1000, U[0,1)",
                       [1 << 20], 1, 1000, {(-1,): 0.25, (0,): 0.5, (1,): 0.25}, "u01", 1),
        "cfg2": Config("cfg2", "2D periodic 5-point Jacobi (all 0.2), 4096x4096 fp64, T=1e4, U[0,1)",
                       [4096, 4096], 1, 10000,
                       {(0, 0): 0.2, (1, 0): 0.2, (-1, 0): 0.2, (0, 1): 0.2, (0, -1): 0.2}, "u01", 2),
        "cfg3": Config("cfg3", "2D periodic 9-point box, seeded non-negative weights summing to 1, 8192x8192 fp64, "
                       "T=1e5, U[-1,1)", [8192, 8192], 1, 100000, _box9_weights(1003), "sym", 3),
        "cfg4": Config("cfg4", "3D periodic 7-point heat (0.4 / 0.1), 1024^3 fp64, T=1000, U[0,1)",
                       [1024, 1024, 1024], 1, 1000, heat7, "u01", 4),
        "cfg5": Config("cfg5", "1D leapfrog wave as a 2-field first-order system, C=0.5, N=2^26 fp64, T=1e6, "
                       "Gaussian bumps, zero velocity", [1 << 26], 2, 1000000, leap, "bumps", 5),
    }
