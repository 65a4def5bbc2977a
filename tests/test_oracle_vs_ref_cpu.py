"""The restated oracle (oracle/liborc.so) against the REFERENCE ITSELF:
oracle/_ref/libfftstencil_ref.so is the reference's own periodic-path sources
compiled unmodified (oracle/Makefile `ref`; Eigen3, absent here, replaced by
oracle/eigen_shim).  Same seeded inputs through both, function by function.

Bar: bit-for-bit.  The restatement follows the reference operation for
operation and both are built with the reference's flags, so every case below
is required to be identical, not merely close.
"""

import numpy as np
import pytest

from oracle import oracle as orc
from oracle import ref as refmod
from refutil import Rng, random_complex_grid, random_grid, random_kernel

pytestmark = pytest.mark.skipif(not refmod.build(), reason="oracle/_ref not built and /root/reference absent")


@pytest.fixture(scope="module")
def ref():
    return refmod.module()


SHAPES = [([64], 1), ([60], 1), ([1], 1), ([2], 1), ([37], 2), ([128], 2), ([16, 16], 1), ([12, 10], 1), ([8, 1, 8], 1),
          ([9, 16], 2), ([8, 8, 8], 1), ([5, 6, 7], 1), ([4, 4, 4, 4], 1), ([32, 3], 3), ([2100], 1)]


def _case(seed, dims, m):
    rng = Rng(seed)
    sigma = max(0, min(2, (min(dims) - 1) // 2))
    k = random_kernel(rng, len(dims), sigma, m)
    a0 = random_grid(rng, int(np.prod(dims)) * m)
    off, blk = k.arrays()
    return a0, off, blk


@pytest.mark.parametrize("dims,m", SHAPES)
def test_solve_periodic_bitwise(ref, dims, m):
    for seed, T in ((11, 0), (12, 1), (13, 2), (14, 17), (15, 1000), (16, 123457)):
        a0, off, blk = _case(seed, dims, m)
        x = orc.solve_periodic(a0, dims, m, off, blk, T, vector=m > 1)
        y = ref.solve_periodic(a0, dims, m, off, blk, T, vector=m > 1)
        assert np.array_equal(x, y), (dims, m, T, np.abs(x - y).max())


def test_stage_functions_bitwise(ref):
    for seed, (dims, m) in enumerate(SHAPES):
        rng = Rng(100 + seed)
        n = int(np.prod(dims))
        z = random_complex_grid(rng, n * m)
        for inv in (False, True):
            assert np.array_equal(orc.multi_fft(z, dims, m, inverse=inv), ref.multi_fft(z, dims, m, inverse=inv))
        _, off, blk = _case(200 + seed, dims, m)
        lam_o = orc.spectrum_from_kernel(dims, m, off, blk)
        lam_r = ref.spectrum_from_kernel(dims, m, off, blk)
        assert np.array_equal(lam_o, lam_r)
        for T in (0, 1, 5, 1024, 99999):
            assert np.array_equal(orc.pow_spectrum(lam_o, dims, m, T), ref.pow_spectrum(lam_o, dims, m, T))
        lam2 = random_complex_grid(rng, n * m * m)
        assert np.array_equal(orc.multiply_spectra(lam_o, lam2, dims, m), ref.multiply_spectra(lam_o, lam2, dims, m))
        assert np.array_equal(orc.hadamard(lam_o, z, dims, m), ref.hadamard(lam_o, z, dims, m))
        if m == 1:
            assert np.array_equal(orc.pseudo_inverse_spectrum(lam_o, dims), ref.pseudo_inverse_spectrum(lam_o, dims))


def test_implicit_bitwise(ref):
    for seed, dims in enumerate(([64], [60], [16, 16], [12, 10], [8, 8, 8])):
        rng = Rng(300 + seed)
        r = len(dims)
        # Crank-Nicolson-like pair: Q = I - a L, S = I + a L with L the axis Laplacian
        taps_q, taps_s = {}, {}
        zero = tuple([0] * r)
        a = 0.05 + 0.2 * rng.uniform()
        taps_q[zero], taps_s[zero] = 1.0 + 2 * a * r, 1.0 - 2 * a * r
        for ax in range(r):
            for s in (-1, 1):
                o = [0] * r
                o[ax] = s
                taps_q[tuple(o)], taps_s[tuple(o)] = -a, a
        keys = sorted(taps_q)
        off = np.array(keys, dtype=np.int64).reshape(len(keys), r)
        q = (off, np.array([taps_q[k] for k in keys]).reshape(-1, 1, 1))
        s_ = (off, np.array([taps_s[k] for k in keys]).reshape(-1, 1, 1))
        a0 = random_grid(rng, int(np.prod(dims)))
        for T in (0, 1, 40):
            x = orc.solve_periodic_implicit(a0, dims, q, s_, T)
            y = ref.solve_periodic_implicit(a0, dims, q, s_, T)
            assert np.array_equal(x, y)


def test_naive_and_dense_bitwise(ref):
    for seed, (dims, m) in enumerate(SHAPES[:13]):
        a0, off, blk = _case(400 + seed, dims, m)
        assert np.array_equal(orc.step_periodic(a0, dims, m, off, blk), ref.step_periodic(a0, dims, m, off, blk))
        assert np.array_equal(orc.evolve_periodic_naive(a0, dims, m, off, blk, 9),
                              ref.evolve_periodic_naive(a0, dims, m, off, blk, 9))
        if int(np.prod(dims)) * m <= 300:
            assert np.array_equal(orc.dense_stencil_matrix(dims, m, off, blk), ref.dense_stencil_matrix(dims, m, off, blk))


def test_errors_match(ref):
    a0 = np.ones(4)
    off = np.array([[-1], [0], [1]], dtype=np.int64)
    # blow-up: NumericError from both (proj/tests/test_periodic.cpp:230-239)
    blk = np.array([3.0, 3.0, 3.0]).reshape(3, 1, 1)
    big = np.arange(64, dtype=np.float64)
    for mod in (orc, ref):
        with pytest.raises(mod.OracleNumericError):
            mod.solve_periodic(big, [64], 1, off, blk, 4000)
    # kernel that does not fit the grid, vector entry with m = 1: SpecError from both
    wide = np.array([[-4], [0], [4]], dtype=np.int64)
    for mod in (orc, ref):
        with pytest.raises(mod.OracleSpecError):
            mod.solve_periodic(a0, [4], 1, wide, np.ones((3, 1, 1)) / 3, 2)
        with pytest.raises(mod.OracleSpecError):
            mod.solve_periodic(a0, [4], 1, off, np.ones((3, 1, 1)) / 3, 2, vector=True)
    # same message text
    for mod in (orc, ref):
        try:
            mod.solve_periodic(a0, [4], 1, wide, np.ones((3, 1, 1)) / 3, 2)
        except mod.OracleSpecError as e:
            msg = str(e)
        if mod is orc:
            first = msg
    assert first == msg


def test_baseline_configs_reduced_bitwise(ref):
    """The five BASELINE configs' stencils on reduced grids (same generators as bench.py)."""
    from paper_2105_06676_b200 import synthetic
    for name, dims in (("cfg1", [4096]), ("cfg2", [128, 128]), ("cfg3", [256, 128]), ("cfg4", [32, 32, 32]),
                       ("cfg5", [1024])):
        cfg = synthetic.configs()[name].scaled(dims)
        a0 = cfg.initial()
        m = cfg.fields
        keys = sorted(cfg.taps)
        off = np.array(keys, dtype=np.int64).reshape(len(keys), len(dims))
        blk = np.array([np.asarray(cfg.taps[k], dtype=np.float64).reshape(m, m) for k in keys])
        T = min(cfg.T, 5000)
        x = orc.solve_periodic(a0, dims, m, off, blk, T, vector=m > 1)
        y = ref.solve_periodic(a0, dims, m, off, blk, T, vector=m > 1)
        assert np.array_equal(x, y), name
