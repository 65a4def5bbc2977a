"""Pins the CPU oracle (test infrastructure) against the reference's own
known answers and property tests.  No GPU needed.

Each test cites the reference test it re-expresses.
"""
import numpy as np
import pytest

import refutil as R
from refutil import Rng


def _k(case):
    off = np.array(case["offsets"], dtype=np.int64)
    blk = np.array(case["values"], dtype=np.float64).reshape(-1, 1, 1)
    return off, blk


# ----------------------------------------------------------- golden vectors
def test_golden_fft_delta_and_ones(orc, golden):
    for name in ("fft_delta", "fft_ones"):
        c = golden[name]
        x = np.array(c["input_re"], dtype=np.complex128)
        got = orc.multi_fft(x, c["dims"])
        want = np.array(c["want_re"]) + 1j * np.array(c["want_im"])
        assert np.abs(got - want).max() <= c["tol"], name


def test_golden_spectra(orc, golden):
    c = golden["identity_spectrum"]
    lam = orc.spectrum_from_kernel(c["dims"], 1, *_k(c))
    assert np.abs(lam - complex(*c["want_all"])).max() < c["tol"]
    c = golden["appendix_generator"]
    lam = orc.spectrum_from_kernel(c["dims"], 1, *_k(c))
    assert abs(lam[0] - complex(*c["want_lambda0"])) < c["tol"]
    c = golden["shift_spectrum"]
    lam = orc.spectrum_from_kernel(c["dims"], 1, *_k(c))
    want = np.array(c["want_re"]) + 1j * np.array(c["want_im"])
    assert np.abs(lam - want).max() < c["tol"]


def test_golden_pow_and_pinv(orc, golden):
    c = golden["pow_scalar"]
    lam = np.array([complex(*v) for v in c["lambda"]])
    for chk in c["checks"]:
        got = orc.pow_spectrum(lam, [lam.size], 1, chk["T"])[chk["index"]]
        if chk["tol"] == 0.0:
            assert got == complex(*chk["want"])
        else:
            assert abs(got - complex(*chk["want"])) < chk["tol"]
    c = golden["pinv"]
    lam = np.array([complex(*v) for v in c["lambda"]])
    got = orc.pseudo_inverse_spectrum(lam, [3])
    want = np.array([complex(*v) for v in c["want"]])
    assert np.abs(got - want).max() < c["tol"]
    assert got[1] == 0
    ones = np.ones(3, dtype=np.complex128)
    assert np.abs(orc.pseudo_inverse_spectrum(ones, [3]) - ones).max() == 0
    with pytest.raises(orc.OracleSpecError):
        orc.pseudo_inverse_spectrum(np.zeros(12, dtype=np.complex128), [3], m=2)


def test_golden_appendix_matrix_and_step(orc, golden):
    c = golden["appendix_matrix"]
    mat = orc.dense_stencil_matrix(c["dims"], 1, *_k(c))
    assert (mat == np.array(c["want"], dtype=float)).all()
    c = golden["appendix_one_step"]
    out = orc.solve_periodic(np.array(c["a0"], float), c["dims"], 1, *_k(c), c["T"])
    assert np.abs(out - np.array(c["want"], float)).max() <= c["tol"]


def test_golden_errors(orc, golden):
    c = golden["blowup_numeric_error"]
    rng = Rng(c["seed"])
    a = R.random_grid(rng, 16)
    with pytest.raises(orc.OracleNumericError):
        orc.solve_periodic(a, c["dims"], 1, *_k(c), c["T"])
    c = golden["vector_rejects_scalar"]
    with pytest.raises(orc.OracleSpecError):
        orc.solve_periodic(np.zeros(8), c["dims"], 1, *_k(c), c["T"], vector=True)


def test_golden_splitmix(orc, golden):
    c = golden["splitmix_seed7"]
    rng = Rng(c["seed"])
    want = np.array([rng.symmetric() for _ in range(c["n"])])
    assert (orc.splitmix_fill(c["seed"], c["n"], True) == want).all()


def test_golden_cli_fixtures(orc, golden):
    c = golden["cli_verify_heat1d"]
    a0 = orc.splitmix_fill(c["seed"], 256, True)
    fast = orc.solve_periodic(a0, c["dims"], 1, *_k(c), c["T"])
    slow = orc.evolve_periodic_naive(a0, c["dims"], 1, *_k(c), c["T"])
    assert np.abs(fast - slow).max() <= c["tol_rel1p"] * (1 + np.abs(slow).max())
    c = golden["cli_solve_delta"]
    a0 = np.zeros(64)
    a0[0] = 1.0
    fast = orc.solve_periodic(a0, c["dims"], 1, *_k(c), c["T"])
    slow = orc.evolve_periodic_naive(a0, c["dims"], 1, *_k(c), c["T"])
    assert np.abs(fast - slow).max() <= c["tol_rel1p"] * (1 + np.abs(slow).max())


# ----------------------------------------------------------- FFT properties
def test_fft_vs_direct_dft(orc):
    """proj/tests/test_fft.cpp:26-40"""
    rng = Rng(23)
    for n in (7, 12, 15, 32, 1000):
        g = R.random_complex_grid(rng, n)
        got = orc.multi_fft(g, [n])
        want = R.direct_dft(g)
        assert np.abs(got - want).max() <= 1e-10 * (1 + np.abs(want).max())


def test_multi_fft_vs_nested_sum(orc):
    """proj/tests/test_fft.cpp:42-55"""
    rng = Rng(29)
    for dims, m in (([12], 1), ([6, 10], 2), ([3, 4, 5], 1)):
        n = int(np.prod(dims)) * m
        g = R.random_complex_grid(rng, n)
        got = orc.multi_fft(g, dims, m)
        want = R.direct_multi_dft(g, dims, m)
        assert np.abs(got - want).max() <= 1e-10 * (1 + np.abs(want).max())
        goti = orc.multi_fft(g, dims, m, inverse=True)
        wanti = R.direct_multi_dft(g, dims, m, inverse=True)
        assert np.abs(goti - wanti).max() <= 1e-10


def test_fft_round_trip(orc):
    """proj/tests/test_fft.cpp:57-67"""
    rng = Rng(31)
    for dims, m in (([7], 1), ([12], 1), ([64, 64], 1), ([17, 241], 1), ([11, 13, 5], 2), ([1, 9], 1), ([4096], 1)):
        g = R.random_complex_grid(rng, int(np.prod(dims)) * m)
        back = orc.multi_fft(orc.multi_fft(g, dims, m), dims, m, inverse=True)
        assert np.abs(back - g).max() <= 1e-10 * (1 + np.abs(g).max())


# ----------------------------------------------------------- spectral
def test_convolution_theorem(orc):
    """proj/tests/test_spectral.cpp:59-97: F S F^-1 is block diagonal with our spectrum."""
    rng = Rng(37)
    checked = 0
    for _ in range(12):
        rank = 1 + rng.next() % 2
        m = 1 + rng.next() % 2
        dims = [rng.range(2, 16 if rank == 1 else 4) for _ in range(rank)]
        if np.prod(dims) > 16:
            continue
        sigma = min(1, min(dims) - 1)
        k = R.random_kernel(rng, rank, max(sigma, 0), m)
        if k.max_reach()[0] >= min(dims):
            continue
        off, blk = k.arrays()
        S = orc.dense_stencil_matrix(dims, m, off, blk).astype(np.complex128)
        conj = R.dense_dft_matrix(dims, m) @ S @ R.dense_idft_matrix(dims, m)
        lam = orc.spectrum_from_kernel(dims, m, off, blk).reshape(-1, m, m)
        n = S.shape[0]
        for r in range(n):
            for c in range(n):
                fr, fc = r // m, c // m
                want = lam[fr, r % m, c % m] if fr == fc else 0.0
                assert abs(conj[r, c] - want) <= 1e-10
        checked += 1
    assert checked > 0


def test_pow_block_matches_repeated_multiply(orc):
    """proj/tests/test_spectral.cpp:115-132"""
    rng = Rng(41)
    lam = np.zeros((3, 2, 2), dtype=np.complex128)
    for j in range(3):
        a = 0.9 * rng.symmetric()
        b = 0.3 * rng.symmetric()
        c = rng.symmetric()
        lam[j] = [[complex(a, b), c], [0.0, 1.0]]
    got = orc.pow_spectrum(lam, [3], 2, 8).reshape(3, 2, 2)
    for j in range(3):
        want = np.linalg.matrix_power(lam[j], 8)
        assert np.abs(got[j] - want).max() <= 1e-12 * (1 + np.abs(want).max())


def test_pow_semigroup(orc):
    """proj/tests/test_spectral.cpp:134-147"""
    rng = Rng(43)
    n = 24
    lam = np.array([complex(rng.symmetric(), rng.symmetric()) for _ in range(n)])
    for a, b in ((3, 5), (1, 31), (16, 16), (0, 32)):
        lhs = orc.pow_spectrum(lam, [8, 3], 1, a + b)
        prod = orc.multiply_spectra(orc.pow_spectrum(lam, [8, 3], 1, a), orc.pow_spectrum(lam, [8, 3], 1, b), [8, 3], 1)
        assert np.abs(lhs - prod).max() <= 1e-10 * (1 + np.abs(lhs).max())


def test_hadamard(orc):
    """proj/tests/test_spectral.cpp:176-206"""
    rng = Rng(47)
    x = R.random_complex_grid(rng, 8)
    ident = np.tile(np.eye(2, dtype=np.complex128), (4, 1, 1))
    assert np.abs(orc.hadamard(ident, x, [4], 2) - x).max() <= 1e-15
    assert np.abs(orc.hadamard(np.zeros((4, 2, 2), complex), x, [4], 2)).max() == 0
    lam = np.array([[[complex(rng.symmetric(), rng.symmetric()) for _ in range(2)] for _ in range(2)] for _ in range(4)])
    y = orc.hadamard(lam, x, [4], 2).reshape(4, 2)
    for j in range(4):
        want = lam[j] @ x.reshape(4, 2)[j]
        assert np.abs(y[j] - want).max() <= 1e-12


# ----------------------------------------------------------- periodic solver
def test_identity_kernel_any_T(orc):
    """proj/tests/test_periodic.cpp:30-37"""
    rng = Rng(53)
    a = R.random_grid(rng, 64)
    k = R.kern_from({(0,): 1.0}, 1)
    for T in (1, 97, 1 << 40):
        assert np.abs(orc.solve_periodic(a, [64], 1, *k.arrays(), T) - a).max() <= 1e-12


def test_heat_vs_naive(orc):
    """proj/tests/test_periodic.cpp:48-55"""
    rng = Rng(59)
    a = R.random_grid(rng, 32)
    k = R.heat1d(0.125)
    fast = orc.solve_periodic(a, [32], 1, *k.arrays(), 100)
    slow = orc.evolve_periodic_naive(a, [32], 1, *k.arrays(), 100)
    assert np.abs(fast - slow).max() <= 1e-9 * (1 + np.abs(slow).max())


def test_T0_bit_exact(orc):
    """proj/tests/test_periodic.cpp:57-62"""
    rng = Rng(61)
    a = R.random_grid(rng, 64)
    k = R.random_kernel(rng, 2, 1)
    assert (orc.solve_periodic(a, [8, 8], 1, *k.arrays(), 0) == a).all()


def test_randomized_vs_naive(orc):
    """proj/tests/test_periodic.cpp:64-84 (40 random cases, d <= 3, m in {1,2})."""
    rng = Rng(67)
    times = (0, 1, 2, 3, 7, 16, 100)
    for trial in range(40):
        rank = 1 + rng.next() % 3
        dims = [rng.range(4, 12 if rank == 3 else 32) for _ in range(rank)]
        m = 2 if trial % 4 == 0 else 1
        sigma = rng.range(1, 2)
        k = R.random_kernel(rng, rank, sigma, m)
        a = R.random_grid(rng, int(np.prod(dims)) * m)
        T = times[rng.next() % 7]
        fast = orc.solve_periodic(a, dims, m, *k.arrays(), T)
        slow = orc.evolve_periodic_naive(a, dims, m, *k.arrays(), T)
        assert np.abs(fast - slow).max() <= 1e-8 * (1 + np.abs(slow).max()), (dims, m, T)


def test_semigroup_and_shift(orc):
    """proj/tests/test_periodic.cpp:86-107"""
    rng = Rng(71)
    k = R.heat1d(0.2)
    a = R.random_grid(rng, 48)
    for s, t in ((3, 5), (31, 33), (64, 1)):
        whole = orc.solve_periodic(a, [48], 1, *k.arrays(), s + t)
        split = orc.solve_periodic(orc.solve_periodic(a, [48], 1, *k.arrays(), s), [48], 1, *k.arrays(), t)
        assert np.abs(whole - split).max() <= 1e-9 * (1 + np.abs(whole).max())
    rng = Rng(73)
    dims = [10, 12]
    k = R.random_kernel(rng, 2, 1)
    a = R.random_grid(rng, 120)
    lhs = orc.solve_periodic(R.rotate_grid(a, dims, 1, (3, 7)), dims, 1, *k.arrays(), 9)
    rhs = R.rotate_grid(orc.solve_periodic(a, dims, 1, *k.arrays(), 9), dims, 1, (3, 7))
    assert np.abs(lhs - rhs).max() <= 1e-10


def test_affine_two_field(orc):
    """proj/tests/test_periodic.cpp:141-182"""
    rng = Rng(83)
    n, T, c = 64, 50, 0.37
    s = R.heat1d(0.125)
    folded = R.Kern(1, 2)
    for off, blk in s.taps.items():
        folded.add(off, [[blk[0, 0], 0.0], [0.0, 0.0]])
    folded.add((0,), [[0.0, 1.0], [0.0, 1.0]])
    a = np.zeros(2 * n)
    direct = np.zeros(n)
    for i in range(n):
        v = rng.symmetric()
        a[2 * i], a[2 * i + 1], direct[i] = v, c, v
    fast = orc.solve_periodic(a, [n], 2, *folded.arrays(), T, vector=True)
    for _ in range(T):
        direct = orc.step_periodic(direct, [n], 1, *s.arrays()) + c
    assert np.abs(fast[0::2] - direct).max() <= 1e-9


def test_implicit(orc):
    """proj/tests/test_periodic.cpp:184-228"""
    ident = R.kern_from({(0,): 1.0}, 1)
    s = R.heat1d(0.125)
    rng = Rng(89)
    a = R.random_grid(rng, 24)
    imp = orc.solve_periodic_implicit(a, [24], ident.arrays(), s.arrays(), 13)
    exp = orc.solve_periodic(a, [24], 1, *s.arrays(), 13)
    assert np.abs(imp - exp).max() <= 1e-12
    assert (orc.solve_periodic_implicit(a, [24], ident.arrays(), s.arrays(), 0) == a).all()
    beta = 0.125
    q = R.kern_from({(-1,): -beta, (0,): 1 + 2 * beta, (1,): -beta}, 1)
    s = R.kern_from({(-1,): beta, (0,): 1 - 2 * beta, (1,): beta}, 1)
    rng = Rng(97)
    a0 = R.random_grid(rng, 16)
    Q = orc.dense_stencil_matrix([16], 1, *q.arrays())
    S = orc.dense_stencil_matrix([16], 1, *s.arrays())
    state = a0.copy()
    for t in range(1, 4):
        state = np.linalg.solve(Q, S @ state)
        spectral = orc.solve_periodic_implicit(a0, [16], q.arrays(), s.arrays(), t)
        assert np.abs(spectral - state).max() <= 1e-9


def test_spec_errors(orc):
    """proj/src/kernel.cpp:38-49 preconditions."""
    k = R.kern_from({(5,): 1.0}, 1)
    with pytest.raises(orc.OracleSpecError):
        orc.solve_periodic(np.zeros(4), [4], 1, *k.arrays(), 1)
    k = R.kern_from({(0, 0): 1.0}, 2)
    with pytest.raises(orc.OracleSpecError):
        orc.solve_periodic(np.zeros(4), [4], 1, *k.arrays(), 1)
    with pytest.raises(orc.OracleSpecError):
        orc.solve_periodic(np.zeros(4), [4], 1, np.zeros((0, 1), np.int64), np.zeros((0, 1, 1)), 1)
