"""GPU parity: the sm_100a path (through the C ABI) against the reference's
known answers, its property tests, and the CPU oracle on the same seeded
inputs.  Each test cites the reference test it re-expresses.

Tolerances: the reference's own (1e-12 .. 1e-8 absolute-relative, as cited),
and relative L2 <= 1e-10 against the oracle for the fp64 configs (BASELINE
north_star).
"""
import numpy as np
import pytest

import refutil as R
from refutil import Rng

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if fs.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU parity tests must run on a B200")


def K(k: R.Kern) -> "fs.StencilKernel":
    out = fs.StencilKernel(k.rank, k.fields)
    for off in sorted(k.taps):
        out.add_tap(off, k.taps[off] if k.fields > 1 else float(k.taps[off][0, 0]))
    return out


def G(dims, data, m=1):
    return fs.FieldGrid(fs.GridShape(dims, m), data)


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ------------------------------------------------------------------ golden vectors
def test_golden_known_answers(golden):
    c = golden["appendix_one_step"]
    k = R.kern_from({tuple(o): v for o, v in zip(c["offsets"], c["values"])}, 1)
    out = fs.solve_periodic(G(c["dims"], c["a0"]), K(k), c["T"])
    assert np.abs(out.data - np.array(c["want"], float)).max() <= c["tol"]
    for path in (0, 1):
        out = fs.solve_periodic(G(c["dims"], c["a0"]), K(k), c["T"], path=path)
        assert np.abs(out.data - np.array(c["want"], float)).max() <= 1e-10

    c = golden["shift_spectrum"]
    lam = fs.spectrum_from_kernel(K(R.kern_from({(1,): 1.0}, 1)), fs.GridShape(c["dims"]))
    want = np.array(c["want_re"]) + 1j * np.array(c["want_im"])
    assert np.abs(lam.blocks - want).max() < c["tol"]
    c = golden["appendix_generator"]
    lam = fs.spectrum_from_kernel(K(R.appendix_kernel()), fs.GridShape(c["dims"]))
    assert abs(lam.blocks[0] - complex(*c["want_lambda0"])) < c["tol"]
    c = golden["identity_spectrum"]
    lam = fs.spectrum_from_kernel(K(R.kern_from({(0, 0): 1.0}, 2)), fs.GridShape(c["dims"]))
    assert np.abs(lam.blocks - 1.0).max() < c["tol"]

    for name in ("fft_delta", "fft_ones"):
        c = golden[name]
        got = fs.multi_fft(fs.ComplexGrid(fs.GridShape(c["dims"]), np.array(c["input_re"], complex)))
        want = np.array(c["want_re"]) + 1j * np.array(c["want_im"])
        assert np.abs(got.data - want).max() <= c["tol"]

    c = golden["pow_scalar"]
    lam = fs.DiagonalSpectrum(fs.GridShape([2]), [complex(*v) for v in c["lambda"]])
    for chk in c["checks"]:
        got = fs.pow_spectrum(lam, chk["T"]).blocks[chk["index"]]
        if chk["tol"] == 0.0:
            assert got == complex(*chk["want"])
        else:
            assert abs(got - complex(*chk["want"])) < chk["tol"]
    c = golden["pinv"]
    got = fs.pseudo_inverse_spectrum(fs.DiagonalSpectrum(fs.GridShape([3]), [complex(*v) for v in c["lambda"]]))
    assert np.abs(got.blocks - np.array([complex(*v) for v in c["want"]])).max() < c["tol"]
    assert got.blocks[1] == 0


def test_golden_errors(golden):
    c = golden["blowup_numeric_error"]
    a = R.random_grid(Rng(c["seed"]), 16)
    k = R.kern_from({(0,): 1e8, (1,): 1e8}, 1)
    with pytest.raises(fs.NumericError):
        fs.solve_periodic(G([16], a), K(k), c["T"])
    with pytest.raises(fs.NumericError):
        fs.solve_periodic(G([16], a), K(k), c["T"], path=1)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_vector(G([8], np.zeros(8)), K(R.kern_from({(0,): 1.0}, 1)), 1)


def test_2d_fused_errors_and_identity(orc):
    """2D fused plan: the non-finite scan of the C2R rows raises
    NumericError (periodic.cpp:55-56); the identity stencil returns a0 to
    rounding."""
    dims = [512, 1024]
    a = orc.splitmix_fill(91, 512 * 1024, True)
    with pytest.raises(fs.NumericError):
        fs.solve_periodic(G(dims, a), K(R.kern_from({(0, 0): 2.0}, 2)), 2000)
    got = fs.solve_periodic(G(dims, a), K(R.kern_from({(0, 0): 1.0}, 2)), 12345).data
    assert np.max(np.abs(got - a)) <= 1e-13


def test_golden_cli_fixtures(golden, orc):
    c = golden["cli_verify_heat1d"]
    k = R.kern_from({tuple(o): v for o, v in zip(c["offsets"], c["values"])}, 1)
    a0 = orc.splitmix_fill(c["seed"], 256, True)
    fast = fs.solve_periodic(G([256], a0), K(k), c["T"]).data
    slow = orc.evolve_periodic_naive(a0, [256], 1, *k.arrays(), c["T"])
    assert np.abs(fast - slow).max() <= c["tol_rel1p"] * (1 + np.abs(slow).max())


# ------------------------------------------------------------------ FFT (proj/tests/test_fft.cpp)
def test_fft_vs_direct_dft():
    rng = Rng(23)
    for n in (7, 12, 15, 32, 1000):
        g = R.random_complex_grid(rng, n)
        got = fs.multi_fft(fs.ComplexGrid(fs.GridShape([n]), g)).data
        want = R.direct_dft(g)
        assert np.abs(got - want).max() <= 1e-10 * (1 + np.abs(want).max()), n


@pytest.mark.parametrize("dims", [[1000], [3001], [12289], [40000], [300, 50], [24, 777], [7, 12, 513]])
def test_bluestein_axes_vs_numpy(dims):
    """Non-pow2 axes above 256 run the GPU Bluestein transform (fft.cpp:103-139):
    forward and inverse against numpy, including lengths past the old
    direct-DFT cap and a P > 8192 (split) convolution."""
    rng = np.random.default_rng(sum(dims))
    z = rng.standard_normal(int(np.prod(dims))) + 1j * rng.standard_normal(int(np.prod(dims)))
    shape = fs.GridShape(dims)
    got = fs.multi_fft(fs.ComplexGrid(shape, z)).data
    want = np.fft.fftn(z.reshape(dims)).reshape(-1)
    assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max(), dims
    back = fs.multi_ifft(fs.ComplexGrid(shape, want)).data  # normalized (fft.cpp:151-154)
    assert np.abs(back - z).max() <= 1e-11 * np.abs(z).max(), dims


@pytest.mark.parametrize("dims,T", [([20000], 300), ([1000, 300], 40), ([4097], 1000)])
def test_bluestein_solve_vs_oracle(orc, dims, T):
    """solve_periodic on non-pow2 grids beyond the direct-DFT range (general
    plan + Bluestein) vs the oracle (which runs the reference's Bluestein)."""
    k = R.random_kernel(Rng(300 + T), len(dims), 2, 1, 0.95)
    a0 = orc.splitmix_fill(77, int(np.prod(dims)), True)
    got = fs.solve_periodic(G(dims, a0), K(k), T).data
    want = orc.solve_periodic(a0, dims, 1, *k.arrays(), T)
    assert rel_l2(got, want) <= 1e-10


def test_multi_fft_vs_nested_sum():
    rng = Rng(29)
    for dims, m in (([12], 1), ([6, 10], 2), ([3, 4, 5], 1), ([16, 32], 1), ([8, 4, 64], 2)):
        g = R.random_complex_grid(rng, int(np.prod(dims)) * m)
        shape = fs.GridShape(dims, m)
        got = fs.multi_fft(fs.ComplexGrid(shape, g)).data
        want = R.direct_multi_dft(g, dims, m)
        assert np.abs(got - want).max() <= 1e-10 * (1 + np.abs(want).max())
        goti = fs.multi_ifft(fs.ComplexGrid(shape, g)).data
        wanti = R.direct_multi_dft(g, dims, m, inverse=True)
        assert np.abs(goti - wanti).max() <= 1e-10


def test_fft_round_trip_and_vs_oracle(orc):
    rng = Rng(31)
    for dims, m in (([7], 1), ([12], 1), ([64, 64], 1), ([17, 241], 1), ([11, 13, 5], 2), ([1, 9], 1),
                    ([4096], 1), ([8192], 1), ([1 << 15], 1), ([1 << 17], 2), ([512, 1024], 1)):
        g = R.random_complex_grid(rng, int(np.prod(dims)) * m) if np.prod(dims) < 5000 else \
            (np.random.default_rng(7).uniform(-1, 1, int(np.prod(dims)) * m)
             + 1j * np.random.default_rng(8).uniform(-1, 1, int(np.prod(dims)) * m))
        shape = fs.GridShape(dims, m)
        fwd = fs.multi_fft(fs.ComplexGrid(shape, g))
        back = fs.multi_ifft(fwd).data
        assert np.abs(back - g).max() <= 1e-10 * (1 + np.abs(g).max()), dims
        want = orc.multi_fft(g, dims, m)
        assert rel_l2(fwd.data, want) <= 1e-13, dims


# ------------------------------------------------------------------ spectral (proj/tests/test_spectral.cpp)
def test_spectrum_vs_oracle_and_dense(orc):
    rng = Rng(37)
    for _ in range(12):
        rank = 1 + rng.next() % 2
        m = 1 + rng.next() % 2
        dims = [rng.range(2, 16 if rank == 1 else 4) for _ in range(rank)]
        if np.prod(dims) > 16:
            continue
        k = R.random_kernel(rng, rank, max(min(1, min(dims) - 1), 0), m)
        if k.max_reach()[0] >= min(dims):
            continue
        lam = fs.spectrum_from_kernel(K(k), fs.GridShape(dims, m)).blocks
        want = orc.spectrum_from_kernel(dims, m, *k.arrays())
        assert np.abs(lam - want).max() <= 1e-12
        S = orc.dense_stencil_matrix(dims, m, *k.arrays()).astype(complex)
        conj = R.dense_dft_matrix(dims, m) @ S @ R.dense_idft_matrix(dims, m)
        lam3 = lam.reshape(-1, m, m)
        for r in range(S.shape[0]):
            for c in range(S.shape[0]):
                w = lam3[r // m, r % m, c % m] if r // m == c // m else 0.0
                assert abs(conj[r, c] - w) <= 1e-10


def test_pow_hadamard_multiply(orc):
    rng = Rng(41)
    lam = np.zeros((3, 2, 2), complex)
    for j in range(3):
        a, b, c = 0.9 * rng.symmetric(), 0.3 * rng.symmetric(), rng.symmetric()
        lam[j] = [[complex(a, b), c], [0, 1]]
    got = fs.pow_spectrum(fs.DiagonalSpectrum(fs.GridShape([3], 2), lam), 8).blocks.reshape(3, 2, 2)
    for j in range(3):
        want = np.linalg.matrix_power(lam[j], 8)
        assert np.abs(got[j] - want).max() <= 1e-12 * (1 + np.abs(want).max())
    rng = Rng(43)
    shape = fs.GridShape([8, 3])
    L = fs.DiagonalSpectrum(shape, [complex(rng.symmetric(), rng.symmetric()) for _ in range(24)])
    for a, b in ((3, 5), (1, 31), (16, 16), (0, 32)):
        lhs = fs.pow_spectrum(L, a + b).blocks
        prod = fs.multiply_spectra(fs.pow_spectrum(L, a), fs.pow_spectrum(L, b)).blocks
        assert np.abs(lhs - prod).max() <= 1e-10 * (1 + np.abs(lhs).max())
    rng = Rng(47)
    shape = fs.GridShape([4], 2)
    x = fs.ComplexGrid(shape, R.random_complex_grid(rng, 8))
    ident = fs.DiagonalSpectrum(shape, np.tile(np.eye(2), (4, 1, 1)))
    assert np.abs(fs.hadamard(ident, x).data - x.data).max() <= 1e-15
    lamr = np.array([[[complex(rng.symmetric(), rng.symmetric()) for _ in range(2)] for _ in range(2)]
                     for _ in range(4)])
    y = fs.hadamard(fs.DiagonalSpectrum(shape, lamr), x).data
    assert np.abs(y - orc.hadamard(lamr, x.data, [4], 2)).max() <= 1e-15
    with pytest.raises(fs.SpecError):
        fs.hadamard(ident, fs.ComplexGrid(fs.GridShape([5], 2)))
    with pytest.raises(fs.SpecError):
        fs.pseudo_inverse_spectrum(fs.DiagonalSpectrum(fs.GridShape([3], 2)))


# ------------------------------------------------------------------ periodic (proj/tests/test_periodic.cpp)
def test_identity_any_T():
    a = R.random_grid(Rng(53), 64)
    k = K(R.kern_from({(0,): 1.0}, 1))
    for T in (1, 97, 1 << 40):
        for path in (0, 1):
            assert np.abs(fs.solve_periodic(G([64], a), k, T, path=path).data - a).max() <= 1e-12


def test_heat_vs_naive(orc):
    a = R.random_grid(Rng(59), 32)
    k = R.heat1d(0.125)
    fast = fs.solve_periodic(G([32], a), K(k), 100).data
    slow = orc.evolve_periodic_naive(a, [32], 1, *k.arrays(), 100)
    assert np.abs(fast - slow).max() <= 1e-9 * (1 + np.abs(slow).max())


def test_T0_bit_exact():
    rng = Rng(61)
    a = R.random_grid(rng, 64)
    k = R.random_kernel(rng, 2, 1)
    assert (fs.solve_periodic(G([8, 8], a), K(k), 0).data == a).all()


@pytest.mark.parametrize("path", [0, 1])
def test_randomized_vs_naive(orc, path):
    """test_periodic.cpp:64-84 and acceptance criterion 2 (dims 4..32 incl. primes)."""
    rng = Rng(67)
    times = (0, 1, 2, 3, 7, 16, 100)
    for trial in range(40):
        rank = 1 + rng.next() % 3
        dims = [rng.range(4, 12 if rank == 3 else 32) for _ in range(rank)]
        m = 2 if trial % 4 == 0 else 1
        k = R.random_kernel(rng, rank, rng.range(1, 2), m)
        a = R.random_grid(rng, int(np.prod(dims)) * m)
        T = times[rng.next() % 7]
        fast = fs.solve_periodic(G(dims, a, m), K(k), T, path=path).data
        slow = orc.evolve_periodic_naive(a, dims, m, *k.arrays(), T)
        assert np.abs(fast - slow).max() <= 1e-8 * (1 + np.abs(slow).max()), (dims, m, T)


def test_acceptance_oracle_equivalence(orc):
    """proj/tests/acceptance.cpp:82-107 (300 cases, dims 4..32, target norm 0.95)."""
    rng = Rng(2002)
    times = (0, 1, 2, 3, 7, 16, 100)
    worst = 0.0
    for trial in range(300):
        rank = 1 + rng.next() % 3
        dims = [rng.range(4, 32) for _ in range(rank)]
        m = 2 if trial % 5 == 0 else 1
        k = R.random_kernel(rng, rank, rng.range(1, 2), m, 0.95)
        a = R.random_grid(rng, int(np.prod(dims)) * m)
        T = times[rng.next() % 7]
        fast = fs.solve_periodic(G(dims, a, m), K(k), T).data
        slow = orc.evolve_periodic_naive(a, dims, m, *k.arrays(), T)
        worst = max(worst, np.abs(fast - slow).max() / (1 + np.abs(slow).max()))
    assert worst <= 1e-8


def test_semigroup_shift_vector_affine(orc):
    rng = Rng(71)
    k = K(R.heat1d(0.2))
    a = R.random_grid(rng, 48)
    for s, t in ((3, 5), (31, 33), (64, 1)):
        whole = fs.solve_periodic(G([48], a), k, s + t).data
        split = fs.solve_periodic(fs.solve_periodic(G([48], a), k, s), k, t).data
        assert np.abs(whole - split).max() <= 1e-9 * (1 + np.abs(whole).max())
    rng = Rng(73)
    dims = [10, 12]
    kk = R.random_kernel(rng, 2, 1)
    a = R.random_grid(rng, 120)
    lhs = fs.solve_periodic(G(dims, R.rotate_grid(a, dims, 1, (3, 7))), K(kk), 9).data
    rhs = R.rotate_grid(fs.solve_periodic(G(dims, a), K(kk), 9).data, dims, 1, (3, 7))
    assert np.abs(lhs - rhs).max() <= 1e-10
    # block-diagonal kernels decouple (test_periodic.cpp:109-139)
    k0, k1 = K(R.heat1d(0.125)), K(R.heat1d(0.25))
    e01, e10 = fs.StencilKernel(1), fs.StencilKernel(1)
    e01.add_tap([0], 0.0)
    e10.add_tap([0], 0.0)
    folded = fs.fold_kernels([[k0, e01], [e10, k1]])
    a = R.random_grid(Rng(79), 32)
    whole = fs.solve_periodic_vector(G([16], a, 2), folded, 20).data
    f0 = fs.solve_periodic(G([16], a[0::2]), k0, 20).data
    f1 = fs.solve_periodic(G([16], a[1::2]), k1, 20).data
    assert np.abs(whole[0::2] - f0).max() <= 1e-12 * (1 + np.abs(f0).max())
    assert np.abs(whole[1::2] - f1).max() <= 1e-12 * (1 + np.abs(f1).max())
    assert (fs.solve_periodic_vector(G([16], a, 2), folded, 0).data == a).all()
    # affine encoding (test_periodic.cpp:141-182)
    rng = Rng(83)
    n, T, c = 64, 50, 0.37
    s = R.heat1d(0.125)
    fk = fs.StencilKernel(1, 2)
    for off, blk in s.taps.items():
        fk.add_tap(off, [[blk[0, 0], 0.0], [0.0, 0.0]])
    fk.add_tap([0], [[0.0, 1.0], [0.0, 1.0]])
    a = np.zeros(2 * n)
    direct = np.zeros(n)
    for i in range(n):
        v = rng.symmetric()
        a[2 * i], a[2 * i + 1], direct[i] = v, c, v
    fast = fs.solve_periodic_vector(G([n], a, 2), fk, T).data
    for _ in range(T):
        direct = orc.step_periodic(direct, [n], 1, *s.arrays()) + c
    assert np.abs(fast[0::2] - direct).max() <= 1e-9


def test_implicit(orc):
    ident = K(R.kern_from({(0,): 1.0}, 1))
    s = K(R.heat1d(0.125))
    a = R.random_grid(Rng(89), 24)
    imp = fs.solve_periodic_implicit(ident, s, G([24], a), 13).data
    exp = fs.solve_periodic(G([24], a), s, 13).data
    assert np.abs(imp - exp).max() <= 1e-12
    assert (fs.solve_periodic_implicit(ident, s, G([24], a), 0).data == a).all()
    beta = 0.125
    q = R.kern_from({(-1,): -beta, (0,): 1 + 2 * beta, (1,): -beta}, 1)
    sk = R.kern_from({(-1,): beta, (0,): 1 - 2 * beta, (1,): beta}, 1)
    a0 = R.random_grid(Rng(97), 16)
    Q = orc.dense_stencil_matrix([16], 1, *q.arrays())
    S = orc.dense_stencil_matrix([16], 1, *sk.arrays())
    state = a0.copy()
    for t in range(1, 4):
        state = np.linalg.solve(Q, S @ state)
        got = fs.solve_periodic_implicit(K(q), K(sk), G([16], a0), t).data
        assert np.abs(got - state).max() <= 1e-9
        want = orc.solve_periodic_implicit(a0, [16], q.arrays(), sk.arrays(), t)
        assert np.abs(got - want).max() <= 1e-12


@pytest.mark.parametrize("dims,T", [([1024, 256], 200), ([512, 64, 32], 30), ([2048, 128], 1), ([512, 2048], 40)])
def test_implicit_fused_vs_oracle(orc, dims, T):
    """solve_periodic_implicit on the fused plan (real symbols, N0 in the TMA
    multiplier path): Crank-Nicolson q = I - (b/2) L, s = I + (b/2) L of the
    axial Laplacian, vs the oracle (periodic.cpp:108-124)."""
    r = len(dims)
    b = 0.2
    qd, sd = {(0,) * r: 1.0 + b * r}, {(0,) * r: 1.0 - b * r}
    for a in range(r):
        for sgn in (-1, 1):
            off = tuple(sgn if i == a else 0 for i in range(r))
            qd[off], sd[off] = -b / 2, b / 2
    q, sk = R.kern_from(qd, r), R.kern_from(sd, r)
    a0 = orc.splitmix_fill(61 + T, int(np.prod(dims)), True)
    got = fs.solve_periodic_implicit(K(q), K(sk), G(dims, a0), T).data
    want = orc.solve_periodic_implicit(a0, dims, q.arrays(), sk.arrays(), T)
    assert rel_l2(got, want) <= 1e-10


def test_implicit_fused_pinv_threshold(orc):
    """A singular mass kernel (the Laplacian itself: lamQ(0) = 0) exercises the
    1e-12 max|lamQ| pseudo-inverse threshold on the fused plan."""
    dims = [1024, 128]
    q = R.kern_from({(0, 0): 4.0, (1, 0): -1.0, (-1, 0): -1.0, (0, 1): -1.0, (0, -1): -1.0}, 2)
    sk = R.kern_from({(0, 0): 0.5, (1, 0): 0.125, (-1, 0): 0.125, (0, 1): 0.125, (0, -1): 0.125}, 2)
    a0 = orc.splitmix_fill(73, 1024 * 128, True)
    got = fs.solve_periodic_implicit(K(q), K(sk), G(dims, a0), 3).data
    want = orc.solve_periodic_implicit(a0, dims, q.arrays(), sk.arrays(), 3)
    assert rel_l2(got, want) <= 1e-10


def test_cached_and_timings():
    cache = fs.SpectrumCache()
    a = R.random_grid(Rng(5), 4096)
    k = K(R.heat1d(0.25))
    st = fs.StageTimings()
    out1 = fs.solve_periodic_cached(G([64, 64], a), K(R.random_kernel(Rng(6), 2, 1)), 9, cache, st)
    out2 = fs.solve_periodic(G([64, 64], a), K(R.random_kernel(Rng(6), 2, 1)), 9)
    assert np.abs(out1.data - out2.data).max() == 0.0
    assert st.sum() > 0 and st.forward_fft > 0 and st.inverse_fft > 0
    before = st.sum()
    fs.solve_periodic(G([4096], a), k, 5, st)
    assert st.sum() > before  # accumulated, not reset


def test_cache_is_keyed_by_dims_only():
    """SpectrumCache::get (periodic.cpp:67-74) memoises by dims alone: a later
    call with the same dims but another kernel reuses the first kernel's
    spectrum; other dims get their own.  The passed kernel is still checked
    by require_fits."""
    cache = fs.SpectrumCache()
    a = R.random_grid(Rng(15), 64 * 32)
    kA, kB = K(R.random_kernel(Rng(16), 2, 1)), K(R.random_kernel(Rng(17), 2, 1))
    first = fs.solve_periodic_cached(G([64, 32], a), kA, 4, cache).data
    again = fs.solve_periodic_cached(G([64, 32], a), kB, 4, cache).data
    assert np.array_equal(first, fs.solve_periodic(G([64, 32], a), kA, 4).data)
    assert np.array_equal(again, first)
    other = fs.solve_periodic_cached(G([32, 64], a), kB, 4, cache).data
    assert np.array_equal(other, fs.solve_periodic(G([32, 64], a), kB, 4).data)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_cached(G([1, 1], a[:1]), kB, 4, cache)


# ------------------------------------------------------------------ per-plan parity vs the oracle
PLAN_CASES = [
    # (dims, m, taps-kind, T)   fused R2C rank 2/3, 1D row-pair (m = 1, 2), general
    ([256, 256], 1, "box9", 1000),
    ([128, 512], 1, "jacobi5", 100),
    ([64, 32, 128], 1, "heat7", 50),
    ([32, 64, 16], 1, "random", 7),
    ([1 << 12], 1, "heat3", 1000),
    ([1 << 16], 1, "heat3", 1000),
    ([1 << 12], 2, "leapfrog", 1000),
    ([1 << 14], 2, "leapfrog", 5000),
    ([96, 40], 1, "random", 11),
    ([1 << 14, 2], 1, "random", 3),
    ([8192, 64], 1, "box9", 1000),       # 8192-point fused columns (parity halves)
    ([4, 64], 1, "jacobi5", 30),         # axis 0 below the fused kernels' range: general plan
    ([2, 32, 16], 1, "random", 5),
    ([8, 16, 32], 1, "heat7", 9),
    ([16, 2, 32], 1, "heat7", 7),        # 2-point axis-1 pass
    ([16, 4, 64], 1, "random", 3),
    ([8192, 32], 1, "random", 5),        # ... with a complex symbol
    # 2D fused plan across row lengths and TMA tile widths
    ([512, 1024], 1, "random", 13),      # L = 1024, 8-column tiles, complex symbol
    ([1024, 2048], 1, "box9", 1000),     # L = 2048, 4-column tiles
    ([2048, 4096], 1, "jacobi5", 500),   # L = 4096, 2-column tiles
    ([4096, 1024], 1, "random", 3),      # one-column tiles
    ([512, 4096], 1, "box9", 100000),
]


def _case_kernel(kind, rank, seed):
    rng = Rng(seed)
    if kind == "box9":
        u = [rng.uniform() for _ in range(9)]
        offs = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1)]
        return R.kern_from({o: w / sum(u) for o, w in zip(offs, u)}, 2)
    if kind == "jacobi5":
        return R.kern_from({(0, 0): 0.2, (1, 0): 0.2, (-1, 0): 0.2, (0, 1): 0.2, (0, -1): 0.2}, 2)
    if kind == "heat7":
        t = {(0, 0, 0): 0.4}
        for a in range(3):
            for s in (-1, 1):
                o = [0, 0, 0]
                o[a] = s
                t[tuple(o)] = 0.1
        return R.kern_from(t, 3)
    if kind == "heat3":
        return R.kern_from({(-1,): 0.25, (0,): 0.5, (1,): 0.25}, 1)
    if kind == "leapfrog":
        C2 = 0.25
        k = R.Kern(1, 2)
        k.add((0,), [[2 - 2 * C2, -1.0], [1.0, 0.0]])
        k.add((-1,), [[C2, 0.0], [0.0, 0.0]])
        k.add((1,), [[C2, 0.0], [0.0, 0.0]])
        return k
    return R.random_kernel(rng, rank, 1, 1, 0.95)


@pytest.mark.parametrize("dims,m,kind,T", PLAN_CASES)
def test_plans_vs_oracle(orc, dims, m, kind, T):
    k = _case_kernel(kind, len(dims), 1000 + T)
    n = int(np.prod(dims)) * m
    a0 = orc.splitmix_fill(7 + len(dims), n, True)
    want = orc.solve_periodic(a0, dims, m, *k.arrays(), T)
    truth = orc.solve_periodic_ld(a0, dims, m, *k.arrays(), T) if kind == "leapfrog" else None
    for path in (0, 1):
        got = fs.solve_periodic(G(dims, a0, m), K(k), T, path=path).data
        if truth is None:
            assert rel_l2(got, want) <= 1e-10, (dims, m, kind, T, path, rel_l2(got, want))
        else:
            # cfg5 family: the leapfrog symbol is a near-Jordan block at low
            # frequency, so two fp64 pipelines legitimately differ by more than
            # 1e-10.  Protocol: against the
            # long-double truth, the GPU error must not exceed the oracle's.
            e_gpu, e_orc = rel_l2(got, truth), rel_l2(want, truth)
            assert e_gpu <= max(1e-12, 1.5 * e_orc), (dims, path, e_gpu, e_orc)
    info = fs.plan_describe(fs.GridShape(dims, m), K(k))
    assert info["path"] in (1, 2, 3)


def test_plan_kinds_selected():
    k2 = K(_case_kernel("jacobi5", 2, 0))
    assert fs.plan_describe(fs.GridShape([4096, 4096]), k2)["path"] == 1
    k3 = K(_case_kernel("heat7", 3, 0))
    assert fs.plan_describe(fs.GridShape([64, 64, 64]), k3)["path"] == 1
    assert fs.plan_describe(fs.GridShape([1 << 20]), K(_case_kernel("heat3", 1, 0)))["path"] == 2
    assert fs.plan_describe(fs.GridShape([1 << 20], 2), K(_case_kernel("leapfrog", 1, 0)))["path"] == 2
    assert fs.plan_describe(fs.GridShape([12, 12]), k2)["path"] == 3


# ------------------------------------------------------------------ configs (BASELINE) at full or reduced size
def test_cfg1_full_vs_oracle(orc):
    """cfg1: 1D heat N=2^20, T=1000 (BASELINE configs[0]) at full size."""
    k = _case_kernel("heat3", 1, 0)
    a0 = orc.splitmix_fill(1, 1 << 20, False)
    want = orc.solve_periodic(a0, [1 << 20], 1, *k.arrays(), 1000)
    got = fs.solve_periodic(G([1 << 20], a0), K(k), 1000).data
    assert rel_l2(got, want) <= 1e-10


def test_cfg2_full_vs_oracle_and_properties(orc):
    """cfg2: 2D Jacobi 4096^2, T=1e4 at full size: vs the oracle, vs the
    independent general GPU pipeline, and the semigroup property."""
    k = _case_kernel("jacobi5", 2, 0)
    dims = [4096, 4096]
    a0 = orc.splitmix_fill(2, 4096 * 4096, False)
    got = fs.solve_periodic(G(dims, a0), K(k), 10000).data
    want = orc.solve_periodic(a0, dims, 1, *k.arrays(), 10000)
    assert rel_l2(got, want) <= 1e-10
    half = fs.solve_periodic(fs.solve_periodic(G(dims, a0), K(k), 5000), K(k), 5000).data
    assert rel_l2(half, got) <= 1e-10


def test_cfg3_reduced_vs_oracle(orc):
    """cfg3 shape family (9-point random box, T=1e5) at 1024^2 vs the oracle."""
    k = _case_kernel("box9", 2, 1003)
    dims = [1024, 1024]
    a0 = orc.splitmix_fill(3, 1024 * 1024, True)
    got = fs.solve_periodic(G(dims, a0), K(k), 100000).data
    want = orc.solve_periodic(a0, dims, 1, *k.arrays(), 100000)
    assert rel_l2(got, want) <= 1e-10


def test_cfg4_reduced_vs_oracle(orc):
    """cfg4 family (3D 7-point heat, T=1000) at 64^3 vs the oracle."""
    k = _case_kernel("heat7", 3, 0)
    dims = [64, 64, 64]
    a0 = orc.splitmix_fill(4, 64 ** 3, False)
    got = fs.solve_periodic(G(dims, a0), K(k), 1000).data
    want = orc.solve_periodic(a0, dims, 1, *k.arrays(), 1000)
    assert rel_l2(got, want) <= 1e-10


# ------------------------------------------------------------------ 1D row-pair plan with a split column FFT
@pytest.mark.parametrize("n,m,kind,T", [(1 << 16, 2, "leapfrog", 3000), (1 << 15, 1, "heat3", 500),
                                        (1 << 14, 1, "random", 9)])
def test_rowpair_split_columns(orc, monkeypatch, n, m, kind, T):
    """The 2^26 cfg5 layout (column FFT split 128 x 128, rows digit-reversed)
    forced at small N via FSX_COLSPLIT (read when the plan is created)."""
    monkeypatch.setenv("FSX_COLSPLIT", "8")
    k = _case_kernel(kind, 1, 2000 + T)
    a0 = orc.splitmix_fill(11, n * m, True)
    want = orc.solve_periodic(a0, [n], m, *k.arrays(), T)
    # a shape not used elsewhere so the split plan is built here: add a length-1 axis
    got = fs.solve_periodic(G([1, n], a0, m), _K2(k), T).data
    if kind == "leapfrog":
        truth = orc.solve_periodic_ld(a0, [n], m, *k.arrays(), T)
        assert rel_l2(got, truth) <= max(1e-12, 1.5 * rel_l2(want, truth))
    else:
        assert rel_l2(got, want) <= 1e-10
    assert fs.plan_describe(fs.GridShape([1, n], m), _K2(k))["path"] == 2


def _K2(k: R.Kern):
    """The same taps on a [1, n] grid (leading length-1 axis, offset 0)."""
    out = fs.StencilKernel(2, k.fields)
    for off in sorted(k.taps):
        out.add_tap((0,) + tuple(off), k.taps[off] if k.fields > 1 else float(k.taps[off][0, 0]))
    return out


def test_cfg5_protocol(orc):
    """cfg5 (leapfrog 2-field system, C = 0.5, T = 1e6, Gaussian bumps).
    Full size 2^26 runs the fused row-pair plan (split column FFT) and must be
    finite.  Parity follows the SURVEY 8c protocol at N = 2^16 with the same
    stencil, T and initial-state family: against the long-double truth the
    GPU error must not exceed the fp64 oracle's (the config is fp64
    ill-conditioned, so GPU-vs-oracle itself is not 1e-10)."""
    from paper_2105_06676_b200.synthetic import configs, leapfrog_bumps

    cfg = configs()["cfg5"]
    got = fs.solve_periodic(G(cfg.dims, cfg.initial(), 2), cfg.kernel(), cfg.T).data
    assert np.isfinite(got).all()
    assert fs.plan_describe(fs.GridShape(cfg.dims, 2), cfg.kernel())["path"] == 2
    off, blk = cfg.kernel().arrays()
    for n in (1 << 12, 1 << 14, 1 << 16):
        a0 = leapfrog_bumps(n, cfg.seed + 1000, K=4, width=64.0)
        truth = orc.solve_periodic_ld(a0, [n], 2, off, blk, cfg.T)
        mine = fs.solve_periodic(G([n], a0, 2), cfg.kernel(), cfg.T).data
        e_gpu = rel_l2(mine, truth)
        try:
            want = orc.solve_periodic(a0, [n], 2, off, blk, cfg.T)
        except orc.OracleNumericError:
            # the fp64 reference path itself gives up here: its imaginary
            # residue exceeds 1e-6 max|real| (proj/src/periodic.cpp:60-63) --
            # measured at n = 2^16; the real-to-complex GPU path has no
            # imaginary part and stays close to the truth
            print(f"cfg5 protocol n={n}: GPU vs truth {e_gpu:.3e} (fp64 oracle raises NumericError)")
            assert e_gpu <= 1e-6, (n, e_gpu)
            continue
        e_orc = rel_l2(want, truth)
        print(f"cfg5 protocol n={n}: GPU vs truth {e_gpu:.3e}, fp64 oracle vs truth {e_orc:.3e}")
        assert e_gpu <= max(1e-12, 1.5 * e_orc), (n, e_gpu, e_orc)
        # the Cayley-Hamilton power (pow_real2_ch) keeps the GPU two orders
        # below the oracle's matrix loop here (measured 1.2e-8 / 3.0e-8 against
        # 3.3e-6 / 1.8e-5; scripts/pow_accuracy.py)
        assert e_gpu <= 1e-6, (n, e_gpu)


def cfg5_truth(cfg, a0, band_sigmas=7.0):
    """The exact answer of cfg5's problem (not of the fp64 reference): the
    Gaussian-bump state's spectrum (numpy fp64 FFT) times the T-th power of the
    symbol [[2 - 2C^2 + 2C^2 cos t, -1], [1, 0]] evaluated and raised in long
    double (Cayley-Hamilton doubling: 19 squarings, ~1e-8 worst relative at
    2^26 in long double) over the band that holds the bumps' energy (|U| above
    exp(-band_sigmas^2) of its peak); the rest of the spectrum is below 1e-20
    of the peak and is left at 0."""
    n = cfg.dims[0]
    U = np.fft.fft(a0[0::2])
    V = np.fft.fft(a0[1::2])
    w = 64.0  # leapfrog_bumps width
    kb = int(band_sigmas * n / (np.pi * w)) + 1
    k = np.concatenate([np.arange(0, kb), np.arange(n - kb, n)]).astype(np.longdouble)
    c = np.cos(2 * np.pi * k / np.longdouble(n))
    C2 = np.longdouble(0.25)
    t = 2 - 2 * C2 + 2 * C2 * c  # trace; det = 1
    p = np.ones_like(t)
    tr = t.copy()
    for b in bin(cfg.T)[3:]:
        p, tr = p * tr, tr * tr - 2
        if b == "1":
            pn = (p * t + tr) / 2
            tr, p = pn * t - 2 * p, pn
    q = (tr - p * t) / 2
    A00, A01, A10, A11 = p * t + q, -p, p, q
    idx = np.concatenate([np.arange(0, kb), np.arange(n - kb, n)])
    Uo = np.zeros(n, complex)
    Vo = np.zeros(n, complex)
    Uo[idx] = A00.astype(np.float64) * U[idx] + A01.astype(np.float64) * V[idx]
    Vo[idx] = A10.astype(np.float64) * U[idx] + A11.astype(np.float64) * V[idx]
    out = np.empty(2 * n)
    out[0::2] = np.fft.ifft(Uo).real
    out[1::2] = np.fft.ifft(Vo).real
    return out


def test_cfg5_full_size_vs_truth():
    """cfg5 at its full size (N = 2^26 x 2 fields, T = 1e6, BASELINE's bumps)
    against the exact answer (cfg5_truth).  The fp64 reference cannot be the
    yardstick here: its matrix-power loop is off by up to 12x per low
    frequency at this N and T (scripts/pow_accuracy.py)."""
    from paper_2105_06676_b200.synthetic import configs

    cfg = configs()["cfg5"]
    a0 = cfg.initial()
    got = fs.solve_periodic(G(cfg.dims, a0, 2), cfg.kernel(), cfg.T).data
    truth = cfg5_truth(cfg, a0)
    e = rel_l2(got, truth)
    print(f"cfg5 full size (2^26 x 2, T=1e6): GPU vs exact rel L2 {e:.3e}")
    assert e <= 1e-5, e


# ------------------------------------------------------------------ pipelined batch API
@pytest.mark.parametrize("dims,m,kind,T", [([256, 128], 1, "box9", 1000), ([1 << 14], 2, "leapfrog", 500),
                                          ([32, 16, 64], 1, "heat7", 40)])
def test_batch_equals_single_solves(orc, dims, m, kind, T):
    """fsx_solve_periodic_batch: each item bitwise equal to its own solve_periodic
    (two lanes = two plan copies running the same kernels)."""
    k = K(_case_kernel(kind, len(dims), 9000 + T))
    n = int(np.prod(dims)) * m
    grids = [G(dims, orc.splitmix_fill(300 + i, n, True), m) for i in range(5)]
    outs = fs.solve_periodic_batch(grids, k, T)
    for g, o in zip(grids, outs):
        assert np.array_equal(o, fs.solve_periodic(g, k, T).data)
    assert fs.solve_periodic_batch([], k, T) == []
    same = fs.solve_periodic_batch(grids[:2], k, 0)
    assert np.array_equal(same[1], grids[1].data)


def test_batch_reports_failing_item():
    """A non-finite input in item 2 raises NumericError naming it (realize_checked)."""
    k = fs.StencilKernel(2).add_tap([0, 0], 0.5).add_tap([1, 0], 0.25).add_tap([0, -1], 0.25)
    grids = [G([64, 64], np.random.default_rng(i).random(4096)) for i in range(4)]
    grids[2].data[17] = np.nan
    with pytest.raises(fs.NumericError, match="batch item 2"):
        fs.solve_periodic_batch(grids, k, 10)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_batch([grids[0], G([32, 32], np.zeros(1024))], k, 10)


@pytest.mark.parametrize("dims,m,T", [([32, 16], 5, 7), ([64], 8, 5), ([8, 4, 6], 6, 3)])
def test_many_fields_vs_oracle(orc, dims, m, T):
    """m-vector cells beyond the 2-field fast plans (general plan, block symbol
    and block power for m up to 8; periodic.cpp:101-106 with Eigen blocks)."""
    k = R.random_kernel(Rng(500 + m), len(dims), 1, m, 0.9)
    a0 = orc.splitmix_fill(90 + m, int(np.prod(dims)) * m, True)
    got = fs.solve_periodic_vector(G(dims, a0, m), K(k), T).data
    want = orc.solve_periodic(a0, dims, m, *k.arrays(), T, vector=True)
    assert rel_l2(got, want) <= 1e-10
