"""Exact spectral cut (fsx_options.spectral_cut, 2D fused plan): the columns
whose multipliers provably underflow to 0 are neither stored, transformed
nor read.  The full solve makes those columns exactly 0, so the cut solve
must equal it bit for bit (up to the sign of an exact zero), and both must
match the oracle at the fp64 bar."""
import numpy as np
import pytest

import refutil as R
from refutil import Rng

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if fs.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tests must run on a B200")


def K(k):
    out = fs.StencilKernel(k.rank, k.fields)
    for off in sorted(k.taps):
        out.add_tap(off, float(k.taps[off][0, 0]))
    return out


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


JACOBI = {(0, 0): 0.2, (1, 0): 0.2, (-1, 0): 0.2, (0, 1): 0.2, (0, -1): 0.2}


def box9(seed):
    rng = Rng(seed)
    u = [rng.uniform() for _ in range(9)]
    offs = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1)]
    return {o: w / sum(u) for o, w in zip(offs, u)}


CASES = [
    ([1024, 1024], JACOBI, 10000, True),     # cfg2 family: real symbol
    ([1024, 1024], box9(1003), 100000, True),  # cfg3 family: complex symbol, halves not involved
    ([512, 2048], box9(7), 1000, False),      # 4-column tiles, L = 2048 (T too small: nothing provably 0)
    ([8192, 1024], JACOBI, 5000, True),       # 8192-point columns (parity halves pass)
    ([4096, 4096], JACOBI, 10000, True),      # cfg2 full size
    ([512, 8192], JACOBI, 20000, True),       # 4096-complex rows (three-stage row kernels)
    ([256, 1024], {(0, 0): 0.5, (0, 1): 0.5}, 300, True),   # complex, |lam| = |cos(theta_x / 2)|: top columns
]


@pytest.mark.parametrize("dims,taps,T,expect_cut", CASES)
def test_cut_bitwise_equal_and_vs_oracle(orc, dims, taps, T, expect_cut):
    k = R.kern_from(taps, 2)
    n = int(np.prod(dims))
    a0 = orc.splitmix_fill(11 + T % 7, n, True)
    g = fs.FieldGrid(fs.GridShape(dims), a0)
    full = fs.solve_periodic(g, K(k), T).data
    cut = fs.solve_periodic(g, K(k), T, spectral_cut=1).data
    assert np.array_equal(full, cut)
    kept, total = fs.spectral_cut_columns(fs.GridShape(dims), K(k), T)
    assert total == dims[1] // 2 + 1 and 1 <= kept <= total
    if expect_cut:
        assert kept < total
    if n <= 1 << 21:
        want = orc.solve_periodic(a0, dims, 1, *k.arrays(), T)
        assert rel_l2(cut, want) <= 1e-10


@pytest.mark.parametrize("dims,taps,T,expect_cut", CASES + [([8192, 2048], box9(5), 100000, True)])
def test_zero_column_shortcut_is_bitwise(orc, dims, taps, T, expect_cut, monkeypatch):
    """The default fused pass takes the multipliers of host-proved zero columns as 0 without
    evaluating the symbol (FusedSymbol::kzero); FSX_ZEROCOL=0 evaluates every column.  Same
    bits, including the sign of every zero."""
    k = R.kern_from(taps, 2)
    n = int(np.prod(dims))
    a0 = orc.splitmix_fill(5 + T % 11, n, True)
    g = fs.FieldGrid(fs.GridShape(dims), a0)
    monkeypatch.setenv("FSX_ZEROCOL", "1")
    fast = fs.solve_periodic(g, K(k), T).data
    monkeypatch.setenv("FSX_ZEROCOL", "0")
    slow = fs.solve_periodic(g, K(k), T).data
    assert np.array_equal(fast.view(np.int64), slow.view(np.int64))


def test_cut_does_not_apply():
    shape = fs.GridShape([64, 64, 64])
    k3 = R.kern_from({(0, 0, 0): 0.4, (1, 0, 0): 0.3, (-1, 0, 0): 0.3}, 3)
    kept, total = fs.spectral_cut_columns(shape, K(k3), 1000)
    assert kept == total                            # rank 3: no cut
    kept, total = fs.spectral_cut_columns(fs.GridShape([512, 512]), K(R.kern_from(JACOBI, 2)), 1)
    assert kept == total                            # T = 1: nothing underflows
    ident = R.kern_from({(0, 0): 1.0}, 2)
    kept, total = fs.spectral_cut_columns(fs.GridShape([512, 512]), K(ident), 10 ** 6)
    assert kept == total                            # |lam| = 1 everywhere
    chk = R.kern_from({(0, 1): 0.5, (0, -1): 0.5}, 2)   # lam = cos(theta_x): |lam| = 1 at kx = M
    kept, total = fs.spectral_cut_columns(fs.GridShape([512, 512]), K(chk), 10 ** 4)
    assert kept == total


def test_cut_nonfinite_and_batch(orc):
    dims = [1024, 1024]
    k = K(R.kern_from(JACOBI, 2))
    a = orc.splitmix_fill(5, 1024 * 1024, False)
    bad = a.copy()
    bad[12345] = np.nan
    with pytest.raises(fs.NumericError):
        fs.solve_periodic(fs.FieldGrid(fs.GridShape(dims), bad), k, 10000, spectral_cut=1)
    g = fs.FieldGrid(fs.GridShape(dims), a)
    one = fs.solve_periodic(g, k, 10000).data
    outs = fs.solve_periodic_batch([g, g, g], k, 10000, spectral_cut=1)
    for o in outs:
        assert np.array_equal(o, one)


def test_cut_f32_storage_mode(orc):
    """The cut composes with the fp32 storage mode (float rows, same columns)."""
    dims = [1024, 2048]
    k = K(R.kern_from(JACOBI, 2))
    a32 = orc.splitmix_fill(9, 1024 * 2048, False).astype(np.float32)
    full = fs.solve_periodic_f32(fs.GridShape(dims), a32, k, 20000)
    cut = fs.solve_periodic_f32(fs.GridShape(dims), a32, k, 20000, spectral_cut=1)
    assert np.array_equal(full, cut)
    assert fs.spectral_cut_columns(fs.GridShape(dims), k, 20000)[0] < 1025
