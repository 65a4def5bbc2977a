"""fp32 mode (north star: an optional fp32 mode within 1e-4 relative L2 of
the reference's fp64 result).  Float32 grids in and out.  Where the fused
pass runs in fp32 arithmetic (plan 1, real symbol) the bar is 2e-6; elsewhere
the arithmetic is fp64 and the result must be the fp64 solve of the widened
input rounded once to float.  Covers the fused plan
(float row kernels), the 1D and general plans (widen / narrow around the fp64
buffers), the batch and device entry points, T = 0 and the overflow check."""
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

TOL = 1e-4           # the north star's fp32 bar
TIGHT = 2e-7         # one float rounding of the fp64 result (plus the fp64 path's own error)


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def K(k):
    out = fs.StencilKernel(k.rank, k.fields)
    for off in sorted(k.taps):
        out.add_tap(off, k.taps[off] if k.fields > 1 else float(k.taps[off][0, 0]))
    return out


HEAT7 = {(0, 0, 0): 0.4, (1, 0, 0): 0.1, (-1, 0, 0): 0.1, (0, 1, 0): 0.1, (0, -1, 0): 0.1, (0, 0, 1): 0.1,
         (0, 0, -1): 0.1}
CASES = [
    # (dims, m, taps, T, fp32 arithmetic in the fused pass)
    ([1024, 1024], 1, {(0, 0): 0.2, (1, 0): 0.2, (-1, 0): 0.2, (0, 1): 0.2, (0, -1): 0.2}, 10000, True),  # fused 2D
    ([64, 64, 64], 1, HEAT7, 1000, True),     # fused 3D, real symbol
    ([16, 512, 1024], 1, HEAT7, 300, True),   # 3D with fp32 TMA y passes (n1 = 512)
    ([64, 32, 128], 1, None, 50, False),      # fused 3D, random kernel: complex symbol -> fp64 pass
    ([1 << 16], 1, {(-1,): 0.25, (0,): 0.5, (1,): 0.25}, 1000, False),  # 1D row-pair plan
    ([96, 40], 1, None, 11, False),           # general plan
    ([256, 64], 2, None, 7, False),           # vector cells, general plan
]
F32_ARITH = 2e-6     # float FFTs in the fused pass, fp64 symbol power: measured ~1e-7


@pytest.mark.parametrize("dims,m,taps,T,f32c", CASES)
def test_f32_vs_oracle(orc, dims, m, taps, T, f32c):
    k = R.kern_from(taps, len(dims)) if taps else R.random_kernel(Rng(500 + T), len(dims), 1, m, 0.95)
    n = int(np.prod(dims)) * m
    a32 = orc.splitmix_fill(40 + len(dims), n, True).astype(np.float32)
    want = orc.solve_periodic(a32.astype(np.float64), dims, m, *k.arrays(), T)
    got = fs.solve_periodic_f32(fs.GridShape(dims, m), a32, K(k), T)
    assert got.dtype == np.float32
    e = rel_l2(got, want)
    assert e <= TOL, (dims, m, e)
    g64 = fs.solve_periodic(fs.FieldGrid(fs.GridShape(dims, m), a32.astype(np.float64)), K(k), T).data
    if f32c:
        assert e <= F32_ARITH, (dims, m, e)
    else:
        # fp64 arithmetic: the fp64 GPU solve of the widened input, rounded once
        assert e <= TIGHT, (dims, m, e)
        assert np.max(np.abs(got - g64.astype(np.float32))) <= 2 * np.finfo(np.float32).eps * np.max(np.abs(g64))


def test_f32_T0_bit_exact_and_batch_and_device(orc):
    dims = [512, 1024]
    k = K(R.kern_from({(0, 0): 0.5, (1, 1): 0.25, (-1, -1): 0.25}, 2))
    a = orc.splitmix_fill(77, 512 * 1024, True).astype(np.float32)
    assert (fs.solve_periodic_f32(fs.GridShape(dims), a, k, 0) == a).all()
    one = fs.solve_periodic_f32(fs.GridShape(dims), a, k, 300)
    outs = fs.solve_periodic_batch_f32(fs.GridShape(dims), [a, a * 2, a], k, 300)
    assert np.array_equal(outs[0], one) and np.array_equal(outs[2], one)
    assert rel_l2(outs[1], 2 * one.astype(np.float64)) <= 1e-6
    torch = pytest.importorskip("torch")
    d_in = torch.from_numpy(a).cuda()
    d_out = torch.empty_like(d_in)
    fs.solve_periodic_device_f32(fs.GridShape(dims), d_in.data_ptr(), k, 300, d_out.data_ptr(),
                                 stream=torch.cuda.current_stream().cuda_stream)
    fs.device_check(stream=torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(d_out.cpu().numpy(), one)


def test_f32_overflow_is_numeric_error(orc):
    # finite in fp64, beyond the float range: 1.5^300 ~ 1e52
    a = np.ones(256 * 256, np.float32)
    k = K(R.kern_from({(0, 0): 1.5}, 2))
    with pytest.raises(fs.NumericError):
        fs.solve_periodic_f32(fs.GridShape([256, 256]), a, k, 300)
    a1 = np.ones(1 << 12, np.float32)
    with pytest.raises(fs.NumericError):
        fs.solve_periodic_f32(fs.GridShape([1 << 12]), a1, K(R.kern_from({(0,): 1.5}, 1)), 300)


@pytest.mark.parametrize("m", [1, 2])
def test_f32_rowpair_split_columns(orc, monkeypatch, m):
    """The 1D plan's float I/O through the split column passes (the cfg5
    layout, forced small with FSX_COLSPLIT on a fresh [1, 1, n] shape): equal
    to the fp64 GPU solve of the widened input rounded once."""
    monkeypatch.setenv("FSX_COLSPLIT", "8")
    n = 1 << 15
    k = R.Kern(3, m)
    if m == 1:
        for o, c in ((-1, 0.25), (0, 0.5), (1, 0.25)):
            k.add((0, 0, o), [[c]])
    else:
        C2 = 0.25
        k.add((0, 0, 0), [[2 - 2 * C2, -1.0], [1.0, 0.0]])
        k.add((0, 0, -1), [[C2, 0.0], [0.0, 0.0]])
        k.add((0, 0, 1), [[C2, 0.0], [0.0, 0.0]])
    shape = fs.GridShape([1, 1, n], m)
    a32 = orc.splitmix_fill(17 + m, n * m, True).astype(np.float32)
    got = fs.solve_periodic_f32(shape, a32, K(k), 700)
    g64 = fs.solve_periodic(fs.FieldGrid(shape, a32.astype(np.float64)), K(k), 700).data
    assert np.max(np.abs(got - g64.astype(np.float32))) <= 2 * np.finfo(np.float32).eps * np.max(np.abs(g64))
    assert fs.plan_describe(shape, K(k))["path"] == 2
