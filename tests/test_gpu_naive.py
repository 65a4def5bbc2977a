"""GPU direct-stepping verifier.

fsx_evolve_periodic_naive restates the reference's naive oracle
(proj/src/oracle.cpp:26-115): it must agree with the CPU oracle BIT FOR BIT
(same tap order, products and sums rounded separately), and it then gives a
full-size, FFT-free check of the solver at the BASELINE configs' shapes where
the CPU loop (N * T * taps operations) would take hours.

Tolerance for solver vs naive: relative L2 <= 1e-10 (BASELINE north_star),
except cfg5 (fp64-ill-conditioned leapfrog) whose bound is
stated in the test.
"""
import numpy as np
import pytest

import refutil as R
from refutil import Rng

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")
torch = pytest.importorskip("torch")
syn = pytest.importorskip("paper_2105_06676_b200.synthetic")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if fs.device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU verifier tests must run on a B200")


def K(k: R.Kern) -> "fs.StencilKernel":
    out = fs.StencilKernel(k.rank, k.fields)
    for off in sorted(k.taps):
        out.add_tap(off, k.taps[off] if k.fields > 1 else float(k.taps[off][0, 0]))
    return out


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _random_kernel(rank, m, ntaps, reach, seed):
    rng = Rng(seed)
    k = R.Kern(rank, m)
    for _ in range(ntaps):
        off = tuple(rng.range(-reach, reach) for _ in range(rank))
        blk = np.array([[rng.uniform() * 2 - 1 for _ in range(m)] for _ in range(m)]) * (0.9 / ntaps)
        k.add(off, blk)
    return k


NAIVE_CASES = [
    # dims, m, ntaps, reach, T
    ([257], 1, 5, 3, 13),
    ([33, 40], 1, 9, 2, 7),
    ([8, 12, 10], 1, 7, 2, 5),
    ([64], 2, 3, 1, 20),
    ([12, 9], 3, 4, 2, 4),
    ([4, 5, 3, 6], 1, 6, 1, 3),   # rank 4: the divide-decode path
    ([3, 4, 2, 5], 2, 4, 1, 2),
    ([1, 50], 1, 3, 0, 9),        # length-1 axis
]


@pytest.mark.parametrize("dims,m,ntaps,reach,T", NAIVE_CASES)
def test_naive_bitwise_vs_oracle(orc, dims, m, ntaps, reach, T):
    """oracle.cpp:100-115 evolve_periodic_naive: identical bits."""
    reach_fit = min(reach, min(dims) - 1)
    k = _random_kernel(len(dims), m, ntaps, reach_fit, 7000 + T)
    n = int(np.prod(dims)) * m
    a0 = orc.splitmix_fill(40 + T, n, True)
    got = fs.evolve_periodic_naive(fs.FieldGrid(fs.GridShape(dims, m), a0), K(k), T).data
    want = orc.evolve_periodic_naive(a0, dims, m, *k.arrays(), T)
    assert np.array_equal(got.view(np.uint64), np.asarray(want).view(np.uint64))
    one = fs.step_periodic(fs.FieldGrid(fs.GridShape(dims, m), a0), K(k)).data
    assert np.array_equal(one.view(np.uint64), np.asarray(orc.step_periodic(a0, dims, m, *k.arrays())).view(np.uint64))


def test_naive_T0_and_spec_errors():
    """T = 0 returns the input (oracle.cpp:103); require_fits (kernel.cpp:38-49)."""
    k = fs.StencilKernel(1).add_tap([1], 0.5).add_tap([-1], 0.5)
    a = fs.FieldGrid(fs.GridShape([16]), np.arange(16.0))
    assert np.array_equal(fs.evolve_periodic_naive(a, k, 0).data, a.data)
    with pytest.raises(fs.SpecError):
        fs.evolve_periodic_naive(fs.FieldGrid(fs.GridShape([1]), [1.0]), k, 3)
    with pytest.raises(fs.SpecError):
        fs.evolve_periodic_naive(fs.FieldGrid(fs.GridShape([4, 4]), np.zeros(16)), k, 3)


def _device_pair(cfg, T, seed):
    """FFT solve and naive stepping of the same seeded device-resident grid."""
    shape, kern = cfg.shape(), cfg.kernel()
    n = cfg.cells() * cfg.fields
    g = torch.Generator(device="cuda").manual_seed(seed)
    a0 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    fft_out = torch.empty_like(a0)
    naive_out = torch.empty_like(a0)
    fs.solve_periodic_device(shape, a0.data_ptr(), kern, T, fft_out.data_ptr(), stream=0)
    fs.device_check(stream=0)
    fs.evolve_periodic_naive_device(shape, a0.data_ptr(), kern, T, naive_out.data_ptr(), stream=0)
    torch.cuda.synchronize()
    diff = float(torch.linalg.vector_norm(fft_out - naive_out) / torch.linalg.vector_norm(naive_out))
    del a0, fft_out, naive_out
    torch.cuda.empty_cache()
    return diff


@pytest.mark.parametrize("name,T", [("cfg1", 1000), ("cfg2", 10000), ("cfg3", 10000), ("cfg4", 1000)])
def test_solver_vs_naive_full_size(name, T):
    """BASELINE configs at their FULL shapes: the FFT solver against T direct
    steps (cfg1, cfg2, cfg4 at their own T; cfg3 at T = 1e4 of its 1e5 to
    bound the test's runtime -- 1e4 steps of 8192^2)."""
    cfg = syn.configs()[name]
    diff = _device_pair(cfg, T, 123)
    print(f"{name} full size, T={T}: rel L2 (FFT solver vs direct stepping) = {diff:.3e}")
    assert diff <= 1e-10


def test_cfg5_full_size_vs_naive_short_horizon():
    """cfg5 (2^26 cells x 2 fields leapfrog) at full size against direct
    stepping over T = 2000 (the full T = 1e6 is out of reach for the naive
    loop).  The two fp64 computations differ by the conditioning of the
    neutrally stable leapfrog symbol; bound 1e-8."""
    cfg = syn.configs()["cfg5"]
    diff = _device_pair(cfg, 2000, 5)
    print(f"cfg5 full size, T=2000: rel L2 (FFT solver vs direct stepping) = {diff:.3e}")
    assert diff <= 1e-8


@pytest.mark.parametrize("dims,T", [([8192, 16384], 20), ([4, 8192, 4096], 10), ([1 << 26], 50)])
def test_solver_vs_naive_max_plan_sizes(dims, T):
    """The largest grids the fast plans take (plan 1: last axis 16384 = 2 kMaxLine,
    axis 0 8192; 3D; plan 2: 2^26 reals) against direct stepping."""
    cells = int(np.prod(dims))
    shape = fs.GridShape(dims)
    k = fs.StencilKernel(len(dims))
    k.add_tap([0] * len(dims), 0.5)
    for a in range(len(dims)):
        for sgn in (-1, 1):
            off = [0] * len(dims)
            off[a] = sgn
            k.add_tap(off, 0.25 / len(dims))
    g = torch.Generator(device="cuda").manual_seed(7)
    a0 = torch.rand(cells, dtype=torch.float64, device="cuda", generator=g)
    fft_out = torch.empty_like(a0)
    naive_out = torch.empty_like(a0)
    fs.solve_periodic_device(shape, a0.data_ptr(), k, T, fft_out.data_ptr(), stream=0)
    fs.device_check(stream=0)
    fs.evolve_periodic_naive_device(shape, a0.data_ptr(), k, T, naive_out.data_ptr(), stream=0)
    torch.cuda.synchronize()
    diff = float(torch.linalg.vector_norm(fft_out - naive_out) / torch.linalg.vector_norm(naive_out))
    del a0, fft_out, naive_out
    torch.cuda.empty_cache()
    assert diff <= 1e-12, (dims, diff)
