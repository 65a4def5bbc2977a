"""Single-process multi-GPU solve through the C ABI (fsx_options.num_gpus /
devices / exchange, fsx_set_devices) against the oracle.

Only one GPU is available, so P ranks are emulated by repeating device 0 in
the device list: every rank gets its own streams, slab buffers and exchange
buffer on that device, the p2p exchange writes / reads the other ranks'
buffers exactly as it would over NVLink, and the cross-rank ordering is the
same CUDA-event barriers (no kernel waits on another).  The NCCL exchange
needs one rank per device, so it runs at P = 1 (NCCL's self send/recv).
"""
import numpy as np
import pytest

import refutil as R

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")


def _k(kern):
    k = fs.StencilKernel(kern.rank)
    for off, blk in sorted(kern.taps.items()):
        k.add_tap(off, float(blk[0, 0]))
    return k


def _box9(seed):
    rng = R.Rng(seed)
    u = [rng.uniform() for _ in range(9)]
    offs = [(i, j) for i in (-1, 0, 1) for j in (-1, 0, 1)]
    return R.kern_from({o: w / sum(u) for o, w in zip(offs, u)}, 2)


CASES = [
    ([256, 512], "random2", 50, (2, 4, 8)),
    ([64, 64], "random2", 5, (2, 8)),
    ([1024, 8192], "box9", 100000, (4, 8)),      # M = 4096 rows; cfg3's stencil
    ([8192, 256], "random2", 9, (2,)),           # 8192-point fused columns
    ([32, 64, 128], "random3", 20, (2, 4)),      # 3D: chunked copy-engine exchange
    ([64, 128, 64], "random3", 7, (8,)),
    ([16, 8, 32], "random3", 3, (2, 8)),         # 3D, short y lines (non-TMA y pass)
]


@pytest.mark.parametrize("dims,kind,T,Ps", CASES)
def test_multi_p2p_emulated_vs_oracle(orc, dims, kind, T, Ps):
    kern = _box9(1003) if kind == "box9" else R.random_kernel(R.Rng(len(dims) * 100 + T), len(dims), 1, 1, 0.95)
    n = int(np.prod(dims))
    a0 = orc.splitmix_fill(3, n, True)
    want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), T)
    shape = fs.GridShape(dims)
    single = fs.solve_periodic(fs.FieldGrid(shape, a0.copy()), _k(kern), T).data
    for P in Ps:
        devs = [0] * P
        info = fs.plan_describe(shape, _k(kern), devices=devs)
        assert info["ranks"] == P and info["exchange"] == 1, info
        got = fs.solve_periodic(fs.FieldGrid(shape, a0.copy()), _k(kern), T, devices=devs, exchange=1).data
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        gap = np.linalg.norm(got - single) / np.linalg.norm(single)
        print(f"{dims} P={P}: rel L2 vs oracle {err:.3e}, vs single GPU {gap:.3e}")
        assert err <= 1e-10, (dims, P, err)
        # the context is cached: a second call gives the same bits
        again = fs.solve_periodic(fs.FieldGrid(shape, a0.copy()), _k(kern), T, devices=devs, exchange=1).data
        assert np.array_equal(got, again)


def test_multi_nccl_one_rank(orc):
    """The NCCL exchange (grouped ncclSend/ncclRecv, libnccl loaded on use) at P = 1."""
    for dims in ([256, 512], [32, 64, 128]):
        kern = R.random_kernel(R.Rng(5 + len(dims)), len(dims), 1, 1, 0.95)
        a0 = orc.splitmix_fill(11, int(np.prod(dims)), True)
        want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), 17)
        shape = fs.GridShape(dims)
        info = fs.plan_describe(shape, _k(kern), devices=[0], exchange=2)
        assert info["ranks"] == 1 and info["exchange"] == 2
        got = fs.solve_periodic(fs.FieldGrid(shape, a0), _k(kern), 17, devices=[0], exchange=2).data
        err = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert err <= 1e-10, (dims, err)


def test_multi_nccl_rejects_repeated_devices():
    kern = R.random_kernel(R.Rng(9), 2, 1, 1, 0.95)
    a0 = np.linspace(0, 1, 64 * 64)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic(fs.FieldGrid(fs.GridShape([64, 64]), a0), _k(kern), 3, devices=[0, 0], exchange=2)


def test_multi_process_default_and_fallback(orc):
    """fsx_set_devices routes option-less calls; ineligible problems (1D,
    vector cells, axis 0 not divisible) run on one GPU with the same result."""
    kern2 = R.random_kernel(R.Rng(21), 2, 1, 1, 0.95)
    a0 = orc.splitmix_fill(4, 128 * 256, True)
    want = orc.solve_periodic(a0, [128, 256], 1, *kern2.arrays(), 30)
    fs.set_devices([0, 0, 0, 0])
    try:
        assert fs.get_devices() == [0, 0, 0, 0]
        assert fs.plan_describe(fs.GridShape([128, 256]), _k(kern2))["ranks"] == 4
        st = fs.StageTimings()
        got = fs.solve_periodic(fs.FieldGrid(fs.GridShape([128, 256]), a0), _k(kern2), 30, st).data
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10
        assert st.forward_fft > 0 and st.squaring > 0 and st.inverse_fft > 0
        # 1D and a 2D grid whose axis 0 (12) is not a multiple of 4: single GPU
        k1 = R.random_kernel(R.Rng(22), 1, 1, 1, 0.95)
        b0 = orc.splitmix_fill(5, 4096, True)
        assert fs.plan_describe(fs.GridShape([4096]), _k(k1))["ranks"] == 1
        g1 = fs.solve_periodic(fs.FieldGrid(fs.GridShape([4096]), b0), _k(k1), 9).data
        w1 = orc.solve_periodic(b0, [4096], 1, *k1.arrays(), 9)
        assert np.linalg.norm(g1 - w1) / np.linalg.norm(w1) <= 1e-10
        c0 = orc.splitmix_fill(6, 12 * 64, True)
        assert fs.plan_describe(fs.GridShape([12, 64]), _k(kern2))["ranks"] == 1
        g2 = fs.solve_periodic(fs.FieldGrid(fs.GridShape([12, 64]), c0), _k(kern2), 9).data
        w2 = orc.solve_periodic(c0, [12, 64], 1, *kern2.arrays(), 9)
        assert np.linalg.norm(g2 - w2) / np.linalg.norm(w2) <= 1e-10
    finally:
        fs.set_devices([])
    assert fs.get_devices() == []
    with pytest.raises(fs.SpecError):
        fs.set_devices([0, 99])


def test_multi_numeric_error_and_aliasing(orc):
    """A non-finite slab raises NumericError naming the slab; out may alias a0; T = 0 copies."""
    kern = R.random_kernel(R.Rng(31), 2, 1, 1, 0.95)
    shape = fs.GridShape([128, 128])
    a0 = orc.splitmix_fill(8, 128 * 128, True)
    bad = a0.copy()
    bad[3 * 128 * 128 // 4 + 5] = np.nan
    with pytest.raises(fs.NumericError, match="slab"):
        fs.solve_periodic(fs.FieldGrid(shape, bad), _k(kern), 4, devices=[0, 0, 0, 0])
    # the flags were reset: the next solve is clean
    want = orc.solve_periodic(a0, [128, 128], 1, *kern.arrays(), 4)
    buf = a0.copy()
    got = fs.solve_periodic(fs.FieldGrid(shape, buf), _k(kern), 4, devices=[0, 0], out=buf).data
    assert got is buf or np.shares_memory(got, buf)
    assert np.linalg.norm(buf - want) / np.linalg.norm(want) <= 1e-10
    same = fs.solve_periodic(fs.FieldGrid(shape, a0.copy()), _k(kern), 0, devices=[0, 0]).data
    assert np.array_equal(same, a0)


PENCIL_CASES = [
    ([32, 64, 128], 4, 0),      # 2 x 2 (most square)
    ([64, 32, 64], 8, 2),       # 2 x 4
    ([64, 32, 64], 8, 4),       # 4 x 2
    ([32, 16, 32], 2, 1),       # 1 x 2: pencils along axis 1 only
    ([8, 16, 32], 16, 0),       # slabs impossible (8 planes < 16 ranks): auto picks 4 x 4 pencils
    ([1024, 64, 32], 4, 2),     # 1024-point fused columns (TMA), 2 x 2
]


@pytest.mark.parametrize("dims,P,pr", PENCIL_CASES)
def test_multi_pencils_emulated_vs_oracle(orc, dims, P, pr):
    """Pr x Pc pencil grid (fsx_options.decomp = FSX_DECOMP_PENCIL): four
    copy-engine transposes per solve; against the oracle and bit for bit
    against the single-GPU solve (the same kernels per line)."""
    kern = R.random_kernel(R.Rng(sum(dims) + P), 3, 1, 1, 0.95)
    a0 = orc.splitmix_fill(13, int(np.prod(dims)), True)
    T = 11
    want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), T)
    shape = fs.GridShape(dims)
    single = fs.solve_periodic(fs.FieldGrid(shape, a0.copy()), _k(kern), T).data
    devs = [0] * P
    decomp = 2 if dims[0] >= P else 0
    info = fs.plan_describe(shape, _k(kern), devices=devs, decomp=decomp, pencil_rows=pr)
    assert info["ranks"] == P and info["decomp"] == 2, info
    if pr:
        assert info["pencil_rows"] == pr
    got = fs.solve_periodic(fs.FieldGrid(shape, a0.copy()), _k(kern), T, devices=devs, decomp=decomp,
                            pencil_rows=pr).data
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    print(f"{dims} pencils {info['pencil_rows']}x{P // info['pencil_rows']}: rel L2 vs oracle {err:.3e}")
    assert err <= 1e-10, (dims, P, err)
    assert np.array_equal(got, single)


def test_multi_pencil_numeric_error(orc):
    dims = [32, 16, 32]
    kern = R.random_kernel(R.Rng(44), 3, 1, 1, 0.95)
    bad = orc.splitmix_fill(2, int(np.prod(dims)), True)
    bad[-3] = np.inf
    with pytest.raises(fs.NumericError, match="pencil"):
        fs.solve_periodic(fs.FieldGrid(fs.GridShape(dims), bad), _k(kern), 3, devices=[0] * 4, decomp=2)
    # 2D grids have no pencils: decomp = pencil there means one GPU
    info = fs.plan_describe(fs.GridShape([64, 64]), _k(R.random_kernel(R.Rng(45), 2, 1, 1, 0.9)), devices=[0, 0],
                            decomp=2)
    assert info["ranks"] == 1
