"""Re-entrancy of the drop-in: concurrent calls, shared plans across streams,
flag isolation and the SpectrumCache shape rule.

The reference's solvers are pure and safe to call concurrently
(proj/README.md:165-168); its SpectrumCache memoises the spectrum by dims only
(proj/src/periodic.cpp:67-74), so a later call whose grid has another field
count fails in hadamard with a SpecError (proj/src/spectrum.cpp:111-112).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if fs.device_count() < 1:
        pytest.fail("no CUDA device visible")


def jacobi2d():
    k = fs.StencilKernel(2)
    for off in ((0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)):
        k.add_tap(off, 0.2)
    return k


def test_cache_field_count_mismatch_is_spec_error(orc):
    dims = [64]
    k1 = fs.StencilKernel(1).add_tap([0], 0.5).add_tap([1], 0.25).add_tap([-1], 0.25)
    k2 = fs.StencilKernel(1, 2)
    k2.add_tap([0], np.array([[0.5, 0.1], [0.0, 0.5]]))
    k2.add_tap([1], np.array([[0.25, 0.0], [0.0, 0.25]]))
    cache = fs.SpectrumCache()
    a1 = orc.splitmix_fill(1, 64, False)
    out = fs.solve_periodic_cached(fs.FieldGrid(fs.GridShape(dims), a1), k1, 10, cache).data
    want = orc.solve_periodic(a1, dims, 1, *k1.arrays(), 10)
    assert np.abs(out - want).max() <= 1e-12
    a2 = orc.splitmix_fill(2, 128, False)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_cached(fs.FieldGrid(fs.GridShape(dims, 2), a2), k2, 10, cache)
    # and the other order: a 2-field spectrum first
    cache2 = fs.SpectrumCache()
    fs.solve_periodic_cached(fs.FieldGrid(fs.GridShape(dims, 2), a2), k2, 10, cache2)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_cached(fs.FieldGrid(fs.GridShape(dims), a1), k1, 10, cache2)


def test_two_streams_share_one_plan(orc):
    """Device solves of one shape enqueued back to back on two user streams
    (and the library stream) share the plan's workspaces; the plan's event
    orders them, so every result equals its own single solve."""
    dims = [1024, 1024]
    k = jacobi2d()
    sh = fs.GridShape(dims)
    ins = [torch.from_numpy(orc.splitmix_fill(s, 1024 * 1024, False)).cuda() for s in (11, 12, 13, 14)]
    outs = [torch.empty_like(x) for x in ins]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for i, (x, y) in enumerate(zip(ins, outs)):
        fs.solve_periodic_device(sh, x.data_ptr(), k, 500, y.data_ptr(), stream=streams[i % 2].cuda_stream)
    torch.cuda.synchronize()
    fs.device_check(stream=0)
    for x, y in zip(ins, outs):
        want = fs.solve_periodic(fs.FieldGrid(sh, x.cpu().numpy()), k, 500).data
        assert np.array_equal(y.cpu().numpy(), want)


def test_concurrent_host_calls_from_threads(orc):
    """Several host threads calling the synchronous API at once (one device):
    each result equals the oracle's."""
    dims = [256, 256]
    k = jacobi2d()
    off, blk = k.arrays()
    seeds = list(range(21, 29))
    res = {}
    errs = []

    def work(seed):
        try:
            a = orc.splitmix_fill(seed, 256 * 256, False)
            res[seed] = (a, fs.solve_periodic(fs.FieldGrid(fs.GridShape(dims), a), k, 300).data)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(s,)) for s in seeds]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for seed in seeds:
        a, got = res[seed]
        want = orc.solve_periodic(a, dims, 1, off, blk, 300)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


def test_deferred_flags_do_not_leak_into_host_solves():
    """A non-finite device-mode solve left unchecked must not make the next
    host solve raise (separate flag slots); fsx_device_check still reports it."""
    dims = [64, 64]
    k = jacobi2d()
    sh = fs.GridShape(dims)
    bad = torch.full((64 * 64,), float("nan"), dtype=torch.float64, device="cuda")
    out = torch.empty_like(bad)
    fs.solve_periodic_device(sh, bad.data_ptr(), k, 5, out.data_ptr(), stream=0)
    torch.cuda.synchronize()
    good = np.linspace(0.0, 1.0, 64 * 64)
    res = fs.solve_periodic(fs.FieldGrid(sh, good), k, 5).data
    assert np.isfinite(res).all()
    with pytest.raises(fs.NumericError):
        fs.device_check(stream=0)
    fs.device_check(stream=0)  # reset by the previous check


def test_device_check_applies_residue_test_after_general_plan():
    """A device-mode solve on the general (complex) plan: fsx_device_check
    applies the reference's imaginary-residue test (periodic.cpp:60-63)."""
    # a one-sided (non-symmetric) growth kernel on a non-pow2 grid: the
    # general complex pipeline, finite but with a blown-up residue
    n = 300
    k = fs.StencilKernel(1).add_tap([1], 3.0).add_tap([0], 1.0)
    a = torch.from_numpy(np.random.default_rng(0).random(n)).cuda()
    out = torch.empty_like(a)
    assert fs.plan_describe(fs.GridShape([n]), k)["path"] == 3
    host_err = None
    try:
        fs.solve_periodic(fs.FieldGrid(fs.GridShape([n]), a.cpu().numpy()), k, 600)
    except fs.NumericError as e:
        host_err = e
    fs.solve_periodic_device(fs.GridShape([n]), a.data_ptr(), k, 600, out.data_ptr(), stream=0)
    if host_err is None:
        fs.device_check(stream=0)
    else:
        with pytest.raises(fs.NumericError):
            fs.device_check(stream=0)
