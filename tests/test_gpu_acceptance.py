"""Reference acceptance criteria 7 and 8, the bench-mode stage-table contract
and the device grid loader, on the GPU path.

  * criterion 7, log-T scaling (proj/tests/acceptance.cpp:261-294): heat1d on
    N = 2^20 random cells: t(T = 1e9) < 2 t(T = 1e3), both < 10 s, and the
    naive solver at T = 1e3 slower than the FFT solver at T = 1e9;
  * criterion 8, accuracy parity against the double-double modal truth
    (acceptance.cpp:296-320, proj/src/modal.cpp:99-145): heat1d, l = 1000,
    T = 1e4 (and the FFTSTENCIL_SLOW rerun's 1e6): |err_fft - err_naive| <=
    1e-9 (1 + err_naive);
  * bench mode (proj/tests/test_io_cli.cpp:207-236): heat1d, N = 2^20,
    T = 1e5, random init seed 3: every stage listed and
    0.9 total <= sum(stages) <= total;
  * fsx_load_grid_device: a raw grid read straight into device memory equals
    the host read, and solving from it equals the host solve.
"""
import time

import numpy as np
import pytest

import refutil as R

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if fs.device_count() < 1:
        pytest.fail("no CUDA device visible")


def heat1d():
    """builtin_stencil("heat1d") (proj/src/stencils.cpp:9-24): alpha = 0.125"""
    return fs.StencilKernel(1).add_tap([-1], 0.125).add_tap([0], 0.75).add_tap([1], 0.125)


def _timed(a0, k, T):
    best = 1e30
    for _ in range(2):
        t0 = time.perf_counter()
        out = fs.solve_periodic(a0, k, T)
        best = min(best, time.perf_counter() - t0)
        assert np.abs(out.data).max() <= 1e10
    return best


def test_criterion7_log_T_scaling():
    n = 1 << 20
    a0 = fs.FieldGrid(fs.GridShape([n]), R.random_grid(R.Rng(7007), n))
    k = heat1d()
    fs.solve_periodic(a0, k, 10)  # plan set-up (the reference's first solve builds its FFT plans too)
    t_small = _timed(a0, k, 1000)
    t_large = _timed(a0, k, 1000000000)
    t0 = time.perf_counter()
    fs.evolve_periodic_naive(a0, k, 1000)
    t_naive = time.perf_counter() - t0
    print(f"criterion 7: fft T=1e3 {t_small * 1e3:.3f} ms, fft T=1e9 {t_large * 1e3:.3f} ms "
          f"(ratio {t_large / t_small:.2f}), naive T=1e3 {t_naive * 1e3:.3f} ms")
    assert t_large < 2.0 * t_small and t_small < 10.0 and t_large < 10.0 and t_naive > t_large


@pytest.mark.parametrize("T", [10000, 1000000])
def test_criterion8_accuracy_parity_vs_modal_truth(orc, T):
    k = heat1d()
    off, blk = k.arrays()
    init, ref = orc.modal_problem_periodic([1000], off, blk, T)
    a0 = fs.FieldGrid(fs.GridShape([1000]), init)
    fast = fs.solve_periodic(a0, k, T).data
    slow = fs.evolve_periodic_naive(a0, k, T).data
    err_fft = np.abs(fast - ref).max()
    err_naive = np.abs(slow - ref).max()
    gap = abs(err_fft - err_naive)
    err_orc = np.abs(orc.solve_periodic(init, [1000], 1, off, blk, T) - ref).max()
    print(f"criterion 8, T={T}: err_fft {err_fft:.3e}, err_naive {err_naive:.3e}, gap {gap:.3e} "
          f"(reference-path oracle err {err_orc:.3e})")
    assert gap <= 1e-9 * (1 + err_naive)


def test_bench_stage_table_covers_the_total():
    n = 1 << 20
    from paper_2105_06676_b200.synthetic import uniform_sym

    a0 = fs.FieldGrid(fs.GridShape([n]), uniform_sym(3, n))  # init: {random: {seed: 3}}
    table, st, total, _ = fs.run_bench(a0, heat1d(), 100000)
    print(table)
    stage_sum, tot = 0.0, -1.0
    for name in ("forward_fft", "squaring", "hadamard", "inverse_fft", "boundary_recursion", "total"):
        pos = table.find(name)
        assert pos >= 0, name
        v = float(table[pos + len(name):].split()[0])
        if name == "total":
            tot = v
        else:
            stage_sum += v
    assert tot > 0
    assert stage_sum <= tot
    assert stage_sum >= 0.9 * tot


def test_load_grid_device_round_trip(tmp_path):
    torch = pytest.importorskip("torch")
    shape = fs.GridShape([512, 384])
    from paper_2105_06676_b200.synthetic import uniform01

    g = fs.FieldGrid(shape, uniform01(11, 512 * 384))
    p = str(tmp_path / "grid.raw")
    fs.write_grid(g, p, "raw")
    d = torch.empty(512 * 384, dtype=torch.float64, device="cuda")
    got_shape = fs.load_grid_device(p, d.data_ptr())
    assert got_shape.dims() == [512, 384]
    assert np.array_equal(d.cpu().numpy(), g.data)
    k = fs.StencilKernel(2).add_tap([0, 0], 0.6).add_tap([1, 0], 0.2).add_tap([0, -1], 0.2)
    out = torch.empty_like(d)
    fs.solve_periodic_device(shape, d.data_ptr(), k, 50, out.data_ptr(), stream=0)
    fs.device_check(stream=0)
    assert np.array_equal(out.cpu().numpy(), fs.solve_periodic(g, k, 50).data)
    with pytest.raises(fs.IoError):
        fs.load_grid_device(p, d.data_ptr(), shape=fs.GridShape([384, 512]))
