"""fsx_solve_periodic_slabs: one recursion level's
face-slab solves in one call, against the oracle.

The slab shapes are those rb_run hands to solve_periodic_cached
(proj/src/aperiodic.cpp:224-228,240-244; proj/src/band.cpp slab_shape): for
each axis a, two slabs with dims[a] replaced by the band width 4 sigma T1.
Equal shapes are stacked into one batched plan, so each result must match
both the oracle (1e-10) and the sequential solve_periodic_cached call on the
same slab (bit for bit: the same kernels with the stack as an outer block).
"""
import time

import numpy as np
import pytest

import refutil as R

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")


def _k(kern):
    k = fs.StencilKernel(kern.rank, kern.fields)
    offs, blks = kern.arrays()
    for o, b in zip(offs, blks):
        k.add_tap(tuple(int(x) for x in o), b if kern.fields > 1 else float(b[0, 0]))
    return k


def _level(dims, width, fields, seed, orc):
    """The 2d face slabs of one rb_run level (both sides of every axis)."""
    grids = []
    for a in range(len(dims)):
        sd = list(dims)
        sd[a] = width
        for side in range(2):
            n = int(np.prod(sd)) * fields
            data = orc.splitmix_fill(seed + 10 * a + side, n, True)
            grids.append(fs.FieldGrid(fs.GridShape(sd, fields), data))
    return grids


LEVELS = [
    ([96, 128], 48, 1, 12),        # non-pow2 axis: general plan (direct DFT / Bluestein passes)
    ([256, 512], 64, 1, 30),       # pow2 slabs: stacked fused R2C plan
    ([40, 24, 48], 8, 1, 5),       # 3D, non-pow2
    ([64, 32, 128], 16, 1, 7),     # 3D pow2: stacked plan 1 with y passes
    ([72, 96], 24, 2, 9),          # 2-field cells: general plan, m = 2 blocks
    ([600, 40], 20, 1, 11),        # Bluestein axis (600 > 256)
]


@pytest.mark.parametrize("dims,width,fields,T", LEVELS)
def test_slabs_vs_oracle_and_sequential(orc, dims, width, fields, T):
    kern = R.random_kernel(R.Rng(len(dims) * 7 + width), len(dims), 1, fields, 0.95)
    k = _k(kern)
    grids = _level(dims, width, fields, 100 + T, orc)
    st = fs.StageTimings()
    got = fs.solve_periodic_slabs(grids, k, T, cache=fs.SpectrumCache(), st=st)
    assert st.boundary_recursion > 0
    seq_cache = fs.SpectrumCache()
    worst = 0.0
    for g, o in zip(grids, got):
        want = orc.solve_periodic(g.data, g.shape.dims(), fields, *kern.arrays(), T, vector=fields > 1)
        err = np.linalg.norm(o - want) / np.linalg.norm(want)
        worst = max(worst, err)
        assert err <= 1e-10, (g.shape.dims(), err)
        seq = fs.solve_periodic_cached(g, k, T, seq_cache).data
        assert np.array_equal(o, seq), g.shape.dims()
    print(f"{dims} width {width} m={fields}: {len(grids)} slabs, worst rel L2 vs oracle {worst:.2e}")


def test_slabs_cache_semantics(orc):
    """The first kernel seen for a dims vector defines that dims' spectrum
    (proj/src/periodic.cpp:67-74): a cache seeded with another kernel wins."""
    dims = [64, 80]
    kern_a = R.random_kernel(R.Rng(1), 2, 1, 1, 0.9)
    kern_b = R.random_kernel(R.Rng(2), 2, 1, 1, 0.9)
    grids = _level(dims, 16, 1, 7, orc)
    cache = fs.SpectrumCache()
    # seed the cache for the [16, 80] slabs with kernel b
    fs.solve_periodic_cached(grids[0], _k(kern_b), 3, cache)
    got = fs.solve_periodic_slabs(grids, _k(kern_a), 5, cache=cache)
    for g, o in zip(grids, got):
        used = kern_b if g.shape.dims() == [16, 80] else kern_a
        want = orc.solve_periodic(g.data, g.shape.dims(), 1, *used.arrays(), 5)
        assert np.linalg.norm(o - want) / np.linalg.norm(want) <= 1e-10
    # a field-count mismatch against the cached spectrum is a SpecError (hadamard)
    two = fs.FieldGrid(fs.GridShape([16, 80], 2), np.zeros(16 * 80 * 2))
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_slabs([two], _k(R.random_kernel(R.Rng(3), 2, 1, 2, 0.9)), 2, cache=cache)


def test_slabs_errors_and_t0(orc):
    kern = R.random_kernel(R.Rng(4), 2, 1, 1, 0.9)
    grids = _level([48, 64], 12, 1, 3, orc)
    # T = 0: bit-exact copies
    out = fs.solve_periodic_slabs(grids, _k(kern), 0)
    for g, o in zip(grids, out):
        assert np.array_equal(g.data, o)
    # a non-finite slab: NumericError naming it (argument order), for both plan kinds
    for dims, w in (([48, 64], 12), ([64, 128], 16)):
        gs = _level(dims, w, 1, 3, orc)
        gs[2].data[5] = np.nan
        with pytest.raises(fs.NumericError, match=r"slab 2\)"):
            fs.solve_periodic_slabs(gs, _k(kern), 4)
    # empty level
    assert fs.solve_periodic_slabs([], _k(kern), 4) == []
    # kernel reach beyond a slab's dims: SpecError (require_fits)
    far = fs.StencilKernel(2)
    far.add_tap((0, 20), 1.0)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_slabs(_level([48, 64], 12, 1, 3, orc), far, 2)


def test_slabs_faster_than_sequential(orc):
    """Time per level: one batched call against the 2d sequential cached solves."""
    rows = []
    for dims, w, T in (([1024, 1024], 96, 48), ([2048, 2048], 256, 128), ([256, 256, 256], 32, 16)):
        kern = R.random_kernel(R.Rng(9), len(dims), 1, 1, 0.95)
        k = _k(kern)
        grids = _level(dims, w, 1, 5, orc)
        outs = [np.empty_like(g.data) for g in grids]
        cache = fs.SpectrumCache()
        fs.solve_periodic_slabs(grids, k, T, cache=cache, outs=outs)
        for g in grids:
            fs.solve_periodic_cached(g, k, T, cache)
        tb, ts = [], []
        for _ in range(5):
            t0 = time.perf_counter()
            fs.solve_periodic_slabs(grids, k, T, cache=cache, outs=outs)
            tb.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            for g in grids:
                fs.solve_periodic_cached(g, k, T, cache)
            ts.append(time.perf_counter() - t0)
        b, s = min(tb), min(ts)
        rows.append((dims, w, b, s))
        print(f"level of {len(grids)} slabs of {dims} width {w}: batched {b * 1e3:.2f} ms, sequential {s * 1e3:.2f} ms "
              f"({s / b:.2f}x)")
    # the batched call must not be slower than the sequential calls it replaces
    # (pageable host copies dominate the 3D level; 20 % slack for box noise)
    for dims, w, b, s in rows:
        assert b <= s * 1.2, (dims, w, b, s)
