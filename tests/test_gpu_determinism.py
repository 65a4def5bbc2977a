"""Run-to-run bitwise determinism of the kernels that synchronise across
threads, CTAs or streams without a CTA-wide barrier at every step: the
8192-point columns on a CTA pair (DSMEM st.async exchanges, remote mbarrier
arrives), the two-group rows (named barriers, stage row tags), the 1D row
pairs on a CTA pair, the emulated multi-GPU slab and pencil exchanges (event
barriers between streams) and the stacked slab batch.  A data race in any of
them shows up as a result that differs between repetitions (compute-sanitizer
is not available on this pool)."""
import numpy as np
import pytest

import refutil as R

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")

REPS = 12


def _k(kern):
    k = fs.StencilKernel(kern.rank, kern.fields)
    for off, blk in sorted(kern.taps.items()):
        k.add_tap(off, blk if kern.fields > 1 else float(blk[0, 0]))
    return k


@pytest.mark.parametrize("dims,m,T,opts", [
    ([8192, 256], 1, 100000, {}),                       # k_fused8192c
    ([64, 8192], 1, 1000, {}),                          # k_r2c_grp / k_c2r_grp
    ([1 << 24], 1, 1000, {}),                           # k_rowpair_c (N2 = 4096)
    ([1 << 23], 2, 1000, {}),                           # k_rowpair_c, two-for-one
    ([512, 1024], 1, 50, {"devices": [0] * 4}),         # slabs, p2p fused into the rows
    ([64, 32, 128], 1, 20, {"devices": [0] * 4}),       # 3D slabs, chunked copy-engine exchange
    ([32, 32, 64], 1, 20, {"devices": [0] * 4, "decomp": 2}),  # 2 x 2 pencils
])
def test_repeated_solves_are_bitwise_identical(orc, dims, m, T, opts):
    kern = R.random_kernel(R.Rng(sum(dims) + m), len(dims), 1, m, 0.95)
    a0 = orc.splitmix_fill(17, int(np.prod(dims)) * m, True)
    grid = fs.FieldGrid(fs.GridShape(dims, m), a0)
    first = fs.solve_periodic(grid, _k(kern), T, **opts).data.copy()
    for _ in range(REPS):
        again = fs.solve_periodic(grid, _k(kern), T, **opts).data
        assert np.array_equal(first, again), dims


def test_repeated_slab_levels_are_bitwise_identical(orc):
    kern = R.random_kernel(R.Rng(77), 2, 1, 1, 0.95)
    grids = [fs.FieldGrid(fs.GridShape(d), orc.splitmix_fill(i, int(np.prod(d)), True))
             for i, d in enumerate(([96, 1024], [96, 1024], [1024, 96], [1024, 96]))]
    first = [o.copy() for o in fs.solve_periodic_slabs(grids, _k(kern), 48)]
    for _ in range(REPS // 2):
        again = fs.solve_periodic_slabs(grids, _k(kern), 48)
        for f, a in zip(first, again):
            assert np.array_equal(f, a)
