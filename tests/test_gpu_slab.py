"""GPU slab-decomposition stages (fsx_slab_*) against the oracle.

P ranks are emulated on the one available GPU (each rank's stages in turn,
the all-to-all as a device block shuffle: slab_solve_emulated), so the GPU
kernels run with the real multi-rank layouts and global column offsets.
The SlabSolver itself runs over an NCCL process group of world size 1.
The fused-exchange variant (p2p: row kernels store to / load from every
rank's exchange buffer) is emulated the same way with the P buffers as
separate allocations listed in the peer pointer array, and its solver path
(torch symmetric memory + device barriers) runs at world size 1.
"""
import os
import socket

import numpy as np
import pytest

import refutil as R

pytestmark = pytest.mark.gpu

fs = pytest.importorskip("paper_2105_06676_b200")
torch = pytest.importorskip("torch")


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
    ([256, 512], "random2", 50, (1, 2, 4)),
    ([4096, 256], "random2", 9, (2, 8)),
    ([1024, 1024], "box9", 100000, (8,)),
    ([32, 64, 128], "random3", 20, (1, 2, 4)),
    ([64, 1024, 64], "random3", 7, (4,)),
    ([8192, 128], "random2", 9, (2, 8)),     # 8192-point fused columns (parity halves)
]


@pytest.mark.parametrize("dims,kind,T,Ps", CASES)
def test_slab_emulated_vs_oracle(orc, dims, kind, T, Ps):
    from paper_2105_06676_b200.distributed import slab_solve_emulated

    kern = _box9(77) if kind == "box9" else R.random_kernel(R.Rng(len(dims) * 100 + T), len(dims), 1, 1, 0.95)
    n = int(np.prod(dims))
    a0 = orc.splitmix_fill(31, n, True)
    want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), T)
    da = torch.from_numpy(a0).cuda()
    for P in Ps:
        got = slab_solve_emulated(fs.GridShape(dims), da, _k(kern), T, P)
        torch.cuda.synchronize()
        fs.device_check()
        err = np.linalg.norm(got.cpu().numpy() - want) / np.linalg.norm(want)
        assert err <= 1e-10, (dims, P, err)


P2P_CASES = [
    ([256, 512], "random2", 50, (1, 2, 4)),     # M = 256: one-row-per-CTA row kernels
    ([4096, 2048], "random2", 9, (2, 8)),       # M = 1024: pipelined row kernels
    ([1024, 8192], "box9", 100000, (4, 8)),     # M = 4096
    ([64, 64], "random2", 5, (2,)),
]


@pytest.mark.parametrize("dims,kind,T,Ps", P2P_CASES)
def test_slab_p2p_emulated_vs_oracle(orc, dims, kind, T, Ps):
    """Exchange fused into the row passes: rank r's R2C rows store block d into
    buffer d, its C2R rows load from every buffer (1e-10 vs the oracle)."""
    from paper_2105_06676_b200.distributed import slab_solve_emulated_p2p

    kern = _box9(77) if kind == "box9" else R.random_kernel(R.Rng(len(dims) * 100 + T), len(dims), 1, 1, 0.95)
    n = int(np.prod(dims))
    a0 = orc.splitmix_fill(37, n, True)
    want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), T)
    da = torch.from_numpy(a0).cuda()
    for P in Ps:
        got = slab_solve_emulated_p2p(fs.GridShape(dims), da, _k(kern), T, P)
        fs.device_check()
        err = np.linalg.norm(got.cpu().numpy() - want) / np.linalg.norm(want)
        assert err <= 1e-10, (dims, P, err)


def test_slab_p2p_rejects_3d():
    from paper_2105_06676_b200.distributed import slab_solve_emulated_p2p

    with pytest.raises(fs.SpecError):
        slab_solve_emulated_p2p(fs.GridShape([8, 8, 16]), torch.zeros(1024, dtype=torch.float64, device="cuda"),
                                fs.StencilKernel(3).add_tap([0, 0, 1], 1.0), 3, 2)


def test_slab_solver_nccl_world1(orc):
    import torch.distributed as dist

    from paper_2105_06676_b200.distributed import SlabSolver

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        dims = [512, 256]
        kern = R.random_kernel(R.Rng(5), 2, 1, 1, 0.95)
        a0 = orc.splitmix_fill(9, 512 * 256, True)
        want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), 33)
        solver = SlabSolver(fs.GridShape(dims), _k(kern), 33)
        out = torch.empty(512 * 256, dtype=torch.float64, device="cuda")
        solver.solve(torch.from_numpy(a0).cuda(), out)
        torch.cuda.synchronize()
        err = np.linalg.norm(out.cpu().numpy() - want) / np.linalg.norm(want)
        assert err <= 1e-10
    finally:
        dist.destroy_process_group()


def test_slab_solver_p2p_world1(orc):
    """SlabSolver(exchange="p2p") over NCCL world size 1: symmetric-memory
    rendezvous, device barriers and the fused row kernels on the real path."""
    import torch.distributed as dist

    from paper_2105_06676_b200.distributed import SlabSolver

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, init_method=f"tcp://127.0.0.1:{port}")
    try:
        dims = [512, 1024]
        kern = R.random_kernel(R.Rng(6), 2, 1, 1, 0.95)
        a0 = orc.splitmix_fill(10, 512 * 1024, True)
        want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), 21)
        solver = SlabSolver(fs.GridShape(dims), _k(kern), 21, exchange="p2p")
        out = torch.empty(512 * 1024, dtype=torch.float64, device="cuda")
        for _ in range(2):  # twice: the leading barrier of the second solve
            solver.solve(torch.from_numpy(a0).cuda(), out)
        torch.cuda.synchronize()
        err = np.linalg.norm(out.cpu().numpy() - want) / np.linalg.norm(want)
        assert err <= 1e-10
    finally:
        dist.destroy_process_group()
