"""Multi-rank slab decomposition on CPU ranks (gloo, world_size 2).

The product's SlabSolver (paper_2105_06676_b200/distributed.py) drives the
decomposition: slab sizes and offsets from the C ABI (fsx_slab_describe),
the exchange buffers, and the two equal-split all-to-alls over
torch.distributed.  The per-rank numerical stages are replaced by a numpy
reference of the same stage contract (test infrastructure), so the layouts,
global column offsets and exchange pattern are checked end to end against
the CPU oracle without a GPU.  The fused-exchange (p2p) sequence runs the
same way with every rank's exchange buffer a memory-mapped file opened by all
ranks (the CPU stand-in for NVLink symmetric memory) and gloo barriers.  The
GPU stages are checked with the same layouts in tests/test_gpu_slab.py.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import refutil as R


class NumpyStages:
    """Reference of fsx_slab_forward / _spectral / _inverse for one rank."""

    def __init__(self, dims, P, r, info, kern: R.Kern):
        self.dims, self.P, self.r, self.info, self.k = list(dims), P, r, info, kern
        self.L = dims[-1]
        self.M = self.L // 2
        self.Pp = self.M + 8
        self.n0l = dims[0] // P
        self.CB = info["col_block"]

    @staticmethod
    def _c(t):  # float64 tensor -> complex numpy view
        return t.numpy().view(np.complex128)

    def _symbol(self, ks):
        """lam(k) = sum c exp(+2 pi i sum_a k_a o_a / n_a) on broadcast index arrays ks."""
        lam = 0j
        for off, blk in self.k.taps.items():
            ph = sum(ks[a] * off[a] / self.dims[a] for a in range(len(self.dims)))
            lam = lam + blk[0, 0] * np.exp(2j * np.pi * ph)
        return lam

    def forward(self, local_in, send):
        x = local_in.numpy().reshape([self.n0l] + self.dims[1:])
        X = np.fft.rfft(x, axis=-1)
        out = self._c(send)
        if len(self.dims) == 2:
            buf = out.reshape(self.P, self.n0l, self.CB)
            buf[:] = 0
            for d in range(self.P):
                lo, hi = d * self.CB, min((d + 1) * self.CB, self.M + 1)
                if lo < hi:
                    buf[d, :, :hi - lo] = X[:, lo:hi]
        else:
            X = np.fft.fft(X, axis=1)
            n1b = self.dims[1] // self.P
            Hp = np.zeros((self.n0l, self.dims[1], self.Pp), np.complex128)
            Hp[..., :self.M + 1] = X
            buf = out.reshape(self.P, self.n0l, n1b, self.Pp)
            for d in range(self.P):
                buf[d] = Hp[:, d * n1b:(d + 1) * n1b, :]

    def spectral(self, recv, kernel, T):
        n0 = self.dims[0]
        z = self._c(recv)
        N = int(np.prod(self.dims))
        k0 = np.arange(n0)
        if len(self.dims) == 2:
            a = z.reshape(n0, self.CB)
            kx = self.r * self.CB + np.arange(self.CB)
            lam = self._symbol([k0[:, None], kx[None, :]])
            a[:] = np.fft.ifft(np.fft.fft(a, axis=0) * lam ** T / N, axis=0) * n0
        else:
            n1b = self.dims[1] // self.P
            a = z.reshape(n0, n1b, self.Pp)
            ky = self.r * n1b + np.arange(n1b)
            kx = np.arange(self.Pp)
            lam = self._symbol([k0[:, None, None], ky[None, :, None], kx[None, None, :]])
            a[:] = np.fft.ifft(np.fft.fft(a, axis=0) * lam ** T / N, axis=0) * n0

    # p2p contract (fsx_slab_forward_p2p / _inverse_p2p): `peers` lists every
    # rank's exchange buffer; block d of this rank's rows goes to / comes from
    # rows [r n0l, (r+1) n0l) of buffer d
    def forward_p2p(self, local_in, peers):
        x = local_in.numpy().reshape(self.n0l, self.L)
        X = np.fft.rfft(x, axis=-1)
        for d in range(self.P):
            lo, hi = d * self.CB, min((d + 1) * self.CB, self.M + 1)
            dst = peers[d].view(np.complex128).reshape(self.dims[0], self.CB)
            rows = dst[self.r * self.n0l:(self.r + 1) * self.n0l]
            rows[:] = 0
            if lo < hi:
                rows[:, :hi - lo] = X[:, lo:hi]

    def inverse_p2p(self, peers, local_out):
        parts = [peers[d].view(np.complex128).reshape(self.dims[0], self.CB)[self.r * self.n0l:(self.r + 1) * self.n0l]
                 for d in range(self.P)]
        X = np.concatenate(parts, axis=1)[:, :self.M + 1]
        y = np.fft.irfft(X, n=self.L, axis=-1) * self.L
        local_out.numpy()[:] = y.reshape(-1)

    def inverse(self, send, local_out):
        z = self._c(send)
        if len(self.dims) == 2:
            buf = z.reshape(self.P, self.n0l, self.CB)
            X = np.concatenate([buf[d] for d in range(self.P)], axis=1)[:, :self.M + 1]
        else:
            n1b = self.dims[1] // self.P
            buf = z.reshape(self.P, self.n0l, n1b, self.Pp)
            X = np.concatenate([buf[d] for d in range(self.P)], axis=1)[..., :self.M + 1]
            X = np.fft.ifft(X, axis=1) * self.dims[1]
        y = np.fft.irfft(X, n=self.L, axis=-1) * self.L
        local_out.numpy()[:] = y.reshape(-1)


class FilePeerMemory:
    """CPU stand-in for the symmetric-memory exchange buffer: every rank's
    buffer is a memory-mapped file all ranks open, the barrier is gloo's."""

    def __init__(self, nelem, rank, world, root):
        path = lambda r: os.path.join(root, f"xbuf{r}.bin")  # noqa: E731
        np.lib.format.open_memmap(path(rank), mode="w+", dtype=np.float64, shape=(nelem,)).flush()
        dist.barrier()
        self.peers = [np.lib.format.open_memmap(path(r), mode="r+") for r in range(world)]
        self.local = torch.from_numpy(self.peers[rank])

    def barrier(self, channel):
        for p in self.peers:
            p.flush()
        dist.barrier()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, seed, T, outdir, exchange="nccl"):
    from paper_2105_06676_b200 import GridShape, StencilKernel
    from paper_2105_06676_b200.distributed import SlabSolver

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    try:
        rng = R.Rng(seed)
        kern = R.random_kernel(rng, len(dims), 1, 1, 0.95)
        k = StencilKernel(len(dims))
        for off, blk in sorted(kern.taps.items()):
            k.add_tap(off, float(blk[0, 0]))
        a0 = np.random.default_rng(seed).uniform(-1, 1, int(np.prod(dims)))
        n0l = dims[0] // world
        slab = a0.reshape(dims[0], -1)[rank * n0l:(rank + 1) * n0l].reshape(-1).copy()
        shape = GridShape(dims)
        from paper_2105_06676_b200.distributed import slab_describe

        info = slab_describe(shape, world, rank)
        pm = FilePeerMemory(info["xbuf_bytes"] // 8, rank, world, outdir) if exchange == "p2p" else None
        solver = SlabSolver(shape, k, T, stages=NumpyStages(dims, world, rank, info, kern), exchange=exchange,
                            peer_memory=pm)
        out = torch.empty(slab.size, dtype=torch.float64)
        solver.solve(torch.from_numpy(slab), out)
        if exchange == "p2p":
            solver.solve(torch.from_numpy(slab), out)  # second solve: buffers reused behind the leading barrier
        np.save(os.path.join(outdir, f"r{rank}.npy"), out.numpy())
        np.save(os.path.join(outdir, "a0.npy"), a0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,T", [([16, 32], 7), ([8, 64], 50), ([8, 4, 16], 5)])
def test_slab_decomposition_gloo_world2(orc, dims, T):
    world = 2
    seed = 4242 + len(dims)
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), dims, seed, T, td), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(td, f"r{r}.npy")) for r in range(world)])
        a0 = np.load(os.path.join(td, "a0.npy"))
    kern = R.random_kernel(R.Rng(seed), len(dims), 1, 1, 0.95)
    want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), T)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


@pytest.mark.parametrize("dims,T", [([16, 32], 7), ([8, 64], 50)])
def test_slab_p2p_exchange_gloo_world2(orc, dims, T):
    """The fused-exchange (p2p) sequence of SlabSolver -- stores into the
    owners' buffers, barrier, spectral pass, barrier, loads -- with every
    rank's buffer a shared file (the CPU stand-in for symmetric memory)."""
    world = 2
    seed = 5151 + dims[0]
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), dims, seed, T, td, "p2p"), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(td, f"r{r}.npy")) for r in range(world)])
        a0 = np.load(os.path.join(td, "a0.npy"))
    kern = R.random_kernel(R.Rng(seed), len(dims), 1, 1, 0.95)
    want = orc.solve_periodic(a0, dims, 1, *kern.arrays(), T)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


def test_slab_describe_layout():
    from paper_2105_06676_b200 import GridShape, SpecError
    from paper_2105_06676_b200.distributed import slab_describe

    info = slab_describe(GridShape([8192, 8192]), 8, 3)
    assert info["local_dims"] == [1024, 8192] and info["plane_offset"] == 3072
    assert info["col_block"] * 8 >= 4097 and info["col_block"] % 8 == 0
    assert info["xbuf_bytes"] == 8192 * info["col_block"] * 16
    info3 = slab_describe(GridShape([1024, 1024, 1024]), 8, 0)
    assert info3["local_dims"] == [128, 1024, 1024] and info3["col_block"] == 128
    with pytest.raises(SpecError):
        slab_describe(GridShape([12, 16]), 8, 0)
    with pytest.raises(SpecError):
        slab_describe(GridShape([1024]), 2, 0)
