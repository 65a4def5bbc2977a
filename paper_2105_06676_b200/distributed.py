"""Slab-decomposed multi-GPU StencilFFT-P (one process per GPU).

Rank r of P owns planes [r*n0/P, (r+1)*n0/P) of axis 0 of a rank-2/3 scalar
grid.  One solve:

    fsx_slab_forward   local R2C rows (+ local axis-1 pass in 3D), written
                       straight into the all-to-all layout (P column blocks)
    all_to_all         equal-split exchange over NCCL / NVLink
    fsx_slab_spectral  fused axis-0 pass on this rank's column block
                       (global column offset in the symbol)
    all_to_all         back
    fsx_slab_inverse   local C2R rows (+ inverse axis-1 pass in 3D)

The numerical stages run in libfsx.so on the caller's current CUDA stream;
only the exchange goes through ``torch.distributed`` (``nccl`` on GPUs).
The stage object is pluggable so the decomposition itself (layouts,
offsets, exchange pattern) can be exercised on CPU ranks over ``gloo`` with
a reference stage implementation (tests/test_distributed_cpu.py).
"""
from __future__ import annotations

import ctypes

from . import _lib
from .fftstencil import GridShape, StencilKernel, _opts


class FsxSlabInfo(ctypes.Structure):
    _fields_ = [
        ("nranks", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("local_dims", ctypes.c_int64 * _lib.MAX_RANK),
        ("plane_offset", ctypes.c_int64),
        ("col_block", ctypes.c_int64),
        ("xbuf_bytes", ctypes.c_int64),
    ]


def slab_describe(shape: GridShape, nranks: int, rank: int) -> dict:
    info = FsxSlabInfo()
    _lib.check(_lib.load().fsx_slab_describe(ctypes.byref(shape._c()), ctypes.c_int32(nranks), ctypes.c_int32(rank),
                                             ctypes.byref(info)))
    return {"local_dims": list(info.local_dims[:shape.rank()]), "plane_offset": info.plane_offset,
            "col_block": info.col_block, "xbuf_bytes": info.xbuf_bytes, "nranks": nranks, "rank": rank}


class GpuSlabStages:
    """The three device stages of one rank (libfsx.so); tensors are CUDA
    float64 tensors, work is enqueued on torch's current stream."""

    def __init__(self, shape: GridShape, nranks: int, rank: int, device: int = 0):
        self.shape, self.P, self.r, self.device = shape, nranks, rank, device

    def _stream(self):
        import torch

        return torch.cuda.current_stream().cuda_stream

    def forward(self, local_in, send) -> None:
        _lib.check(_lib.load().fsx_slab_forward(
            ctypes.byref(self.shape._c()), ctypes.c_int32(self.P), ctypes.c_int32(self.r),
            ctypes.c_void_p(local_in.data_ptr()), ctypes.c_void_p(send.data_ptr()),
            ctypes.byref(_opts(self.device, 0, self._stream()))))

    def spectral(self, recv, kernel: StencilKernel, T: int) -> None:
        kc, keep = kernel._c()
        _lib.check(_lib.load().fsx_slab_spectral(
            ctypes.byref(self.shape._c()), ctypes.byref(kc), ctypes.c_uint64(int(T)), ctypes.c_int32(self.P),
            ctypes.c_int32(self.r), ctypes.c_void_p(recv.data_ptr()), ctypes.byref(_opts(self.device, 0, self._stream()))))
        del keep

    def inverse(self, send, local_out) -> None:
        _lib.check(_lib.load().fsx_slab_inverse(
            ctypes.byref(self.shape._c()), ctypes.c_int32(self.P), ctypes.c_int32(self.r),
            ctypes.c_void_p(send.data_ptr()), ctypes.c_void_p(local_out.data_ptr()),
            ctypes.byref(_opts(self.device, 0, self._stream()))))

    # exchange fused into the row passes (2D): `peers` = device address of an
    # array of P device pointers (every rank's exchange buffer, NVLink-mapped)
    def forward_p2p(self, local_in, peers: int) -> None:
        _lib.check(_lib.load().fsx_slab_forward_p2p(
            ctypes.byref(self.shape._c()), ctypes.c_int32(self.P), ctypes.c_int32(self.r),
            ctypes.c_void_p(local_in.data_ptr()), ctypes.c_void_p(peers),
            ctypes.byref(_opts(self.device, 0, self._stream()))))

    def inverse_p2p(self, peers: int, local_out) -> None:
        _lib.check(_lib.load().fsx_slab_inverse_p2p(
            ctypes.byref(self.shape._c()), ctypes.c_int32(self.P), ctypes.c_int32(self.r),
            ctypes.c_void_p(peers), ctypes.c_void_p(local_out.data_ptr()),
            ctypes.byref(_opts(self.device, 0, self._stream()))))


class SymmetricPeerMemory:
    """The p2p exchange buffer: torch symmetric memory (each rank's buffer
    mapped into every process over NVLink) and its device-side barrier."""

    def __init__(self, nelem: int, device, group):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.local = symm.empty(nelem, dtype=torch.float64, device=device)
        self.handle = symm.rendezvous(self.local, group if group is not None else dist.group.WORLD)
        self.peers = int(self.handle.buffer_ptrs_dev)  # device array of P device pointers

    def barrier(self, channel: int) -> None:
        self.handle.barrier(channel=channel)


class SlabSolver:
    """solve_periodic over a process group, one slab per rank.

    exchange="nccl": two all_to_all_single calls per solve.
    exchange="p2p" (2D, GPUs): the exchange buffer is torch symmetric memory
    (every rank's buffer mapped into every process over NVLink); the R2C rows
    store their column blocks straight into the owners' buffers and the C2R
    rows load them back, separated by the symmetric-memory device barrier --
    no all-to-all, the NVLink traffic overlaps the row FFTs."""

    def __init__(self, shape: GridShape, kernel: StencilKernel, T: int, group=None, stages=None, device=None,
                 exchange: str = "nccl", peer_memory=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.r = dist.get_rank(group)
        self.shape, self.kernel, self.T = shape, kernel, int(T)
        kernel.require_fits(shape)
        self.info = slab_describe(shape, self.P, self.r)
        if stages is None:
            dev = torch.cuda.current_device() if device is None else device
            stages = GpuSlabStages(shape, self.P, self.r, dev)
            self.tdev = torch.device("cuda", dev)
        else:
            self.tdev = torch.device("cpu")
        self.stages = stages
        n = self.info["xbuf_bytes"] // 8
        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange = exchange
        if exchange == "p2p":
            if shape.rank() != 2:
                raise ValueError("p2p exchange: rank-2 grids")
            if peer_memory is None:
                if self.tdev.type != "cuda":
                    raise ValueError("p2p exchange on CPU ranks needs an explicit peer_memory")
                peer_memory = SymmetricPeerMemory(n, self.tdev, group)
            self.pm = peer_memory
            self.recv = peer_memory.local
            self.peers = peer_memory.peers
            self.send = None
        else:
            self.send = torch.empty(n, dtype=torch.float64, device=self.tdev)
            self.recv = torch.empty(n, dtype=torch.float64, device=self.tdev)

    def local_cells(self) -> int:
        c = 1
        for d in self.info["local_dims"]:
            c *= d
        return c

    def a2a_bytes(self) -> int:
        """Bytes this rank sends to other ranks per all-to-all."""
        return self.info["xbuf_bytes"] * (self.P - 1) // self.P

    def solve(self, local_in, local_out, events=None) -> None:
        """local_in / local_out: this rank's slab (float64, P-th of axis 0).
        `events` (optional list of 6 CUDA events) stamps the stage boundaries."""
        def mark(i):
            if events is not None:
                events[i].record()

        if self.exchange == "p2p":
            # events: [0,1) barrier + R2C rows storing over NVLink, [1,2) barrier,
            # [2,3) fused pass, [3,4) barrier, [4,5) C2R rows loading over NVLink
            mark(0)
            self.pm.barrier(0)  # every rank done reading the buffers (previous solve)
            self.stages.forward_p2p(local_in, self.peers)
            mark(1)
            self.pm.barrier(1)  # all blocks stored into their owners' buffers
            mark(2)
            self.stages.spectral(self.recv, self.kernel, self.T)
            mark(3)
            self.pm.barrier(2)  # every rank's spectral pass done
            mark(4)
            self.stages.inverse_p2p(self.peers, local_out)
            mark(5)
            return
        mark(0)
        self.stages.forward(local_in, self.send)
        mark(1)
        self.dist.all_to_all_single(self.recv, self.send, group=self.group)
        mark(2)
        self.stages.spectral(self.recv, self.kernel, self.T)
        mark(3)
        self.dist.all_to_all_single(self.send, self.recv, group=self.group)
        mark(4)
        self.stages.inverse(self.send, local_out)
        mark(5)


def slab_solve_emulated(shape: GridShape, a0, kernel: StencilKernel, T: int, P: int, out=None):
    """Runs the P-rank slab solve on ONE GPU: every rank's stages execute in
    turn and the all-to-all is a device-to-device block shuffle.  Exercises
    the multi-rank layouts and global offsets of the GPU stages without a
    second device (no rank waits on another)."""
    import torch

    n0 = shape.dim(0)
    if out is None:
        out = torch.empty_like(a0)
    rows = a0.view(n0, -1)
    orows = out.view(n0, -1)
    infos = [slab_describe(shape, P, r) for r in range(P)]
    n = infos[0]["xbuf_bytes"] // 8
    chunk = n // P
    send = [torch.empty(n, dtype=torch.float64, device=a0.device) for _ in range(P)]
    recv = [torch.empty(n, dtype=torch.float64, device=a0.device) for _ in range(P)]
    stages = [GpuSlabStages(shape, P, r, a0.device.index or 0) for r in range(P)]
    n0l = n0 // P
    for r in range(P):
        stages[r].forward(rows[r * n0l:(r + 1) * n0l], send[r])
    for s in range(P):
        for d in range(P):
            recv[d][s * chunk:(s + 1) * chunk].copy_(send[s][d * chunk:(d + 1) * chunk])
    for r in range(P):
        stages[r].spectral(recv[r], kernel, T)
    for d in range(P):
        for s in range(P):
            send[s][d * chunk:(d + 1) * chunk].copy_(recv[d][s * chunk:(s + 1) * chunk])
    for r in range(P):
        stages[r].inverse(send[r], orows[r * n0l:(r + 1) * n0l])
    return out


def slab_solve_emulated_p2p(shape: GridShape, a0, kernel: StencilKernel, T: int, P: int, out=None):
    """The fused-exchange (p2p) slab solve of P ranks on ONE GPU: the P
    exchange buffers are separate allocations on this device and the peer
    pointer array lists them, so each rank's row kernels store to / load from
    the other "ranks'" buffers exactly as over NVLink.  Stages run rank after
    rank (the barriers are implicit; no rank waits on another)."""
    import torch

    n0 = shape.dim(0)
    if out is None:
        out = torch.empty_like(a0)
    rows = a0.view(n0, -1)
    orows = out.view(n0, -1)
    info = slab_describe(shape, P, 0)
    n = info["xbuf_bytes"] // 8
    bufs = [torch.empty(n, dtype=torch.float64, device=a0.device) for _ in range(P)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=a0.device)
    stages = [GpuSlabStages(shape, P, r, a0.device.index or 0) for r in range(P)]
    n0l = n0 // P
    for r in range(P):
        stages[r].forward_p2p(rows[r * n0l:(r + 1) * n0l], peers.data_ptr())
    for r in range(P):
        stages[r].spectral(bufs[r], kernel, T)
    for r in range(P):
        stages[r].inverse_p2p(peers.data_ptr(), orows[r * n0l:(r + 1) * n0l])
    torch.cuda.current_stream().synchronize()
    return out
