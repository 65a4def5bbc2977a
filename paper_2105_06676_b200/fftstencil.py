"""Python mirror of the reference fftstencil periodic API over the C ABI.

Same names, argument meaning and error behaviour as the reference C++
library's hot path (proj/include/fftstencil/{grid,kernel,spectrum,fft,
periodic}.hpp), so the parity tests read like the reference's own tests:

    k = StencilKernel(1); k.add_tap([-1], 0.25); ...
    out = solve_periodic(FieldGrid(GridShape([1 << 20]), a0), k, 1000)

All numerical work runs on the GPU through libfsx.so (include/fsx.h); this
module only builds arguments, validates value types the way the reference
constructors do, and maps status codes to the reference exception types.
"""
from __future__ import annotations

import ctypes
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import CudaError, Error, NumericError, SpecError  # noqa: F401

_DP = ctypes.POINTER(ctypes.c_double)
_I64P = ctypes.POINTER(ctypes.c_int64)


# ---------------------------------------------------------------- value types
class GridShape:
    """proj/include/fftstencil/grid.hpp:21-83 (int64 dims, m fields, overflow-checked)."""

    def __init__(self, dims: Sequence[int], fields: int = 1):
        dims = [int(d) for d in dims]
        if not dims:
            raise SpecError("GridShape: need at least one dimension")
        if len(dims) > _lib.MAX_RANK:
            raise SpecError(f"GridShape: rank > {_lib.MAX_RANK} not supported")
        if fields < 1:
            raise SpecError("GridShape: fields must be >= 1")
        n = 1
        for d in dims:
            if d < 1:
                raise SpecError("GridShape: every dimension must be >= 1")
            n *= d
            if n * fields > (1 << 63) - 1:
                raise SpecError("GridShape: total value count overflows")
        self._dims = tuple(dims)
        self._fields = int(fields)
        self._cells = n

    def rank(self) -> int:
        return len(self._dims)

    def dims(self):
        return list(self._dims)

    def dim(self, axis: int) -> int:
        return self._dims[axis]

    def fields(self) -> int:
        return self._fields

    def cells(self) -> int:
        return self._cells

    def values(self) -> int:
        return self._cells * self._fields

    def min_dim(self) -> int:
        return min(self._dims)

    def __eq__(self, other):
        return isinstance(other, GridShape) and self._dims == other._dims and self._fields == other._fields

    def __repr__(self):
        return f"GridShape({list(self._dims)}, fields={self._fields})"

    def _c(self) -> _lib.FsxShape:
        s = self.__dict__.get("_cs")  # immutable: build the C view once
        if s is None:
            s = _lib.FsxShape()
            s.rank = len(self._dims)
            s.fields = self._fields
            for i, d in enumerate(self._dims):
                s.dims[i] = d
            self._cs = s
        return s


class _Grid:
    dtype = np.float64

    def __init__(self, shape: GridShape, data=None):
        self.shape = shape
        if data is None:
            self.data = np.zeros(shape.values(), dtype=self.dtype)
        else:
            arr = np.ascontiguousarray(np.asarray(data, dtype=self.dtype).reshape(-1))
            if arr.size != shape.values():
                raise SpecError("Grid: data length does not match the shape")
            self.data = arr

    def at(self, cell: int, field: int = 0):
        return self.data[cell * self.shape.fields() + field]

    def copy(self):
        return type(self)(self.shape, self.data.copy())


class FieldGrid(_Grid):
    """Real grid, row-major cells with the field innermost (grid.hpp:17-20, 86-100)."""

    dtype = np.float64


class ComplexGrid(_Grid):
    dtype = np.complex128


class StencilKernel:
    """Sparse offset -> m x m block map (kernel.hpp:19-56, kernel.cpp:7-49)."""

    def __init__(self, rank: int, fields: int = 1):
        if rank < 1:
            raise SpecError("StencilKernel: rank must be >= 1")
        if fields < 1:
            raise SpecError("StencilKernel: fields must be >= 1")
        self._rank, self._fields = int(rank), int(fields)
        self._taps: dict[tuple, np.ndarray] = {}
        self._cc = None  # cached fsx_kernel view (dropped by add_tap)

    def add_tap(self, offset: Iterable[int], block) -> "StencilKernel":
        off = tuple(int(o) for o in offset)
        if len(off) != self._rank:
            raise SpecError("StencilKernel: offset rank mismatch")
        if np.isscalar(block):
            if self._fields != 1:
                raise SpecError("StencilKernel: scalar tap on a multi-field kernel")
            b = np.array([[float(block)]])
        else:
            b = np.array(block, dtype=np.float64)
            if b.shape != (self._fields, self._fields):
                raise SpecError("StencilKernel: block must be fields x fields")
        if not np.isfinite(b).all():
            raise SpecError("StencilKernel: non-finite coefficient")
        self._cc = None
        if off in self._taps:
            self._taps[off] = self._taps[off] + b
        else:
            self._taps[off] = b
        return self

    def taps(self):
        return {k: self._taps[k] for k in sorted(self._taps)}

    def rank(self) -> int:
        return self._rank

    def fields(self) -> int:
        return self._fields

    def empty(self) -> bool:
        return not self._taps

    def radius(self) -> int:
        return max((max((abs(o) for o in off), default=0) for off in self._taps), default=0)

    def max_reach(self):
        reach = [0] * self._rank
        for off in self._taps:
            for a in range(self._rank):
                reach[a] = max(reach[a], abs(off[a]))
        return reach

    def require_nonempty(self):
        if not self._taps:
            raise SpecError("StencilKernel: at least one tap required")

    def require_fits(self, shape: GridShape):
        self.require_nonempty()
        if shape.rank() != self._rank:
            raise SpecError("StencilKernel: grid rank mismatch")
        if shape.fields() != self._fields:
            raise SpecError("StencilKernel: grid field count mismatch")
        for a, r in enumerate(self.max_reach()):
            if r >= shape.dim(a):
                raise SpecError(f"StencilKernel: tap offset exceeds dimension {a}")

    def arrays(self):
        keys = sorted(self._taps)
        off = np.array(keys, dtype=np.int64).reshape(len(keys), self._rank)
        blk = np.array([self._taps[k] for k in keys], dtype=np.float64).reshape(len(keys), self._fields, self._fields)
        return np.ascontiguousarray(off), np.ascontiguousarray(blk)

    def _c(self):
        if self._cc is None:
            off, blk = self.arrays()
            k = _lib.FsxKernel()
            k.rank, k.fields, k.ntaps = self._rank, self._fields, off.shape[0]
            k.offsets = off.ctypes.data_as(_I64P)
            k.blocks = blk.ctypes.data_as(_DP)
            self._cc = (k, (off, blk))
        return self._cc



def _u64_T(T) -> "ctypes.c_uint64":
    """T as the C ABI's uint64_t; the reference's T is uint64_t
    (proj/include/fftstencil/periodic.hpp:43): outside [0, 2^64) is a SpecError
    (never a silent wrap-around)."""
    T = int(T)
    if T < 0 or T >= 1 << 64:
        raise SpecError(f"T must be in [0, 2^64), got {T}")
    return ctypes.c_uint64(T)


def fold_kernels(kset) -> StencilKernel:
    """proj/src/kernel.cpp:51-81: m x m matrix of scalar kernels -> one m x m-block kernel."""
    m = len(kset)
    if m < 1:
        raise SpecError("fold_kernels: empty kernel matrix")
    rank = -1
    for row in kset:
        if len(row) != m:
            raise SpecError("fold_kernels: kernel matrix must be square")
        for k in row:
            if k.fields() != 1:
                raise SpecError("fold_kernels: entries must be scalar kernels")
            if not k.empty():
                if rank == -1:
                    rank = k.rank()
                if k.rank() != rank:
                    raise SpecError("fold_kernels: mixed kernel ranks")
    if rank == -1:
        raise SpecError("fold_kernels: all entries empty")
    folded = StencilKernel(rank, m)
    for i in range(m):
        for j in range(m):
            for off, blk in kset[i][j].taps().items():
                b = np.zeros((m, m))
                b[i, j] = blk[0, 0]
                folded.add_tap(off, b)
    return folded


class StageTimings:
    """proj/include/fftstencil/periodic.hpp:14-23 (seconds, accumulated)."""

    def __init__(self):
        self.forward_fft = 0.0
        self.squaring = 0.0
        self.hadamard = 0.0
        self.inverse_fft = 0.0
        self.boundary_recursion = 0.0

    def sum(self) -> float:
        return self.forward_fft + self.squaring + self.hadamard + self.inverse_fft + self.boundary_recursion

    def _pull(self, c: _lib.FsxStageTimings):
        self.forward_fft, self.squaring, self.hadamard = c.forward_fft, c.squaring, c.hadamard
        self.inverse_fft, self.boundary_recursion = c.inverse_fft, c.boundary_recursion

    def _push(self) -> _lib.FsxStageTimings:
        c = _lib.FsxStageTimings()
        c.forward_fft, c.squaring, c.hadamard = self.forward_fft, self.squaring, self.hadamard
        c.inverse_fft, c.boundary_recursion = self.inverse_fft, self.boundary_recursion
        return c


class SpectrumCache:
    """proj/include/fftstencil/periodic.hpp:28-35 (device plans memoised by dims)."""

    def __init__(self):
        self._h = ctypes.c_void_p(_lib.load().fsx_spectrum_cache_create())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._lib is not None:
            _lib._lib.fsx_spectrum_cache_destroy(h)


class DiagonalSpectrum:
    """proj/include/fftstencil/spectrum.hpp:16-38: frequency-major m x m blocks."""

    def __init__(self, shape: GridShape, blocks=None):
        self.shape = shape
        m = shape.fields()
        n = shape.cells() * m * m
        self.blocks = (np.zeros(n, np.complex128) if blocks is None
                       else np.ascontiguousarray(np.asarray(blocks, np.complex128).reshape(-1)))
        if self.blocks.size != n:
            raise SpecError("DiagonalSpectrum: block count does not match the shape")

    def block_dim(self) -> int:
        return self.shape.fields()

    def entry(self, freq: int, r: int, c: int):
        m = self.shape.fields()
        return self.blocks[freq * m * m + r * m + c]

    def block(self, freq: int) -> np.ndarray:
        m = self.shape.fields()
        return self.blocks[freq * m * m:(freq + 1) * m * m].reshape(m, m)

    def set_block(self, freq: int, b) -> None:
        m = self.shape.fields()
        self.blocks[freq * m * m:(freq + 1) * m * m] = np.asarray(b, np.complex128).reshape(-1)


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: the NULL stream's explicit handle


_OPTS: dict = {}  # option structs are read-only for the library: reuse them


def _opts(device: int = 0, path: int = 0, stream: int | None = None, stage_events: int = 0, spectral_cut: int = 0,
          num_gpus: int = 0, exchange: int = 0, devices=None, decomp: int = 0, pencil_rows: int = 0):
    """fsx_options.  stream None -> the library's own stream; a handle of 0
    (torch's default stream) is passed as cudaStreamLegacy so the work is
    ordered with the caller's NULL-stream work instead of the library stream.
    num_gpus / exchange / devices: the single-process multi-GPU path (fsx.h)."""
    devices = tuple(int(d) for d in devices) if devices is not None else None
    key = (device, path, stream, stage_events, spectral_cut, num_gpus, exchange, devices, decomp, pencil_rows)
    o = _OPTS.get(key)
    if o is None:
        o = _lib.FsxOptions()
        o.device, o.path, o.stage_events, o.spectral_cut = device, path, stage_events, int(bool(spectral_cut))
        o.stream = None if stream is None else (stream or CUDA_STREAM_LEGACY)
        o.num_gpus, o.exchange = num_gpus, exchange
        o.decomp, o.pencil_rows = decomp, pencil_rows
        if devices is not None:
            o._devs = (ctypes.c_int32 * len(devices))(*devices)  # kept alive with the struct
            o.devices = ctypes.cast(o._devs, ctypes.POINTER(ctypes.c_int32))
            o.num_gpus = len(devices)
        if len(_OPTS) > 256:
            _OPTS.clear()
        _OPTS[key] = o
    return o


def set_devices(devices=None, n: int | None = None) -> None:
    """Process default device list of host solves (fsx_set_devices): eligible
    2D/3D grids are then slab-decomposed over these devices by every
    solve_periodic call that does not pass its own ``devices``.  ``[]`` or
    one device -> single GPU.  A repeated ordinal emulates ranks on one GPU."""
    L = _lib.load()
    if devices is None:
        _lib.check(L.fsx_set_devices(None, ctypes.c_int32(int(n or 0))))
        return
    devs = [int(d) for d in devices]
    arr = (ctypes.c_int32 * max(1, len(devs)))(*devs)
    _lib.check(L.fsx_set_devices(arr, ctypes.c_int32(len(devs))))


def get_devices() -> list:
    L = _lib.load()
    n = L.fsx_get_devices(None, ctypes.c_int32(0))
    arr = (ctypes.c_int32 * max(1, n))()
    L.fsx_get_devices(arr, ctypes.c_int32(n))
    return [int(arr[i]) for i in range(n)]


# ---------------------------------------------------------------- solvers
def _solve(fn, a0: FieldGrid, k: StencilKernel, T: int, st: StageTimings | None, path: int, extra=(), out=None,
           spectral_cut: int = 0, multi: dict | None = None):
    L = _lib.load()
    if T < 0 or T >= 1 << 64:
        raise SpecError("T must be a nonnegative 64-bit integer")
    shape_c = a0.shape._c()
    kc, keep = k._c()
    if out is None:
        out = np.empty_like(a0.data)
    elif out.dtype != np.float64 or out.size != a0.data.size or not out.flags.c_contiguous:
        raise SpecError("out must be a contiguous float64 array of the grid's size")
    stc = st._push() if st is not None else None
    status = getattr(L, fn)(ctypes.byref(shape_c), a0.data.ctypes.data_as(_DP), ctypes.byref(kc),
                            _u64_T(T), *extra, out.ctypes.data_as(_DP),
                            ctypes.byref(_opts(path=path, spectral_cut=spectral_cut, **(multi or {}))),
                            ctypes.byref(stc) if stc is not None else None)
    del keep
    _lib.check(status)
    if st is not None:
        st._pull(stc)
    return FieldGrid(a0.shape, out)


def solve_periodic(a0: FieldGrid, k: StencilKernel, T: int, st: StageTimings | None = None, *, path: int = 0,
                   out: np.ndarray | None = None, spectral_cut: int = 0, num_gpus: int = 0, devices=None,
                   exchange: int = 0, decomp: int = 0, pencil_rows: int = 0):
    """proj/src/periodic.cpp:76-86 on the B200 path (fsx_solve_periodic).
    ``out`` optionally supplies the (e.g. pinned) host array the result is written to.
    ``spectral_cut=1``: the exact spectral cut (fsx_options.spectral_cut; same result).
    ``num_gpus`` / ``devices`` / ``exchange`` (0 auto, 1 p2p, 2 nccl): slab-decompose an
    eligible 2D/3D grid over several GPUs of this process (fsx_options; 0 = the
    process default of set_devices)."""
    multi = {"num_gpus": num_gpus, "exchange": exchange, "devices": devices, "decomp": decomp,
             "pencil_rows": pencil_rows}
    return _solve("fsx_solve_periodic", a0, k, T, st, path, out=out, spectral_cut=spectral_cut, multi=multi)


def solve_periodic_vector(a0: FieldGrid, k: StencilKernel, T: int, st: StageTimings | None = None, *, path: int = 0):
    """proj/src/periodic.cpp:101-106 (fsx_solve_periodic_vector)."""
    return _solve("fsx_solve_periodic_vector", a0, k, T, st, path)


def solve_periodic_cached(a0: FieldGrid, k: StencilKernel, T: int, cache: SpectrumCache,
                          st: StageTimings | None = None):
    """proj/src/periodic.cpp:88-99 (fsx_solve_periodic_cached)."""
    L = _lib.load()
    shape_c = a0.shape._c()
    kc, keep = k._c()
    out = np.empty_like(a0.data)
    stc = st._push() if st is not None else None
    status = L.fsx_solve_periodic_cached(ctypes.byref(shape_c), a0.data.ctypes.data_as(_DP), ctypes.byref(kc),
                                         _u64_T(T), cache._h, out.ctypes.data_as(_DP),
                                         ctypes.byref(_opts()), ctypes.byref(stc) if stc is not None else None)
    del keep
    _lib.check(status)
    if st is not None:
        st._pull(stc)
    return FieldGrid(a0.shape, out)


def solve_periodic_implicit(q: StencilKernel, s: StencilKernel, a0: FieldGrid, T: int,
                            st: StageTimings | None = None):
    """proj/src/periodic.cpp:108-124 (fsx_solve_periodic_implicit)."""
    L = _lib.load()
    shape_c = a0.shape._c()
    qc, kq = q._c()
    sc, ks = s._c()
    out = np.empty_like(a0.data)
    stc = st._push() if st is not None else None
    status = L.fsx_solve_periodic_implicit(ctypes.byref(shape_c), a0.data.ctypes.data_as(_DP), ctypes.byref(qc),
                                           ctypes.byref(sc), _u64_T(T), out.ctypes.data_as(_DP),
                                           ctypes.byref(_opts()), ctypes.byref(stc) if stc is not None else None)
    del kq, ks
    _lib.check(status)
    if st is not None:
        st._pull(stc)
    return FieldGrid(a0.shape, out)


def solve_periodic_batch(a0s, k: StencilKernel, T: int, outs=None, spectral_cut: int = 0) -> list:
    """Pipelined batch of independent solves (fsx_solve_periodic_batch): one
    shape, kernel and T for every grid.  ``a0s`` are FieldGrids; ``outs``
    optionally supplies the host result arrays (pinned for full H2D/D2H
    overlap).  Returns the output arrays."""
    if T < 0 or T >= 1 << 64:
        raise SpecError("T must be a nonnegative 64-bit integer")
    grids = list(a0s)
    if not grids:
        return []
    shape = grids[0].shape
    for g in grids:
        if g.shape.dims() != shape.dims() or g.shape.fields() != shape.fields():
            raise SpecError("solve_periodic_batch: all grids must share one shape")
    if outs is None:
        outs = [np.empty_like(g.data) for g in grids]
    outs = list(outs)
    if len(outs) != len(grids):
        raise SpecError("solve_periodic_batch: one output per input")
    for o in outs:
        if o.dtype != np.float64 or o.size != grids[0].data.size or not o.flags.c_contiguous:
            raise SpecError("out must be a contiguous float64 array of the grid's size")
    n = len(grids)
    ins = (ctypes.c_void_p * n)(*[g.data.ctypes.data for g in grids])
    ous = (ctypes.c_void_p * n)(*[o.ctypes.data for o in outs])
    L = _lib.load()
    kc, keep = k._c()
    status = L.fsx_solve_periodic_batch(ctypes.byref(shape._c()), ctypes.c_int64(n), ins, ctypes.byref(kc),
                                        _u64_T(T), ous, ctypes.byref(_opts(spectral_cut=spectral_cut)))
    del keep
    _lib.check(status)
    return outs


def solve_periodic_slabs(a0s, k: StencilKernel, T: int, cache: SpectrumCache | None = None,
                         st: StageTimings | None = None, outs=None) -> list:
    """One recursion level's slab solves (fsx_solve_periodic_slabs): the
    aperiodic recursion's rb_run solves the 2d face slabs of a level with
    solve_periodic_cached one after another (proj/src/aperiodic.cpp:224-228,
    240-244); here the FieldGrids ``a0s`` (shapes may differ) are solved in one
    call -- equal shapes stacked into one batched plan, shape groups
    overlapped on two lanes.  ``cache``: SpectrumCache semantics (first kernel
    per dims).  Returns the output arrays (``outs`` optionally supplies them)."""
    if T < 0 or T >= 1 << 64:
        raise SpecError("T must be a nonnegative 64-bit integer")
    grids = list(a0s)
    n = len(grids)
    if outs is None:
        outs = [np.empty_like(g.data) for g in grids]
    outs = list(outs)
    if len(outs) != n:
        raise SpecError("solve_periodic_slabs: one output per input")
    for g, o in zip(grids, outs):
        if o.dtype != np.float64 or o.size != g.data.size or not o.flags.c_contiguous:
            raise SpecError("out must be a contiguous float64 array of the grid's size")
    shapes = (_lib.FsxShape * max(1, n))(*[g.shape._c() for g in grids])
    ins = (ctypes.c_void_p * max(1, n))(*[g.data.ctypes.data for g in grids])
    ous = (ctypes.c_void_p * max(1, n))(*[o.ctypes.data for o in outs])
    L = _lib.load()
    kc, keep = k._c()
    stc = st._push() if st is not None else None
    status = L.fsx_solve_periodic_slabs(ctypes.c_int64(n), shapes, ins, ctypes.byref(kc), _u64_T(T),
                                        cache._h if cache is not None else None, ous, ctypes.byref(_opts()),
                                        ctypes.byref(stc) if stc is not None else None)
    del keep
    _lib.check(status)
    if st is not None:
        st._pull(stc)
    return outs


def solve_periodic_device(shape: GridShape, d_a0: int, k: StencilKernel, T: int, d_out: int,
                          stream: int | None = None, device: int = 0, path: int = 0, stage_events: int = 0,
                          spectral_cut: int = 0) -> None:
    """Device-resident solve (fsx_solve_periodic_device): pointers are CUDA
    device addresses (e.g. ``tensor.data_ptr()``); enqueued on ``stream``.
    Call :func:`device_check` to synchronize and surface NumericError."""
    L = _lib.load()
    shape_c = shape._c()
    kc, keep = k._c()
    status = L.fsx_solve_periodic_device(ctypes.byref(shape_c), ctypes.c_void_p(d_a0), ctypes.byref(kc),
                                         _u64_T(T), ctypes.c_void_p(d_out),
                                         ctypes.byref(_opts(device, path, stream, stage_events, spectral_cut)))
    del keep
    _lib.check(status)


# ---------------------------------------------------------------- fp32 storage mode
_FP = ctypes.POINTER(ctypes.c_float)


def _f32(a, n: int, what: str) -> np.ndarray:
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or a.size != n or not a.flags.c_contiguous:
        raise SpecError(f"{what} must be a contiguous float32 array of the grid's size")
    return a


def solve_periodic_f32(shape: GridShape, a0: np.ndarray, k: StencilKernel, T: int, st: StageTimings | None = None,
                       *, path: int = 0, out: np.ndarray | None = None, spectral_cut: int = 0) -> np.ndarray:
    """fp32 mode (fsx_solve_periodic_f32): float32 grid in and out; the north
    star's optional fp32 mode (<= 1e-4 relative L2 vs the fp64 reference).
    The symbol power is fp64; the fused column pass of a real symbol runs its
    FFTs in fp32 (~1e-7); other paths are fp64 arithmetic rounded once.
    Returns the float32 result."""
    if T < 0 or T >= 1 << 64:
        raise SpecError("T must be a nonnegative 64-bit integer")
    n = int(np.prod(shape.dims())) * shape.fields()
    a0 = _f32(a0, n, "a0")
    out = np.empty_like(a0) if out is None else _f32(out, n, "out")
    L = _lib.load()
    kc, keep = k._c()
    stc = st._push() if st is not None else None
    status = L.fsx_solve_periodic_f32(ctypes.byref(shape._c()), a0.ctypes.data_as(_FP), ctypes.byref(kc),
                                      _u64_T(T), out.ctypes.data_as(_FP),
                                      ctypes.byref(_opts(path=path, spectral_cut=spectral_cut)),
                                      ctypes.byref(stc) if stc is not None else None)
    del keep
    _lib.check(status)
    if st is not None:
        st._pull(stc)
    return out


def solve_periodic_batch_f32(shape: GridShape, a0s, k: StencilKernel, T: int, outs=None, spectral_cut: int = 0) -> list:
    """Pipelined batch in the fp32 storage mode (fsx_solve_periodic_batch_f32)."""
    if T < 0 or T >= 1 << 64:
        raise SpecError("T must be a nonnegative 64-bit integer")
    n = int(np.prod(shape.dims())) * shape.fields()
    ins = [_f32(a, n, "a0") for a in a0s]
    if not ins:
        return []
    outs = [np.empty_like(a) for a in ins] if outs is None else [_f32(o, n, "out") for o in outs]
    if len(outs) != len(ins):
        raise SpecError("solve_periodic_batch_f32: one output per input")
    m = len(ins)
    pi = (ctypes.c_void_p * m)(*[a.ctypes.data for a in ins])
    po = (ctypes.c_void_p * m)(*[o.ctypes.data for o in outs])
    L = _lib.load()
    kc, keep = k._c()
    status = L.fsx_solve_periodic_batch_f32(ctypes.byref(shape._c()), ctypes.c_int64(m), pi, ctypes.byref(kc),
                                            _u64_T(T), po, ctypes.byref(_opts(spectral_cut=spectral_cut)))
    del keep
    _lib.check(status)
    return outs


def solve_periodic_device_f32(shape: GridShape, d_a0: int, k: StencilKernel, T: int, d_out: int,
                              stream: int | None = None, device: int = 0, path: int = 0, stage_events: int = 0,
                              spectral_cut: int = 0) -> None:
    """Device-resident fp32 storage mode (fsx_solve_periodic_device_f32):
    float32 device buffers; asynchronous like :func:`solve_periodic_device`."""
    L = _lib.load()
    kc, keep = k._c()
    status = L.fsx_solve_periodic_device_f32(ctypes.byref(shape._c()), ctypes.c_void_p(d_a0), ctypes.byref(kc),
                                             _u64_T(T), ctypes.c_void_p(d_out),
                                             ctypes.byref(_opts(device, path, stream, stage_events, spectral_cut)))
    del keep
    _lib.check(status)


# ---------------------------------------------------------------- direct-stepping verifier
def step_periodic(a: FieldGrid, k: StencilKernel) -> FieldGrid:
    """proj/src/oracle.cpp:90-98 on the GPU (fsx_step_periodic): one direct
    stencil step, bitwise equal to the reference loop."""
    return evolve_periodic_naive(a, k, 1)


def evolve_periodic_naive(a0: FieldGrid, k: StencilKernel, T: int) -> FieldGrid:
    """proj/src/oracle.cpp:100-115 on the GPU (fsx_evolve_periodic_naive):
    T direct steps -- an independent check of the FFT solver, not a solver."""
    if T < 0 or T >= 1 << 64:
        raise SpecError("T must be a nonnegative 64-bit integer")
    L = _lib.load()
    kc, keep = k._c()
    out = np.empty_like(a0.data)
    status = L.fsx_evolve_periodic_naive(ctypes.byref(a0.shape._c()), a0.data.ctypes.data_as(_DP), ctypes.byref(kc),
                                         _u64_T(T), out.ctypes.data_as(_DP), ctypes.byref(_opts()))
    del keep
    _lib.check(status)
    return FieldGrid(a0.shape, out)


def evolve_periodic_naive_device(shape: GridShape, d_a0: int, k: StencilKernel, T: int, d_out: int,
                                 stream: int | None = None, device: int = 0) -> None:
    """Device-pointer variant of :func:`evolve_periodic_naive`, enqueued on ``stream``."""
    L = _lib.load()
    kc, keep = k._c()
    status = L.fsx_evolve_periodic_naive_device(ctypes.byref(shape._c()), ctypes.c_void_p(d_a0), ctypes.byref(kc),
                                                _u64_T(T), ctypes.c_void_p(d_out),
                                                ctypes.byref(_opts(device, 0, stream)))
    del keep
    _lib.check(status)


def last_stage_ms(device: int = 0) -> list:
    """[forward, fused spectral, inverse] ms of the last device solve enqueued with stage_events=1."""
    ms = (ctypes.c_double * 3)()
    _lib.check(_lib.load().fsx_last_stage_ms(ctypes.byref(_opts(device)), ms))
    return list(ms)


def device_check(stream: int | None = None, device: int = 0) -> None:
    _lib.check(_lib.load().fsx_device_check(ctypes.byref(_opts(device, 0, stream))))


def spectral_cut_columns(shape: GridShape, k: StencilKernel, T: int) -> tuple:
    """(kept, total) half-spectrum columns of the exact spectral cut for this solve
    (fsx_spectral_cut_columns; kept == total where the cut does not apply)."""
    kc, keep = k._c()
    kept, total = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.load().fsx_spectral_cut_columns(ctypes.byref(shape._c()), ctypes.byref(kc), _u64_T(T),
                                                    ctypes.byref(kept), ctypes.byref(total)))
    del keep
    return kept.value, total.value


def plan_describe(shape: GridShape, k: StencilKernel, path: int = 0, num_gpus: int = 0, devices=None,
                  exchange: int = 0, decomp: int = 0, pencil_rows: int = 0) -> dict:
    L = _lib.load()
    info = _lib.FsxPlanInfo()
    kc, keep = k._c()
    o = _opts(path=path, num_gpus=num_gpus, exchange=exchange, devices=devices, decomp=decomp, pencil_rows=pencil_rows)
    _lib.check(L.fsx_plan_describe(ctypes.byref(shape._c()), ctypes.byref(kc), ctypes.byref(o), ctypes.byref(info)))
    del keep
    return {"path": info.path, "launches": info.launches, "alg_bytes": info.alg_bytes,
            "fused_bytes": info.fused_bytes, "work_bytes": info.work_bytes, "sched_bytes": info.sched_bytes,
            "ranks": info.ranks,
            "exchange": info.exchange, "decomp": info.decomp, "pencil_rows": info.pencil_rows}


# ---------------------------------------------------------------- building blocks
def _cgrid(g) -> ComplexGrid:
    return g if isinstance(g, ComplexGrid) else ComplexGrid(g.shape, g.data.astype(np.complex128))


def multi_fft(g) -> ComplexGrid:
    """proj/src/fft.cpp:190 (+ multi_fft(FieldGrid) = multi_fft(to_complex(g)), fft.hpp:21)."""
    g = _cgrid(g)
    out = np.empty_like(g.data)
    _lib.check(_lib.load().fsx_multi_fft(ctypes.byref(g.shape._c()), g.data.ctypes.data_as(_DP),
                                         out.ctypes.data_as(_DP), ctypes.c_int32(0)))
    return ComplexGrid(g.shape, out)


def multi_ifft(g) -> ComplexGrid:
    """proj/src/fft.cpp:192"""
    g = _cgrid(g)
    out = np.empty_like(g.data)
    _lib.check(_lib.load().fsx_multi_fft(ctypes.byref(g.shape._c()), g.data.ctypes.data_as(_DP),
                                         out.ctypes.data_as(_DP), ctypes.c_int32(1)))
    return ComplexGrid(g.shape, out)


def fft(buf, inverse: bool = False) -> np.ndarray:
    """proj/src/fft.cpp:143-155 for one contiguous line (returns a new array)."""
    x = np.ascontiguousarray(np.asarray(buf, np.complex128).reshape(-1))
    if x.size <= 1:
        return x.copy()
    g = ComplexGrid(GridShape([x.size]), x)
    return (multi_ifft(g) if inverse else multi_fft(g)).data


def spectrum_from_kernel(k: StencilKernel, shape: GridShape) -> DiagonalSpectrum:
    """proj/src/spectrum.cpp:21-45 (analytic symbol on the GPU)."""
    m = shape.fields()
    out = np.empty(shape.cells() * m * m, np.complex128)
    kc, keep = k._c()
    _lib.check(_lib.load().fsx_spectrum_from_kernel(ctypes.byref(shape._c()), ctypes.byref(kc),
                                                    out.ctypes.data_as(_DP)))
    del keep
    return DiagonalSpectrum(shape, out)


def pow_spectrum(lam: DiagonalSpectrum, T: int) -> DiagonalSpectrum:
    """proj/src/spectrum.cpp:47-83"""
    out = np.empty_like(lam.blocks)
    _lib.check(_lib.load().fsx_pow_spectrum(ctypes.byref(lam.shape._c()), lam.blocks.ctypes.data_as(_DP),
                                            _u64_T(T), out.ctypes.data_as(_DP)))
    return DiagonalSpectrum(lam.shape, out)


def pseudo_inverse_spectrum(lam: DiagonalSpectrum) -> DiagonalSpectrum:
    """proj/src/spectrum.cpp:85-96"""
    if lam.block_dim() != 1:
        raise SpecError("pseudo_inverse_spectrum: scalar spectra only")
    out = np.empty_like(lam.blocks)
    _lib.check(_lib.load().fsx_pseudo_inverse_spectrum(ctypes.byref(lam.shape._c()),
                                                       lam.blocks.ctypes.data_as(_DP), out.ctypes.data_as(_DP)))
    return DiagonalSpectrum(lam.shape, out)


def multiply_spectra(a: DiagonalSpectrum, b: DiagonalSpectrum) -> DiagonalSpectrum:
    """proj/src/spectrum.cpp:98-109"""
    if a.shape != b.shape:
        raise SpecError("multiply_spectra: shape mismatch")
    out = np.empty_like(a.blocks)
    _lib.check(_lib.load().fsx_multiply_spectra(ctypes.byref(a.shape._c()), a.blocks.ctypes.data_as(_DP),
                                                b.blocks.ctypes.data_as(_DP), out.ctypes.data_as(_DP)))
    return DiagonalSpectrum(a.shape, out)


def hadamard(lam: DiagonalSpectrum, x: ComplexGrid) -> ComplexGrid:
    """proj/src/spectrum.cpp:111-134"""
    if lam.shape != x.shape:
        raise SpecError("hadamard: shape mismatch")
    x = _cgrid(x)
    out = np.empty_like(x.data)
    _lib.check(_lib.load().fsx_hadamard(ctypes.byref(lam.shape._c()), lam.blocks.ctypes.data_as(_DP),
                                        x.data.ctypes.data_as(_DP), out.ctypes.data_as(_DP)))
    return ComplexGrid(x.shape, out)


def device_count() -> int:
    return int(_lib.load().fsx_device_count())
