"""Grid I/O and the bench-mode stage table.

Python mirror of the reference's grid_io / runner interface over the C ABI
(include/fsx.h, csrc/fsx_io.cpp):

  * ``write_grid(g, path, "raw" | "csv")`` / ``read_grid(path)``
    (proj/include/fftstencil/grid_io.hpp:10-18; raw = little-endian float64 +
    "<path>.meta" sidecar, csv = "i1,...,id,f,value" shortest round-trip);
    malformed input raises :class:`IoError` naming the line or byte count.
  * ``load_grid_device(path, d_ptr)`` reads a raw grid straight into device
    memory (chunked pinned staging, each chunk's H2D overlapping the next
    read) -- the GPU solve's input without a full host copy.
  * ``run_bench(a0, k, T)`` is run_bench (proj/src/runner.cpp:96-115): one
    timed solve with StageTimings, its stage table, optionally the naive
    solver's time.
"""
from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from ._lib import IoError  # noqa: F401
from .fftstencil import FieldGrid, GridShape, StageTimings, StencilKernel, evolve_periodic_naive, solve_periodic

_DP = ctypes.POINTER(ctypes.c_double)
_FORMATS = {"csv": _lib.FSX_GRID_CSV, "raw": _lib.FSX_GRID_RAW}


def _shape_from_c(c: _lib.FsxShape) -> GridShape:
    return GridShape([c.dims[a] for a in range(c.rank)], c.fields)


def write_grid(g: FieldGrid, path: str, fmt: str = "raw") -> None:
    """grid_io.hpp:14 write_grid (GridFormat::Raw / GridFormat::Csv)."""
    if fmt not in _FORMATS:
        raise _lib.SpecError(f"write_grid: unknown format '{fmt}'")
    data = np.ascontiguousarray(g.data, dtype=np.float64)
    _lib.check(_lib.load().fsx_write_grid(ctypes.byref(g.shape._c()), data.ctypes.data_as(_DP),
                                          str(path).encode(), ctypes.c_int32(_FORMATS[fmt])))


def read_grid_shape(path: str) -> GridShape:
    c = _lib.FsxShape()
    _lib.check(_lib.load().fsx_read_grid_shape(str(path).encode(), ctypes.byref(c)))
    return _shape_from_c(c)


def read_grid(path: str) -> FieldGrid:
    """grid_io.hpp:18 read_grid: raw when "<path>.meta" exists, else csv."""
    shape = read_grid_shape(path)
    out = np.empty(shape.cells() * shape.fields(), dtype=np.float64)
    _lib.check(_lib.load().fsx_read_grid(str(path).encode(), ctypes.byref(shape._c()), out.ctypes.data_as(_DP)))
    return FieldGrid(shape, out)


def load_grid_device(path: str, d_out: int, shape: GridShape | None = None, device: int = 0,
                     stream: int | None = None) -> GridShape:
    """A raw grid straight into device memory at ``d_out`` (prod(dims) * fields
    doubles); returns its shape.  ``shape`` (optional) must match the file."""
    shape = shape or read_grid_shape(path)
    o = _lib.FsxOptions()
    o.device = int(device)
    o.stream = stream
    _lib.check(_lib.load().fsx_load_grid_device(str(path).encode(), ctypes.byref(shape._c()), ctypes.c_void_p(d_out),
                                                ctypes.byref(o)))
    return shape


def format_stage_table(st: StageTimings, total: float, naive_seconds: float = -1.0) -> str:
    """runner.cpp:46-62 print_stage_table."""
    buf = ctypes.create_string_buffer(1024)
    _lib.check(_lib.load().fsx_format_stage_table(ctypes.byref(st._push()), ctypes.c_double(total),
                                                  ctypes.c_double(naive_seconds), buf, ctypes.c_int64(len(buf))))
    return buf.value.decode()


def run_bench(a0: FieldGrid, k: StencilKernel, T: int, naive: bool = False) -> tuple:
    """runner.cpp:96-115 run_bench for the periodic path: one FFT solve timed
    with a steady clock and its StageTimings (the stages cover the whole call:
    host set-up is attributed to forward_fft, the final check and copy-out to
    inverse_fft), plus, with ``naive``, the direct-stepping solver's time.
    Returns (table text, StageTimings, total seconds, naive seconds or -1)."""
    st = StageTimings()
    t0 = time.perf_counter()
    solve_periodic(a0, k, T, st)
    total = time.perf_counter() - t0
    naive_s = -1.0
    if naive:
        t0 = time.perf_counter()
        evolve_periodic_naive(a0, k, T)
        naive_s = time.perf_counter() - t0
    return format_stage_table(st, total, naive_s), st, total, naive_s
