"""ctypes binding of libfsx.so (C ABI: include/fsx.h).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
and is REQUIRED: importing the solver API without it raises, there is no
Python or CPU fallback for the numerical path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSX_LIB") or os.path.join(HERE, "libfsx.so")  # FSX_LIB: A/B builds

FSX_OK, FSX_ERR_SPEC, FSX_ERR_NUMERIC, FSX_ERR_CUDA, FSX_ERR_NCCL, FSX_ERR_OOM, FSX_ERR_IO = 0, 1, 2, 3, 4, 5, 6
FSX_GRID_CSV, FSX_GRID_RAW = 0, 1
FSX_EXCHANGE_AUTO, FSX_EXCHANGE_P2P, FSX_EXCHANGE_NCCL = 0, 1, 2
FSX_DECOMP_AUTO, FSX_DECOMP_SLAB, FSX_DECOMP_PENCIL = 0, 1, 2
MAX_RANK = 8
ABI_VERSION = 200  # include/fsx.h FSX_ABI_VERSION: the struct layouts below


class Error(RuntimeError):
    """Base class (proj/include/fftstencil/errors.hpp:9-13)."""


class SpecError(Error, ValueError):
    """Invalid arguments / shapes / kernels (errors.hpp:15-19)."""


class NumericError(Error, ArithmeticError):
    """Non-finite result or residue blow-up (errors.hpp:27-31)."""


class CudaError(Error):
    """CUDA failure (no device, launch error, out of memory)."""


class IoError(Error, OSError):
    """File parsing / reading / writing problems (errors.hpp:20-24)."""


class FsxShape(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("fields", ctypes.c_int32), ("dims", ctypes.c_int64 * MAX_RANK)]


class FsxKernel(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("fields", ctypes.c_int32),
        ("ntaps", ctypes.c_int64),
        ("offsets", ctypes.POINTER(ctypes.c_int64)),
        ("blocks", ctypes.POINTER(ctypes.c_double)),
    ]


class FsxStageTimings(ctypes.Structure):
    _fields_ = [
        ("forward_fft", ctypes.c_double),
        ("squaring", ctypes.c_double),
        ("hadamard", ctypes.c_double),
        ("inverse_fft", ctypes.c_double),
        ("boundary_recursion", ctypes.c_double),
    ]


class FsxOptions(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32),
        ("path", ctypes.c_int32),
        ("stage_events", ctypes.c_int32),
        ("spectral_cut", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("num_gpus", ctypes.c_int32),
        ("exchange", ctypes.c_int32),
        ("devices", ctypes.POINTER(ctypes.c_int32)),
        ("decomp", ctypes.c_int32),
        ("pencil_rows", ctypes.c_int32),
    ]


class FsxPlanInfo(ctypes.Structure):
    _fields_ = [
        ("path", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("alg_bytes", ctypes.c_int64),
        ("fused_bytes", ctypes.c_int64),
        ("work_bytes", ctypes.c_int64),
        ("sched_bytes", ctypes.c_int64),
        ("ranks", ctypes.c_int32),
        ("exchange", ctypes.c_int32),
        ("decomp", ctypes.c_int32),
        ("pencil_rows", ctypes.c_int32),
    ]


# Every symbol include/fsx.h declares (tests check the library exports them).
EXPORTS = (
    "fsx_solve_periodic",
    "fsx_solve_periodic_vector",
    "fsx_spectrum_cache_create",
    "fsx_spectrum_cache_destroy",
    "fsx_solve_periodic_cached",
    "fsx_solve_periodic_implicit",
    "fsx_solve_periodic_device",
    "fsx_solve_periodic_batch",
    "fsx_solve_periodic_slabs",
    "fsx_solve_periodic_f32",
    "fsx_solve_periodic_device_f32",
    "fsx_solve_periodic_batch_f32",
    "fsx_device_check",
    "fsx_last_stage_ms",
    "fsx_step_periodic",
    "fsx_evolve_periodic_naive",
    "fsx_evolve_periodic_naive_device",
    "fsx_slab_describe",
    "fsx_slab_forward",
    "fsx_slab_spectral",
    "fsx_slab_inverse",
    "fsx_slab_forward_p2p",
    "fsx_slab_inverse_p2p",
    "fsx_multi_fft",
    "fsx_spectrum_from_kernel",
    "fsx_pow_spectrum",
    "fsx_pseudo_inverse_spectrum",
    "fsx_multiply_spectra",
    "fsx_hadamard",
    "fsx_last_error",
    "fsx_version",
    "fsx_device_count",
    "fsx_set_devices",
    "fsx_get_devices",
    "fsx_plan_describe",
    "fsx_spectral_cut_columns",
    "fsx_write_grid",
    "fsx_read_grid_shape",
    "fsx_read_grid",
    "fsx_load_grid_device",
    "fsx_format_stage_table",
)

_lib = None


def load():
    """Loads libfsx.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "the StencilFFT-P solver has no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    L.fsx_last_error.restype = ctypes.c_char_p
    L.fsx_version.restype = ctypes.c_int32
    L.fsx_device_count.restype = ctypes.c_int32
    L.fsx_get_devices.restype = ctypes.c_int32
    if L.fsx_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {L.fsx_version()}, this binding expects {ABI_VERSION} "
                          "(rebuild with `make`)")
    L.fsx_spectrum_cache_create.restype = ctypes.c_void_p
    L.fsx_spectrum_cache_destroy.argtypes = [ctypes.c_void_p]
    _lib = L
    return L


def check(status: int) -> None:
    if status == FSX_OK:
        return
    msg = load().fsx_last_error().decode(errors="replace")
    if status == FSX_ERR_SPEC:
        raise SpecError(msg)
    if status == FSX_ERR_NUMERIC:
        raise NumericError(msg)
    if status == FSX_ERR_IO:
        raise IoError(msg)
    raise CudaError(f"[fsx status {status}] {msg}")
