"""ORACLE binding — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes wrapper over ``oracle/liborc.so``, the CPU restatement of the
reference StencilFFT-P path (see the header of ``fftstencil_oracle.cpp`` for
the reference file:line each function follows).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
/ ``--impl reference`` leg may import this module.  The product package
(``paper_2105_06676_b200``) never imports it.

Kernels are passed as ``(offsets, blocks)``: ``offsets`` int64 ``[ntaps, rank]``
and ``blocks`` float64 ``[ntaps, m, m]`` (row-major), the same arrays the
product C-ABI takes.  Grids are float64 arrays of ``prod(dims) * m`` values,
row-major over the dims with the field innermost (proj/include/fftstencil/grid.hpp:17-20).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")


class OracleSpecError(ValueError):
    """Reference SpecError raised by the oracle."""


class OracleNumericError(ArithmeticError):
    """Reference NumericError raised by the oracle."""


_lib = None
_P = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_thread_count.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().orc_last_error().decode()
    if status == 1:
        raise OracleSpecError(msg)
    if status == 2:
        raise OracleNumericError(msg)
    raise RuntimeError(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I64P)


def _dims(dims) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64).reshape(-1))


def _taps(offsets, blocks, rank, m):
    off = np.asarray(offsets, dtype=np.int64)
    blk = np.asarray(blocks, dtype=np.float64)
    if off.ndim == 2 and off.shape[0] > 0 and off.shape[1] != rank:
        raise OracleSpecError("StencilKernel: grid rank mismatch")
    off = np.ascontiguousarray(off.reshape(-1, rank))
    if blk.size != off.shape[0] * m * m:
        raise OracleSpecError("StencilKernel: grid field count mismatch")
    blk = np.ascontiguousarray(blk.reshape(-1, m, m))
    return off, blk


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def thread_count() -> int:
    return int(lib().orc_thread_count())


def solve_periodic(a0, dims, fields, offsets, blocks, T, timings=None, vector=False):
    d = _dims(dims)
    a = np.ascontiguousarray(np.asarray(a0, dtype=np.float64).reshape(-1))
    off, blk = _taps(offsets, blocks, d.size, fields)
    out = np.empty_like(a)
    st = np.zeros(5) if timings is None else timings
    fn = lib().orc_solve_periodic_vector if vector else lib().orc_solve_periodic
    _check(fn(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields), _dp(a), ctypes.c_int64(off.shape[0]),
              _ip(off), _dp(blk), ctypes.c_uint64(int(T)), _dp(out), _dp(st)))
    return out


def solve_periodic_ld(a0, dims, fields, offsets, blocks, T):
    """Same algorithm in x87 long double (64-bit mantissa): config-5 truth."""
    d = _dims(dims)
    a = np.ascontiguousarray(np.asarray(a0, dtype=np.float64).reshape(-1))
    off, blk = _taps(offsets, blocks, d.size, fields)
    out = np.empty_like(a)
    _check(lib().orc_solve_periodic_ld(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields), _dp(a),
                                       ctypes.c_int64(off.shape[0]), _ip(off), _dp(blk),
                                       ctypes.c_uint64(int(T)), _dp(out)))
    return out


def solve_periodic_implicit(a0, dims, q, s, T, timings=None):
    d = _dims(dims)
    a = np.ascontiguousarray(np.asarray(a0, dtype=np.float64).reshape(-1))
    qo, qb = _taps(q[0], q[1], d.size, 1)
    so, sb = _taps(s[0], s[1], d.size, 1)
    out = np.empty_like(a)
    st = np.zeros(5) if timings is None else timings
    _check(lib().orc_solve_periodic_implicit(ctypes.c_int(d.size), _ip(d), _dp(a),
                                             ctypes.c_int64(qo.shape[0]), _ip(qo), _dp(qb),
                                             ctypes.c_int64(so.shape[0]), _ip(so), _dp(sb),
                                             ctypes.c_uint64(int(T)), _dp(out), _dp(st)))
    return out


def multi_fft(x, dims, fields=1, inverse=False):
    d = _dims(dims)
    xc = np.ascontiguousarray(np.asarray(x, dtype=np.complex128).reshape(-1))
    out = np.empty_like(xc)
    _check(lib().orc_multi_fft(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields),
                               xc.ctypes.data_as(_DP), out.ctypes.data_as(_DP), ctypes.c_int(int(inverse))))
    return out


def spectrum_from_kernel(dims, fields, offsets, blocks):
    d = _dims(dims)
    off, blk = _taps(offsets, blocks, d.size, fields)
    n = int(np.prod(d)) * fields * fields
    out = np.empty(n, dtype=np.complex128)
    _check(lib().orc_spectrum_from_kernel(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields),
                                          ctypes.c_int64(off.shape[0]), _ip(off), _dp(blk),
                                          out.ctypes.data_as(_DP)))
    return out


def pow_spectrum(blocks, dims, m, T):
    d = _dims(dims)
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.complex128).reshape(-1))
    out = np.empty_like(b)
    _check(lib().orc_pow_spectrum(ctypes.c_int(d.size), _ip(d), ctypes.c_int(m), b.ctypes.data_as(_DP),
                                  ctypes.c_uint64(int(T)), out.ctypes.data_as(_DP)))
    return out


def pseudo_inverse_spectrum(blocks, dims, m=1):
    d = _dims(dims)
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.complex128).reshape(-1))
    out = np.empty_like(b)
    _check(lib().orc_pseudo_inverse_spectrum(ctypes.c_int(d.size), _ip(d), ctypes.c_int(m),
                                             b.ctypes.data_as(_DP), out.ctypes.data_as(_DP)))
    return out


def multiply_spectra(a, b, dims, m):
    d = _dims(dims)
    A = np.ascontiguousarray(np.asarray(a, dtype=np.complex128).reshape(-1))
    B = np.ascontiguousarray(np.asarray(b, dtype=np.complex128).reshape(-1))
    out = np.empty_like(A)
    _check(lib().orc_multiply_spectra(ctypes.c_int(d.size), _ip(d), ctypes.c_int(m), A.ctypes.data_as(_DP),
                                      B.ctypes.data_as(_DP), out.ctypes.data_as(_DP)))
    return out


def hadamard(lam, x, dims, m):
    d = _dims(dims)
    L = np.ascontiguousarray(np.asarray(lam, dtype=np.complex128).reshape(-1))
    X = np.ascontiguousarray(np.asarray(x, dtype=np.complex128).reshape(-1))
    out = np.empty_like(X)
    _check(lib().orc_hadamard(ctypes.c_int(d.size), _ip(d), ctypes.c_int(m), L.ctypes.data_as(_DP),
                              X.ctypes.data_as(_DP), out.ctypes.data_as(_DP)))
    return out


def step_periodic(a, dims, fields, offsets, blocks):
    d = _dims(dims)
    x = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
    off, blk = _taps(offsets, blocks, d.size, fields)
    out = np.empty_like(x)
    _check(lib().orc_step_periodic(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields), _dp(x),
                                   ctypes.c_int64(off.shape[0]), _ip(off), _dp(blk), _dp(out)))
    return out


def evolve_periodic_naive(a0, dims, fields, offsets, blocks, T):
    d = _dims(dims)
    x = np.ascontiguousarray(np.asarray(a0, dtype=np.float64).reshape(-1))
    off, blk = _taps(offsets, blocks, d.size, fields)
    out = np.empty_like(x)
    _check(lib().orc_evolve_periodic_naive(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields), _dp(x),
                                           ctypes.c_int64(off.shape[0]), _ip(off), _dp(blk),
                                           ctypes.c_uint64(int(T)), _dp(out)))
    return out


def dense_stencil_matrix(dims, fields, offsets, blocks):
    d = _dims(dims)
    off, blk = _taps(offsets, blocks, d.size, fields)
    n = int(np.prod(d)) * fields
    mat = np.empty((n, n))
    _check(lib().orc_dense_stencil_matrix(ctypes.c_int(d.size), _ip(d), ctypes.c_int(fields),
                                          ctypes.c_int64(off.shape[0]), _ip(off), _dp(blk), _dp(mat)))
    return mat


def splitmix_fill(seed: int, n: int, symmetric: bool) -> np.ndarray:
    out = np.empty(int(n))
    lib().orc_splitmix_fill(ctypes.c_uint64(int(seed)), ctypes.c_int64(int(n)), ctypes.c_int(int(symmetric)),
                            _dp(out))
    return out


def modal_problem_periodic(dims, offsets, blocks, T):
    """proj/src/modal.cpp:99-145: (initial grid, exact reference after T steps)
    with the mode amplification lambda^T in double-double arithmetic."""
    d = _dims(dims)
    off, blk = _taps(offsets, blocks, d.size, 1)
    n = int(np.prod(d))
    init = np.empty(n)
    ref = np.empty(n)
    _check(lib().orc_modal_problem_periodic(ctypes.c_int(d.size), _ip(d), ctypes.c_int64(off.shape[0]), _ip(off),
                                            _dp(blk), ctypes.c_uint64(int(T)), _dp(init), _dp(ref)))
    return init, ref
