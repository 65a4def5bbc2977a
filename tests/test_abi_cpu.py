"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/fsx.h declares, and host-side validation maps the
reference's SpecError cases (proj/src/kernel.cpp:7-49, grid.hpp:21-45)
without touching a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2105_06676_b200 as fs
from paper_2105_06676_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "fsx.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(fsx_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.fsx_version() == 200


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_spec_errors_host_side():
    k = fs.StencilKernel(1)
    k.add_tap([5], 1.0)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic(fs.FieldGrid(fs.GridShape([4])), k, 1)
    k2 = fs.StencilKernel(2)
    k2.add_tap([0, 0], 1.0)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic(fs.FieldGrid(fs.GridShape([4])), k2, 1)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic(fs.FieldGrid(fs.GridShape([4])), fs.StencilKernel(1), 1)
    with pytest.raises(fs.SpecError):
        fs.StencilKernel(1).add_tap([0], float("nan"))
    with pytest.raises(fs.SpecError):
        fs.StencilKernel(1, 2).add_tap([0], 1.0)
    with pytest.raises(fs.SpecError):
        fs.GridShape([0])
    with pytest.raises(fs.SpecError):
        fs.GridShape([1 << 40, 1 << 40])
    kk = fs.StencilKernel(1)
    kk.add_tap([0], 1.0)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_vector(fs.FieldGrid(fs.GridShape([8])), kk, 1)
    with pytest.raises(fs.SpecError):
        fs.solve_periodic_implicit(fs.StencilKernel(1, 2).add_tap([0], np.eye(2)), kk,
                                   fs.FieldGrid(fs.GridShape([8], 2)), 1)


def test_c_abi_direct_validation():
    """The raw C ABI (what a C/C++ caller binds) reports FSX_ERR_SPEC codes."""
    L = _lib.load()
    shape = _lib.FsxShape()
    shape.rank, shape.fields, shape.dims[0] = 1, 1, 4
    off = np.array([[7]], np.int64)
    blk = np.array([1.0])
    k = _lib.FsxKernel(1, 1, 1, off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                       blk.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    a = np.zeros(4)
    out = np.zeros(4)
    st = L.fsx_solve_periodic(ctypes.byref(shape), a.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k),
                              ctypes.c_uint64(1), out.ctypes.data_as(ctypes.c_void_p), None, None)
    assert st == _lib.FSX_ERR_SPEC
    assert b"exceeds dimension" in L.fsx_last_error()
    shape.rank = 0
    st = L.fsx_solve_periodic(ctypes.byref(shape), a.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k),
                              ctypes.c_uint64(1), out.ctypes.data_as(ctypes.c_void_p), None, None)
    assert st == _lib.FSX_ERR_SPEC


def test_T0_copies_without_device():
    """T == 0 returns the input bit-exactly (proj/src/periodic.cpp:79)."""
    k = fs.StencilKernel(2)
    k.add_tap([1, -1], 0.5)
    a = np.random.default_rng(0).uniform(-1, 1, 64)
    out = fs.solve_periodic(fs.FieldGrid(fs.GridShape([8, 8]), a), k, 0)
    assert (out.data == a).all()


def test_fold_kernels_and_value_types():
    k0 = fs.StencilKernel(1)
    k0.add_tap([-1], 0.1).add_tap([1], 0.2).add_tap([1], 0.3)
    assert k0.taps()[(1,)][0, 0] == pytest.approx(0.5)
    assert k0.radius() == 1 and k0.max_reach() == [1]
    e = fs.StencilKernel(1)
    f = fs.fold_kernels([[k0, e], [e, k0]])
    assert f.fields() == 2 and f.taps()[(1,)][1, 1] == pytest.approx(0.5)
    with pytest.raises(fs.SpecError):
        fs.fold_kernels([[e]])
    lam = fs.DiagonalSpectrum(fs.GridShape([3], 2))
    lam.set_block(1, [[1, 2], [3, 4]])
    assert lam.entry(1, 1, 0) == 3


def test_T_out_of_range_is_spec_error_on_every_wrapper():
    """T is the reference's uint64_t (periodic.hpp:43): a negative or >= 2^64 T
    raises SpecError in every wrapper, before any device work (no wrap-around)."""
    k = fs.StencilKernel(1).add_tap([0], 0.5).add_tap([1], 0.5)
    sh = fs.GridShape([16])
    g = fs.FieldGrid(sh, np.zeros(16))
    for bad in (-1, 1 << 64):
        with pytest.raises(fs.SpecError):
            fs.solve_periodic_cached(g, k, bad, fs.SpectrumCache())
        with pytest.raises(fs.SpecError):
            fs.solve_periodic_implicit(k, k, g, bad)
        with pytest.raises(fs.SpecError):
            fs.solve_periodic_device(sh, 0, k, bad, 0)
        with pytest.raises(fs.SpecError):
            fs.evolve_periodic_naive_device(sh, 0, k, bad, 0)
        with pytest.raises(fs.SpecError):
            fs.spectral_cut_columns(sh, k, bad)
