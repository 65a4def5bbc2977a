"""Binding of ``oracle/_ref/libfftstencil_ref.so`` -- TEST INFRASTRUCTURE.

That library is the reference's OWN periodic-path sources (fft, spectrum,
periodic, parallel, grid, kernel, oracle, band ``.cpp`` under
``/root/reference/proj/src``), compiled unmodified by ``oracle/Makefile``
(target ``ref``) against ``oracle/eigen_shim`` -- a stand-in for the Eigen3
dependency this image lacks -- plus ``oracle/ref_capi.cpp``, which exports the
same C entry points as the restated oracle.  ``module()`` therefore returns a
second instance of ``oracle/oracle.py`` bound to that library: every wrapper
(``solve_periodic``, ``multi_fft``, ``pow_spectrum`` ...) then runs reference
code.  Functions that exist only in the restatement (``solve_periodic_ld``,
``modal_problem_periodic``, ``splitmix_fill``) are not available on it.

Used by ``tests/test_oracle_vs_ref_cpu.py`` (the restatement against the
reference itself) and by ``bench.py``'s CPU legs (``cpu_baseline.kind =
"reference"``).  ``/root/reference`` is needed only to BUILD the library (in
the development container); the built file travels to the GPU box.
"""
from __future__ import annotations

import importlib.util
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libfftstencil_ref.so")
REF_ROOT = "/root/reference/proj"

_mod = None


def build() -> bool:
    """Builds the library when the reference tree is present; True if the library exists afterwards."""
    if os.path.isdir(os.path.join(REF_ROOT, "src")):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return os.path.exists(REF_LIB)


def available() -> bool:
    return os.path.exists(REF_LIB)


def module():
    """oracle.py bound to the reference library (raises FileNotFoundError if it was not built)."""
    global _mod
    if _mod is None:
        if not available():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref, needs {REF_ROOT})")
        spec = importlib.util.spec_from_file_location("oracle._ref_binding", os.path.join(HERE, "oracle.py"))
        m = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(m)
        m.LIB_PATH = REF_LIB
        m.build = lambda force=False: REF_LIB
        assert m.lib().orc_is_reference() == 1
        _mod = m
    return _mod
