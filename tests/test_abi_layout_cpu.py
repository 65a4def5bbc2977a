"""The ctypes mirror (paper_2105_06676_b200/_lib.py) of every struct in
include/fsx.h has the C layout: size and field offsets compared against a C
program compiled from the header (a mismatch would silently misread options
such as the multi-GPU device list)."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

STRUCTS = {
    "fsx_shape": ("FsxShape", ["rank", "fields", "dims"]),
    "fsx_kernel": ("FsxKernel", ["rank", "fields", "ntaps", "offsets", "blocks"]),
    "fsx_stage_timings": ("FsxStageTimings", ["forward_fft", "squaring", "hadamard", "inverse_fft",
                                              "boundary_recursion"]),
    "fsx_options": ("FsxOptions", ["device", "path", "stage_events", "spectral_cut", "stream", "num_gpus",
                                   "exchange", "devices", "decomp", "pencil_rows"]),
    "fsx_plan_info": ("FsxPlanInfo", ["path", "launches", "alg_bytes", "fused_bytes", "work_bytes", "sched_bytes",
                                      "ranks", "exchange", "decomp", "pencil_rows"]),
    "fsx_slab_info": ("distributed.FsxSlabInfo", ["nranks", "rank", "local_dims", "plane_offset", "col_block",
                                                  "xbuf_bytes"]),
}


@pytest.fixture(scope="module")
def c_layout(tmp_path_factory):
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "fsx.h"', "int main(void) {"]
    for cname, (_, fields) in STRUCTS.items():
        src.append(f'    printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in fields:
            src.append(f'    printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src += ["    return 0;", "}"]
    d = tmp_path_factory.mktemp("abi")
    c = d / "layout.c"
    c.write_text("\n".join(src) + "\n")
    exe = d / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    layout = {}
    for line in out.splitlines():
        name, field, val = line.split()
        layout[(name, field)] = int(val)
    return layout


@pytest.mark.parametrize("cname", sorted(STRUCTS))
def test_ctypes_mirror_matches_header(c_layout, cname):
    import importlib

    pyname, fields = STRUCTS[cname]
    mod, _, attr = pyname.rpartition(".")
    cls = getattr(importlib.import_module("paper_2105_06676_b200." + (mod or "_lib")), attr)
    assert ctypes.sizeof(cls) == c_layout[(cname, "size")], cname
    assert [f[0] for f in cls._fields_] == fields, cname
    for f in fields:
        assert getattr(cls, f).offset == c_layout[(cname, f)], (cname, f)
