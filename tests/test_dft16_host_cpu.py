"""Host-side check of the device butterflies of csrc/fsx_device.cuh: the
radix-16 pass with folded twiddles (dft16_tw_fused, selectable with
-DFSX_FUSED16=1) and the default path (twiddle products + Dft<16>) against a
long-double direct sum, fp64 and fp32, both transform directions.  The header
is compiled by plain g++ (tests/cpp/dft16_fused_host_test.cpp stubs the few
device intrinsics it names)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dft16_butterflies_on_host(tmp_path):
    exe = tmp_path / "dft16_test"
    subprocess.run(
        ["g++", "-std=c++17", "-O1", "-ffp-contract=off", "-I/usr/local/cuda/include",
         "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "paper_2105_06676_b200", "csrc"),
         os.path.join(ROOT, "tests", "cpp", "dft16_fused_host_test.cpp"), "-o", str(exe)],
        check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "OK" in out.stdout
