# r02u: Pr x Pc pencils in the single-process multi-GPU path (emulated ranks) + parity suites touched by c_off_x
set -x
D=gpurun_out/r02u
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -s > $D/pytest_multi.txt 2>&1; echo "rc=$?" >> $D/pytest_multi.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_cut.py tests/test_gpu_f32.py tests/test_cpp_dropin.py -x -q > $D/pytest_rest.txt 2>&1; echo "rc=$?" >> $D/pytest_rest.txt
grep -E "pencils|passed|failed|rc=|Error" $D/pytest_multi.txt | head -30; tail -3 $D/pytest_rest.txt
