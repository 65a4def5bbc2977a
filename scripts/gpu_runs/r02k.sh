# r02k: slab-level batch (fsx_solve_periodic_slabs) tests + the plan/batch/cache suites it touches
set -x
mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_slabs.py -x -q -s > gpurun_out/r02k/pytest_slabs.txt 2>&1; echo "rc=$?" >> gpurun_out/r02k/pytest_slabs.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_multi.py -x -q > gpurun_out/r02k/pytest_rest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02k/pytest_rest.txt
tail -25 gpurun_out/r02k/pytest_slabs.txt; tail -3 gpurun_out/r02k/pytest_rest.txt
