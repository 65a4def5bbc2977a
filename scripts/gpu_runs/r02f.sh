# r02f: multi-GPU C-ABI tests (emulated ranks), C++ drop-in, TMA cluster micro-benchmark
set -x
mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_cpp_dropin.py -x -q -s > gpurun_out/r02f/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02f/pytest.txt
timeout 120 ./scripts/micro/tma_cluster > gpurun_out/r02f/tma_cluster.txt 2>&1
tail -30 gpurun_out/r02f/pytest.txt; cat gpurun_out/r02f/tma_cluster.txt
