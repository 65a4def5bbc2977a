# r03e: run-to-run determinism of the cross-CTA / cross-stream kernels; C++ drop-in with the slab wrapper
set -x
D=gpurun_out/r03e
mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_determinism.py tests/test_cpp_dropin.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -4 $D/pytest.txt
