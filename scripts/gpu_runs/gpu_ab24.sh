timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "batch" > gpurun_out/pytest_ab24.log 2>&1; tail -3 gpurun_out/pytest_ab24.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab24_cfg2.log 2>&1; tail -c 900 gpurun_out/ab24_cfg2.log
