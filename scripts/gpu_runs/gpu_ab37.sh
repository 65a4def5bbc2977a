# row-pair: two interleaved 2x2 power chains
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_naive.py -m gpu -q -x -p no:cacheprovider -k "rowpair or cfg5 or plans or naive" > gpurun_out/pytest_ab37.log 2>&1; tail -2 gpurun_out/pytest_ab37.log
timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab37_cfg5.log 2>&1
timeout 300 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab37_cfg1.log 2>&1
python scripts/summarize.py gpurun_out/ab37_cfg*.log
