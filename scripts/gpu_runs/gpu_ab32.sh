timeout 1000 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab32.log 2>&1; tail -2 gpurun_out/pytest_ab32.log
for i in 1 2; do timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab32_cfg2_$i.log 2>&1; done
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab32_cfg4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab32_launch.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab32_ncu.log 2>&1
python scripts/summarize.py gpurun_out/ab32_cfg*.log
python scripts/launches.py gpurun_out/ab32_launch.csv
