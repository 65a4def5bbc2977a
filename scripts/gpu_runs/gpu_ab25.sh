# no underflow test in the vectorized power
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab25.log 2>&1; tail -2 gpurun_out/pytest_ab25.log
for cfg in cfg2 cfg3 cfg4 cfg1 cfg5; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab25_${cfg}.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab25_launch2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab25_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab25_launch3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab25_ncu3.log 2>&1
python scripts/summarize.py gpurun_out/ab25_cfg*.log
python scripts/launches.py gpurun_out/ab25_launch2.csv gpurun_out/ab25_launch3.csv
