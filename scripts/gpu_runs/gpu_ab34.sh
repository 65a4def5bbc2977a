# TMA strided C2C passes with four-step twiddles (1D plan columns)
timeout 1000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab34.log 2>&1; tail -2 gpurun_out/pytest_ab34.log
for cfg in cfg5 cfg1 cfg2 cfg4; do
  for V in 1 0; do
    FSX_TMA_AXIS=$V timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab34_${cfg}_$V.log 2>&1
  done
done
python scripts/summarize.py gpurun_out/ab34_cfg*.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab34_launch5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab34_ncu.log 2>&1
python scripts/launches.py gpurun_out/ab34_launch5.csv
