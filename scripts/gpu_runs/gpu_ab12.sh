# full pass-twiddle tables in the column FFTs; W_32 split constants in c2r
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab12.log 2>&1; tail -3 gpurun_out/pytest_ab12.log
for cfg in cfg2 cfg3 cfg4 cfg1 cfg5; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab12_${cfg}.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab12_launch.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab12_ncu.log 2>&1
python scripts/summarize.py gpurun_out/ab12_cfg*.log
python scripts/launches.py gpurun_out/ab12_launch.csv
