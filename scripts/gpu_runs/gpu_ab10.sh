# A/B: row passes cp.async staged (FSX_ROWS=1) vs bulk-copy staged (FSX_ROWS=3)
FSX_ROWS=3 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab10.log 2>&1; tail -3 gpurun_out/pytest_ab10.log
for cfg in cfg2 cfg3 cfg4; do
  for V in 1 3; do
    FSX_ROWS=$V timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab10_${cfg}_$V.log 2>&1
  done
done
for V in 1 3; do
  FSX_ROWS=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab10_launch$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab10_ncu$V.log 2>&1
done
python scripts/summarize.py gpurun_out/ab10_cfg*.log
python scripts/launches.py gpurun_out/ab10_launch*.csv
