# one-stage 2-CTA/SM rows for M = 4096 (cfg3) vs two-stage 1 CTA/SM
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab22.log 2>&1; tail -2 gpurun_out/pytest_ab22.log
for V in 1 2; do
  FSX_ROW_STAGES=$V timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab22_cfg3_$V.log 2>&1
  FSX_ROW_STAGES=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab22_launch3_$V.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab22_ncu3.log 2>&1
done
python scripts/summarize.py gpurun_out/ab22_cfg*.log
python scripts/launches.py gpurun_out/ab22_launch3_*.csv
