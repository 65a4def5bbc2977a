timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab3.log 2>&1; tail -2 gpurun_out/pytest_ab3.log
for T in 1 0; do
  FSX_TMA=$T timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3_cfg2_tma$T.log 2>&1
  FSX_TMA=$T timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3_cfg3_tma$T.log 2>&1
  FSX_TMA=$T timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab3_cfg4_tma$T.log 2>&1
done
timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab3_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab3_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab3_ncu.log 2>&1
