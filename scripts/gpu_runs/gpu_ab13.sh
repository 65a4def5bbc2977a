# cfg4 launch list with full tables only for N < 4096 column tiles
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab13_cfg4.log 2>&1
timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab13_cfg2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab13_launch_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab13_ncu.log 2>&1
python scripts/summarize.py gpurun_out/ab13_cfg*.log
python scripts/launches.py gpurun_out/ab13_launch_cfg4.csv
