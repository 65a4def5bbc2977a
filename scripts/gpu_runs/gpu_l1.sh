timeout 200 python bench.py --config cfg1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/l1_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l1_launch_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/l1_ncu.log 2>&1
timeout 200 python bench.py --config cfg5 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/l5_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l5_launch_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/l5_ncu.log 2>&1
python scripts/launches.py gpurun_out/l1_launch_cfg1.csv gpurun_out/l5_launch_cfg5.csv
