# host enqueue overhead: cached ctypes views + one-time kernel attribute/occupancy setup
for cfg in cfg2 cfg1 cfg3; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab17_${cfg}.log 2>&1
done
python scripts/summarize.py gpurun_out/ab17_cfg*.log
grep -ho '"host_enqueue_us": [0-9.]*' gpurun_out/ab17_cfg*.log
