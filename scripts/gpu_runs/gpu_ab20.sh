# smem group coefficients again (cfg4 regression check)
for cfg in cfg4 cfg2; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab20_${cfg}.log 2>&1
done
python scripts/summarize.py gpurun_out/ab20_cfg*.log
