# cfg3 regression hunt: scalar pow back in spectral_regs
for cfg in cfg3 cfg2 cfg4; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab16_${cfg}.log 2>&1
done
python scripts/summarize.py gpurun_out/ab16_cfg*.log
