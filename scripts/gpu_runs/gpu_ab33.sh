# rows: one stage x 4 CTAs/SM (128 regs) vs two stages x 3 CTAs/SM
for V in 1 2; do
  FSX_ROW_STAGES=$V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab33_launch_$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab33_ncu.log 2>&1
  FSX_ROW_STAGES=$V timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab33_cfg2_$V.log 2>&1
done
python scripts/summarize.py gpurun_out/ab33_cfg2_*.log
python scripts/launches.py gpurun_out/ab33_launch_*.csv
