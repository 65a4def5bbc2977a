for V in 128 512; do
  FSX_TMA_AXIS=$V timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab39_cfg5_$V.log 2>&1
done
python scripts/summarize.py gpurun_out/ab39_*.log
