# halves: symbol from 8 reads per group + quarter turns
timeout 1000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab30.log 2>&1; tail -2 gpurun_out/pytest_ab30.log
for V in 1 0; do
  FSX_HALVES=$V timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab30_cfg3_$V.log 2>&1
done
python scripts/summarize.py gpurun_out/ab30_cfg3_*.log
