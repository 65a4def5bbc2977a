# 8192 halves: one CTA (1) vs two-CTA cluster (2) vs plain (0)
FSX_HALVES=2 timeout 1000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_naive.py -m gpu -q -x -p no:cacheprovider -k "8192 or plans or cfg3 or slab" > gpurun_out/pytest_ab31.log 2>&1; tail -2 gpurun_out/pytest_ab31.log
for V in 2 1 0; do
  FSX_HALVES=$V timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab31_cfg3_$V.log 2>&1
done
python scripts/summarize.py gpurun_out/ab31_cfg3_*.log
