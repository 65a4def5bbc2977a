timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg2 or golden or cfg3" > gpurun_out/pytest_ab2.log 2>&1; tail -2 gpurun_out/pytest_ab2.log
for V in 0 1 2; do
  FSX_PIPE=0 FSX_FUSED_VARIANT=$V timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab2_cfg2_v$V.log 2>&1
done
FSX_PIPE=1 timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab2_cfg2_pipe.log 2>&1
FSX_PIPE=0 timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab2_cfg3_nopipe.log 2>&1
FSX_PIPE=0 timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab2_cfg4_nopipe.log 2>&1
FSX_PIPE=1 timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab2_cfg4_pipe.log 2>&1
