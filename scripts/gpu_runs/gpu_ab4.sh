timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg or golden" > gpurun_out/pytest_ab4.log 2>&1; tail -2 gpurun_out/pytest_ab4.log
FSX_TMA_PERSIST=1 timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg or golden" > gpurun_out/pytest_ab4p.log 2>&1; tail -2 gpurun_out/pytest_ab4p.log
for P in 0 1; do
  FSX_TMA_PERSIST=$P timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab4_cfg2_p$P.log 2>&1
  FSX_TMA_PERSIST=$P timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab4_cfg4_p$P.log 2>&1
done
