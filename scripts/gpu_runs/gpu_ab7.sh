FSX_TMA_PERSIST=1 timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg or slab" > gpurun_out/pytest_ab7.log 2>&1; tail -2 gpurun_out/pytest_ab7.log
for P in 1 0; do
  FSX_TMA_PERSIST=$P timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab7_cfg2_p$P.log 2>&1
  FSX_TMA_PERSIST=$P timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab7_cfg4_p$P.log 2>&1
done
FSX_TMA_PERSIST=1 timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab7_plain.log 2>&1 && FSX_TMA_PERSIST=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab7_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab7_ncu.log 2>&1
