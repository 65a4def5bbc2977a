timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg2 or cfg3 or golden or slab" > gpurun_out/pytest_ab5.log 2>&1; tail -2 gpurun_out/pytest_ab5.log
for V in 1 0; do
  FSX_4STEP=$V timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab5_cfg2_4s$V.log 2>&1
done
timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab5_plain.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab5_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab5_ncu.log 2>&1
