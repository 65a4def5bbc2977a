# PDL between the plan-1 passes
for cfg in cfg2 cfg1 cfg3; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab18_${cfg}.log 2>&1
done
python scripts/summarize.py gpurun_out/ab18_cfg*.log
grep -ho '"host_enqueue_us": [0-9.]*' gpurun_out/ab18_cfg*.log
FSX_PDL=0 timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab18_nopdl_cfg2.log 2>&1
python scripts/summarize.py gpurun_out/ab18_nopdl_cfg2.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab18.log 2>&1; tail -3 gpurun_out/pytest_ab18.log
