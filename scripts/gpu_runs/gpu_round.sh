set -x
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; tail -2 gpurun_out/pytest_gpu5.log
for c in cfg2 cfg3 cfg1 cfg4; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench5_$c.log 2>&1; done
FSX_PIPE=0 timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench5_cfg2_nopipe.log 2>&1
timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain5.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu5.log 2>&1
