# A/B: pipelined vs one-tile kernels on cfg2 (+cfg3), with per-kernel launch lists
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "plans or cfg2 or golden or fft" > gpurun_out/pytest_ab.log 2>&1; tail -2 gpurun_out/pytest_ab.log
for P in 1 0; do
  FSX_PIPE=$P timeout 300 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_cfg2_pipe$P.log 2>&1
  FSX_PIPE=$P timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_cfg3_pipe$P.log 2>&1
  FSX_PIPE=$P timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_plain$P.log 2>&1 && FSX_PIPE=$P timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launches_pipe$P.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_ncu$P.log 2>&1
done
