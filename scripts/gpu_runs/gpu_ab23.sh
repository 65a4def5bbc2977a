# TMEM-parked multipliers for the 8192-point fused columns
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_ab23.log 2>&1; tail -2 gpurun_out/pytest_ab23.log
timeout 300 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab23_cfg3.log 2>&1
python scripts/summarize.py gpurun_out/ab23_cfg3.log
