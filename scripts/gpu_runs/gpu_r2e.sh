# prologue without shared tap terms: parity + cfg2/cfg4 bench
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_naive.py -m gpu -q -x -p no:cacheprovider > gpurun_out/e_pytest.log 2>&1; tail -3 gpurun_out/e_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
for c in cfg2 cfg4; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/e_bench_$c.log 2>&1; python -c "$S" < gpurun_out/e_bench_$c.log; done
