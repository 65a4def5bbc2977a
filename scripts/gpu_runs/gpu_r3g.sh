# power loops: the first product as a copy
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_naive.py tests/test_gpu_cut.py -m gpu -q -x -p no:cacheprovider > gpurun_out/g3_pytest.log 2>&1; tail -2 gpurun_out/g3_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for c in cfg5 cfg5 cfg2; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/g3_$c.log 2>&1; python -c "$S" < gpurun_out/g3_$c.log; done
