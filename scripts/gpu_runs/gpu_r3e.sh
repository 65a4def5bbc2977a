# real fused symbols: +-og pairs counted once (2 Re A e)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py tests/test_gpu_f32.py tests/test_gpu_slab.py -m gpu -q -x -p no:cacheprovider > gpurun_out/e3_pytest.log 2>&1; tail -2 gpurun_out/e3_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for c in cfg2 cfg2 cfg4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/e3_$c.log 2>&1; python -c "$S" < gpurun_out/e3_$c.log; done
