# 1D real packing: four frequencies per step in the row-pair pass
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py -m gpu -q -x -p no:cacheprovider > gpurun_out/h_pytest.log 2>&1; tail -2 gpurun_out/h_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
for c in cfg1; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/h_bench_$c.log 2>&1; python -c "$S" < gpurun_out/h_bench_$c.log; done
