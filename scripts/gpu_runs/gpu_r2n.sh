# fp32 storage mode: float I/O fused into the 1D plan's split column passes
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/n_pytest.log 2>&1; tail -2 gpurun_out/n_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],d['config'].get('storage','')[:3],round(d['ms_per_step'],4),'e2e %.3g'%d['e2e']['value'])"
for p in 64 32; do timeout 600 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --precision $p > gpurun_out/n_bench_cfg5_$p.log 2>&1; python -c "$S" < gpurun_out/n_bench_cfg5_$p.log; done
