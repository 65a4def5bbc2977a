# fp32 mode: 3D y passes in fp32 arithmetic
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/w_pytest.log 2>&1; tail -2 gpurun_out/w_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],d['config'].get('storage','')[:3],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),'e2e %.3g'%d['e2e']['value'])"
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --precision 32 > gpurun_out/w_bench_cfg4_f32.log 2>&1; python -c "$S" < gpurun_out/w_bench_cfg4_f32.log
