# fp32 storage mode: tests + bench lines (fp64 default and fp32) for cfg2
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; tail -3 gpurun_out/f_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],d['config'].get('storage'),round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),'pipe',round(d['pipeline']['frac'],3),'e2e %.3g single %.3g'%(d['e2e']['value'],d['e2e']['single_call_value']))"
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu > gpurun_out/f_bench_cfg2.log 2>&1; python -c "$S" < gpurun_out/f_bench_cfg2.log
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --precision 32 > gpurun_out/f_bench_cfg2_f32.log 2>&1; python -c "$S" < gpurun_out/f_bench_cfg2_f32.log
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --precision 32 > gpurun_out/f_bench_cfg4_f32.log 2>&1; python -c "$S" < gpurun_out/f_bench_cfg4_f32.log
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu --precision 32 > gpurun_out/f_bench_cfg5_f32.log 2>&1; python -c "$S" < gpurun_out/f_bench_cfg5_f32.log
