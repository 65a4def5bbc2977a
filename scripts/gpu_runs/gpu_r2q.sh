# fp32 mode: the fused pass in fp32 arithmetic (A/B with FSX_F32_COMPUTE=0)
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_cut.py -m gpu -q -x -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),'e2e %.3g'%d['e2e']['value'])"
for c in cfg2 cfg4; do for v in 1 0; do echo -n "f32compute=$v "; FSX_F32_COMPUTE=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --precision 32 > gpurun_out/q_bench_${c}_$v.log 2>&1; python -c "$S" < gpurun_out/q_bench_${c}_$v.log; done; done
