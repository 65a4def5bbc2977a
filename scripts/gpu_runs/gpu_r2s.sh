# persistent ping-pong 8192-point fused pass (FSX_HALVES=2) vs the halves kernel
FSX_HALVES=2 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py -m gpu -q -x -p no:cacheprovider -k "8192 or cut" > gpurun_out/s_pytest.log 2>&1; tail -3 gpurun_out/s_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
for v in 1 2; do echo -n "halves=$v "; FSX_HALVES=$v timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/s_bench_$v.log 2>&1; python -c "$S" < gpurun_out/s_bench_$v.log; done
