# cfg1: symmetric symbol with one phase read per |offset| (mode 0)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py -m gpu -q -x -p no:cacheprovider > gpurun_out/c3_pytest.log 2>&1; tail -2 gpurun_out/c3_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for i in 1 2; do timeout 300 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/c3_$i.log 2>&1; python -c "$S" < gpurun_out/c3_$i.log; done
