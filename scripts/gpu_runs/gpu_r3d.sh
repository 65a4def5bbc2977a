# cfg3: complex symbol with offset-0 groups and +-og partners sharing phase reads
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py tests/test_gpu_slab.py -m gpu -q -x -p no:cacheprovider > gpurun_out/d3_pytest.log 2>&1; tail -2 gpurun_out/d3_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for i in 1 2; do timeout 300 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/d3_$i.log 2>&1; python -c "$S" < gpurun_out/d3_$i.log; done
