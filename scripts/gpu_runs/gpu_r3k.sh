# 1024-point fused pass with 2-column tiles (FSX_FUSED_NARROW=1) vs 4-column tiles
FSX_FUSED_NARROW=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py -m gpu -q -x -p no:cacheprovider > gpurun_out/k3_pytest.log 2>&1; tail -2 gpurun_out/k3_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for v in 0 1 0 1; do echo -n "narrow=$v "; FSX_FUSED_NARROW=$v timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/k3_$v.log 2>&1; python -c "$S" < gpurun_out/k3_$v.log; done
