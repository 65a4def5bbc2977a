# cfg1: rows of 512 (N1 = 1024) vs rows of 1024 (N1 = 512)
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for v in 0 1 0 1; do echo -n "floor=$v "; FSX_N2_FLOOR=$v timeout 300 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/a3_$v.log 2>&1; python -c "$S" < gpurun_out/a3_$v.log; done
FSX_N2_FLOOR=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cfg1 or plans or rowpair" 2>&1 | tail -1
