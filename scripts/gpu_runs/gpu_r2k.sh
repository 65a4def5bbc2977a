# L2 persisting window on H (A/B)
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
python -c "import torch;p=torch.cuda.get_device_properties(0);print('L2',p.L2_cache_size>>20,'MiB')"
for c in cfg2 cfg3 cfg4; do for v in 0 1; do FSX_L2PERSIST=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/k_bench_${c}_$v.log 2>&1; echo -n "persist=$v "; python -c "$S" < gpurun_out/k_bench_${c}_$v.log; done; done
FSX_L2PERSIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "cfg2 or plans" 2>&1 | tail -1
