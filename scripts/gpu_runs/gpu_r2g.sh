# fused passes storing from registers (FSX_COLS_DST=1) vs smem + TMA store
FSX_COLS_DST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/g_pytest.log 2>&1; tail -2 gpurun_out/g_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
for c in cfg2 cfg3 cfg4; do for d in 0 1; do FSX_COLS_DST=$d timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g_bench_${c}_$d.log 2>&1; echo -n "dst=$d "; python -c "$S" < gpurun_out/g_bench_${c}_$d.log; done; done
