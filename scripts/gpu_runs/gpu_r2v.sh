# fp32 mode: fp32 row FFTs; fp64 row kernels re-instantiated (check no regression)
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_parity.py tests/test_gpu_cut.py -m gpu -q -x -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1; tail -2 gpurun_out/v_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],d['config'].get('storage','')[:3],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for c in cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/v_bench_$c.log 2>&1; python -c "$S" < gpurun_out/v_bench_$c.log; done
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --precision 32 > gpurun_out/v_bench_cfg2_f32.log 2>&1; python -c "$S" < gpurun_out/v_bench_cfg2_f32.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1
python scripts/launches.py gpurun_out/v_launches.csv | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v_launches_f32.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut --precision 32 > /dev/null 2>&1
python scripts/launches.py gpurun_out/v_launches_f32.csv | tail -3
