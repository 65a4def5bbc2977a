# cfg5 row-pair: 2 vs 4 interleaved 2x2 power chains
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
for v in nx2 nx4; do cp ab/libfsx_$v.so paper_2105_06676_b200/libfsx.so; echo -n "$v "; timeout 600 python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/i_bench_$v.log 2>&1; python -c "$S" < gpurun_out/i_bench_$v.log; done
cp ab/libfsx_nx4.so paper_2105_06676_b200/libfsx.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "leapfrog or cfg5 or rowpair or plans" > gpurun_out/i_pytest.log 2>&1; tail -2 gpurun_out/i_pytest.log
