# row-pair layout: parity + A/B vs the per-row layout + launch list
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/c_pytest.log 2>&1; tail -3 gpurun_out/c_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4),round(d['roofline']['frac'],3))"
for c in cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c_bench_$c.log 2>&1; python -c "$S" < gpurun_out/c_bench_$c.log; done
FSX_PAIR=0 timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c_bench_cfg2_nopair.log 2>&1; python -c "$S" < gpurun_out/c_bench_cfg2_nopair.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/c_ncu.log 2>&1
python scripts/launches.py gpurun_out/c_launches_cfg2.csv | tail -12
