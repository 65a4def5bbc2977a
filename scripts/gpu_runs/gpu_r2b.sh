# complex-symbol vectorised power (cfg3) + stall profile of the cfg2 fused pass
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b_pytest.log 2>&1; tail -3 gpurun_out/b_pytest.log
for c in cfg3 cfg2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_bench_$c.log 2>&1; tail -1 gpurun_out/b_bench_$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['config']['workload'][:5],d['ms_per_step'],d['roofline']['kernel_ms'],d['roofline']['frac'])"; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma|k_fused8192h" -s 2 -c 1 -o gpurun_out/b_prof_cfg2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused8192h" -s 1 -c 1 -o gpurun_out/b_prof_cfg3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_ncu3.log 2>&1
ls gpurun_out/
