# narrow TMA column tiles for small 1D problems (FSX_AXIS_NARROW=0/2/4)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py -m gpu -q -x -p no:cacheprovider > gpurun_out/z_pytest.log 2>&1; tail -2 gpurun_out/z_pytest.log
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for v in 0 2 4 0 2; do echo -n "narrow=$v "; FSX_AXIS_NARROW=$v timeout 300 python bench.py --config cfg1 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/z_$v.log 2>&1; python -c "$S" < gpurun_out/z_$v.log; done
FSX_AXIS_NARROW=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z_launches.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1
python scripts/launches.py gpurun_out/z_launches.csv | tail -3
