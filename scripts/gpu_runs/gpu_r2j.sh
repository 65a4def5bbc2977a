# exact spectral cut: tests + bench lines (cfg2, cfg3)
timeout 900 python -m pytest tests/test_gpu_cut.py tests/test_gpu_parity.py tests/test_gpu_f32.py -m gpu -q -x -p no:cacheprovider > gpurun_out/j_pytest.log 2>&1; tail -3 gpurun_out/j_pytest.log
for c in cfg2 cfg3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/j_bench_$c.log 2>&1; python -c "
import json,sys;d=json.loads(open('gpurun_out/j_bench_$c.log').read().strip().splitlines()[-1]);c=d.get('spectral_cut');print('$c',round(d['ms_per_step'],4),c)"; done
