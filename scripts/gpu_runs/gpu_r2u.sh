# spectral cut: fused-pass tile skip (3D)
timeout 900 python -m pytest tests/test_gpu_cut.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/u_pytest.log 2>&1; tail -2 gpurun_out/u_pytest.log
for c in cfg4 cfg2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/u_bench_$c.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/u_bench_$c.log').read().strip().splitlines()[-1]);c=d.get('spectral_cut');print('$c',round(d['ms_per_step'],4),round(c['ms_per_step'],4),c['bitwise_equal_to_full'],c['columns_kept'])"; done
