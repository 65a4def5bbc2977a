# r04v: zero-column shortcut in the fp32 mode's fused pass (k_cols_tma_f32<4096,2>): A/B on cfg2 --precision 32, fp32 tests
set -x
D=gpurun_out/r04v
mkdir -p $D
for rep in 1 2 3; do
  FSX_LIB=$PWD/ab/libfsx_old.so timeout 600 python bench.py --config cfg2 --precision 32 --steps 30 --warmup 3 --no-cpu --no-e2e --no-cut > $D/old_$rep.json 2>/dev/null
  timeout 600 python bench.py --config cfg2 --precision 32 --steps 30 --warmup 3 --no-cpu --no-e2e --no-cut > $D/new_$rep.json 2>/dev/null
done
for f in $D/old_*.json $D/new_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
timeout 900 python -m pytest tests/test_gpu_f32.py tests/test_gpu_cut.py -q > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt
