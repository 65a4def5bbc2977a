# r04r: zero columns of the parked-multiplier path (k_cols_tma<4096,2>, cfg2) through zero_products: A/B against
# the previous build on cfg2, bitwise zero-column test, cut / parity tests
set -x
D=gpurun_out/r04r
mkdir -p $D
for rep in 1 2 3; do
  FSX_LIB=$PWD/ab/libfsx_old.so timeout 600 python bench.py --config cfg2 --steps 30 --warmup 3 --no-cpu --no-e2e --no-cut > $D/old_$rep.json 2>/dev/null
  timeout 600 python bench.py --config cfg2 --steps 30 --warmup 3 --no-cpu --no-e2e --no-cut > $D/new_$rep.json 2>/dev/null
done
for f in $D/old_*.json $D/new_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
timeout 1200 python -m pytest tests/test_gpu_cut.py tests/test_gpu_parity.py tests/test_reference_outputs.py -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
