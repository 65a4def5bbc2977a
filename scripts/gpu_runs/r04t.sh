# r04t: light twiddle prefetch (LPF) in k_rowpair_c's row FFTs against the previous build, cfg5
set -x
D=gpurun_out/r04t
mkdir -p $D
for rep in 1 2 3; do
  FSX_LIB=$PWD/ab/libfsx_old.so timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/old_$rep.json 2>/dev/null
  timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/new_$rep.json 2>/dev/null
done
for f in $D/old_*.json $D/new_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "rowpair or cfg5 or many_fields or plans" > $D/pytest.txt 2>&1; tail -2 $D/pytest.txt
