# r04g: cfg1 four-step split sweep (FSX_N2LOG: row length 2^b2; default b2 = 10, N1 = 512 columns)
set -x
D=gpurun_out/r04g
mkdir -p $D
for rep in 1 2; do
for b2 in 8 9 10 11 12; do
  FSX_N2LOG=$b2 timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/n2log_${b2}_$rep.json 2>$D/n2log_${b2}_$rep.err
done
done
for f in $D/n2log_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['roofline']['kernel'])"; done
for b2 in 8 9; do FSX_N2LOG=$b2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "cfg1 or rowpair or plans" > $D/pytest_$b2.txt 2>&1; tail -1 $D/pytest_$b2.txt; done
