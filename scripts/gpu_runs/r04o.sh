# r04o: first-wave stagger in k_fused8192c (FSX_F8192_STAGGER ns: odd pairs of the first wave start late), cfg3
set -x
D=gpurun_out/r04o
mkdir -p $D
for rep in 1 2; do
for ns in 0 4000 8000 12000; do
  FSX_F8192_STAGGER=$ns timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/st${ns}_$rep.json 2>/dev/null
done
done
for f in $D/st*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
