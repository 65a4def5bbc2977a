# r03a: L2 promotion of the column tensor maps (FSX_L2PROMO 0/64/128/256) on cfg3 / cfg2
set -x
D=gpurun_out/r03a
mkdir -p $D
for p in 256 128 64 0 256; do
FSX_L2PROMO=$p timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c3_$p.json 2>/dev/null
FSX_L2PROMO=$p timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_$p.json 2>/dev/null
python -c "
import json
for c in ('c3','c2'):
    d=json.loads(open('$D/'+c+'_$p.json').read().strip().splitlines()[-1]); print(c, $p, d['ms_per_step'], d['roofline']['kernel_ms'])"
done
