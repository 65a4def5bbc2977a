# r04a: re-entry check at HEAD (smoke, cfg3/cfg5 bench) + source-level ncu of cfg5's row pairs and cfg3's fused columns
set -x
D=gpurun_out/r04a
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > $D/bench_cfg3.json 2> $D/bench_cfg3.err
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu > $D/bench_cfg5.json 2> $D/bench_cfg5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rowpair_c -s 2 -c 1 -o $D/rowpair_c python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_cfg5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fused8192c -s 2 -c 1 -o $D/fused8192c python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_cfg3.log 2>&1
cat $D/smoke.txt
for c in cfg3 cfg5; do python -c "
import json; d=json.loads(open('$D/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), '%.3e'%d['value'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), round(d['pipeline']['frac'],3))"; done
