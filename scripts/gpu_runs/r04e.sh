# r04e: radix-16 passes with the twiddles folded into the butterflies (FSX_FUSED16): A/B against the
# previous arithmetic on one box (ab/libfsx_old.so = -DFSX_FUSED16=0), full GPU suite on the new build,
# source-level ncu of the cfg3 / cfg5 / cfg2 dominant kernels exported to csv on the box
set -x
D=gpurun_out/r04e
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/smi.txt 2>&1
for rep in 1 2; do
for c in cfg3 cfg2 cfg5 cfg4 cfg1; do
  FSX_LIB=$PWD/ab/libfsx_old.so timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ab_old_${c}_$rep.json 2>/dev/null
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ab_new_${c}_$rep.json 2>/dev/null
done
done
for f in $D/ab_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d.get('stages_ms'))"; done
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
for spec in "cfg3 k_fused8192c fused8192c" "cfg5 k_rowpair_c rowpair_c" "cfg2 k_cols_tma cols_tma_cfg2"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 -s 2 -c 1 -o /tmp/$3 -f python bench.py --config $1 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_full_$1.log 2>&1
  ncu -i /tmp/$3.ncu-rep --page raw --csv > $D/$3_raw.csv 2>/dev/null
  ncu -i /tmp/$3.ncu-rep --page source --csv --print-source sass > $D/$3_src.csv 2>/dev/null
  rm -f /tmp/$3.ncu-rep
done
du -sh $D
