# r04d: numbers at HEAD 39fc4e8 for every config (bench lines with e2e and CPU baseline for cfg3),
# per-kernel ncu counts, reference arm on cfg3, stress sweep, full GPU suite, smoke
set -x
D=gpurun_out/r04d
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/smi.txt 2>&1
timeout 900 python bench.py > $D/bench_cfg3.json 2> $D/bench_cfg3.err
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $D/bench_$c.json 2> $D/bench_$c.err
done
timeout 300 python bench.py --config cfg2 --precision 32 --steps 10 --warmup 3 --no-cpu > $D/bench_cfg2_f32.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref_cfg3.json 2> $D/bench_ref.err
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none -c 40 --csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_$c.csv 2>/dev/null
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 900 python scripts/stress_parity.py 300 41 4000000 > $D/stress_s41.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
for c in cfg1 cfg2 cfg3 cfg4 cfg5 cfg2_f32; do python -c "
import json; d=json.loads(open('$D/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],4), '%.3e'%d['value'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), round(d['pipeline']['frac'],3), '%.3e'%d.get('e2e',{}).get('value',0))"; done
tail -1 $D/bench_ref_cfg3.json | cut -c1-300; cat $D/smoke.txt; tail -3 $D/stress_s41.txt; tail -3 $D/pytest.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fused8192c -s 2 -c 1 -o $D/fused8192c python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_full_cfg3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_rowpair_c -s 2 -c 1 -o $D/rowpair_c python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_full_cfg5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cols_tma -s 2 -c 1 -o $D/cols_tma_cfg2 python bench.py --config cfg2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_full_cfg2.log 2>&1
ls -la $D
