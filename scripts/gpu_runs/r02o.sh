# r02o: round-2 numbers at HEAD for every config: bench lines (with e2e), launch lists, FP64 + DRAM counts of the dominant kernels
set -x
D=gpurun_out/r02o
mkdir -p $D
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $D/bench_$c.json 2> $D/bench_$c.err
done
timeout 300 python bench.py --config cfg2 --precision 32 --steps 10 --warmup 3 --no-cpu > $D/bench_cfg2_f32.json 2>/dev/null
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none -c 40 --csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_$c.csv 2>/dev/null
done
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python -c "
import json; d=json.loads(open('$D/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['pipeline']['frac'], d.get('e2e',{}).get('value'))"; done
