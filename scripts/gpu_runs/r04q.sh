# r04q: numbers at HEAD for every config (bench lines with e2e and CPU baseline for cfg3), per-kernel
# ncu counts, reference arm (oracle/_ref) on cfg3, stress sweep, full GPU suite, smoke
set -x
D=gpurun_out/r04q
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/smi.txt 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref_cfg3.json 2> $D/bench_ref.err
timeout 900 python bench.py > $D/bench_cfg3.json 2> $D/bench_cfg3.err
for c in cfg1 cfg2 cfg4 cfg5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > $D/bench_$c.json 2> $D/bench_$c.err
done
timeout 300 python bench.py --config cfg2 --precision 32 --steps 10 --warmup 3 --no-cpu > $D/bench_cfg2_f32.json 2>/dev/null
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none -c 40 --csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_$c.csv 2>/dev/null
done
python scripts/kernels_by_config.py HEAD $D/kernels_by_config.json cfg1=$D/ncu_cfg1.csv cfg2=$D/ncu_cfg2.csv cfg3=$D/ncu_cfg3.csv cfg4=$D/ncu_cfg4.csv cfg5=$D/ncu_cfg5.csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
timeout 900 python scripts/stress_parity.py 300 71 4000000 > $D/stress_s71.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
python scripts/summarize.py $D/bench_cfg3.json $D/bench_cfg1.json $D/bench_cfg2.json $D/bench_cfg4.json $D/bench_cfg5.json $D/bench_cfg2_f32.json
tail -1 $D/bench_ref_cfg3.json | cut -c1-300; cat $D/smoke.txt; tail -3 $D/stress_s71.txt; tail -3 $D/pytest.txt
