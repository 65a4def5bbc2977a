# FP64 instruction counts and DRAM bytes of the cfg2 / cfg3 / cfg4 fused passes after the symbol changes
P=r01h
F="--metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none --csv"
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
for c in cfg2 cfg4; do timeout 900 ncu $F -k regex:"k_cols_tma" --log-file gpurun_out/${P}_fp64_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1; done
for c in cfg2 cfg3 cfg4; do timeout 900 ncu $M --log-file gpurun_out/${P}_dram_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1; python scripts/launches.py gpurun_out/${P}_dram_$c.csv | tail -5; done
