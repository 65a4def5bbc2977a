M="--metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none --csv"
timeout 600 ncu $M --kernel-name-base demangled -k regex:"k_cols_tma<\(int\)1024, \(int\)2" --log-file gpurun_out/fp64_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/fp64_cfg4.log 2>&1
tail -3 gpurun_out/fp64_cfg4.csv
