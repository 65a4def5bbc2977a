# FP64 peak + per-launch DP instruction counts of the fused kernels
./scripts/micro/fp64_peak > gpurun_out/fp64_peak.json; cat gpurun_out/fp64_peak.json
M="--metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none --csv"
timeout 300 ncu $M -k regex:"k_cols_tma" --log-file gpurun_out/fp64_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu $M -k regex:"k_fused8192h" --log-file gpurun_out/fp64_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu $M -k regex:"k_cols_tma<1024, 2" --log-file gpurun_out/fp64_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu $M -k regex:"k_rowpair" --log-file gpurun_out/fp64_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu $M -k regex:"k_rowpair" --log-file gpurun_out/fp64_cfg1.csv python bench.py --config cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/fp64_*
