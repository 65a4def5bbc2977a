# full ncu capture of the row kernels + fused pass (cfg2), after a clean run
timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/pr2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c|k_cols_tma|k_c2r" -s 3 -c 3 -o gpurun_out/pr2_prof_cfg2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/pr2_ncu_full.log 2>&1
tail -3 gpurun_out/pr2_ncu_full.log
