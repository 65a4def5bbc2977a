timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c_pair|k_c2r_pair|k_cols_tma" -s 3 -c 3 -o gpurun_out/d_prof_cfg2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/d_ncu.log 2>&1
tail -2 gpurun_out/d_ncu.log
