# ncu --set full of the fp32 mode's kernels on cfg2 (rows + fused pass in fp32 arithmetic)
P=r01f
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c|k_cols_tma|k_c2r" -s 3 -c 3 -o gpurun_out/${P}_prof_cfg2_f32 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut --precision 32 > gpurun_out/y_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${P}_prof_cfg2_f32.ncu-rep gpurun_out/${P}_ncu_full_cfg2_f32_summary.json "ncu --set full --clock-control none --import-source on, cfg2 fp32 mode (bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut --precision 32)"
rm -f gpurun_out/${P}_prof_cfg2_f32.ncu-rep
