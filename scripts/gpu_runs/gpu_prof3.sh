# launch lists for cfg3/cfg4 and full captures of their fused column kernels
timeout 300 python bench.py --config cfg3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p3_plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p3_launch_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/p3_ncu3.log 2>&1
timeout 300 python bench.py --config cfg4 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p3_plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma" -s 5 -c 2 -o gpurun_out/p3_prof_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/p3_ncu4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma|k_r2c|k_c2r" -s 3 -c 3 -o gpurun_out/p3_prof_cfg3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/p3_ncu3f.log 2>&1
python scripts/launches.py gpurun_out/p3_launch_cfg3.csv
tail -2 gpurun_out/p3_ncu4.log gpurun_out/p3_ncu3f.log
