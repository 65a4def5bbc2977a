timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p6_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c_bulk|k_c2r_bulk" -s 2 -c 2 -o gpurun_out/p6_prof_rows python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p6_ncu.log 2>&1
tail -1 gpurun_out/p6_ncu.log
