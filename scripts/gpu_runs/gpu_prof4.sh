timeout 200 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma" -s 1 -c 1 -o gpurun_out/p4_prof_cols python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p4_ncu.log 2>&1
tail -1 gpurun_out/p4_ncu.log
