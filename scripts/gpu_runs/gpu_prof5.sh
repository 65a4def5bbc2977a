timeout 200 python bench.py --config cfg3 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused8192h" -s 1 -c 1 -o gpurun_out/p5_prof_halves python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/p5_ncu.log 2>&1
tail -1 gpurun_out/p5_ncu.log
