FSX_HALVES=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused8192p" -s 1 -c 1 -o gpurun_out/t_prof python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > gpurun_out/t_ncu.log 2>&1
tail -2 gpurun_out/t_ncu.log
