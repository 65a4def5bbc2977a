# r02c: ncu --set full of the cfg3 fused kernel (k_fused8192c) and cfg2 fused kernel
set -x
mkdir -p gpurun_out/r02c
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02c/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused8192c -s 2 -c 1 -o gpurun_out/r02c/prof_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02c/ncu3.log 2>&1
python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02c/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cols_tma -s 2 -c 1 -o gpurun_out/r02c/prof_cfg2 python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02c/ncu2.log 2>&1
ls -la gpurun_out/r02c
