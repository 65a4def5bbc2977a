# r02l: ncu --set full of the cfg3 row kernels (k_r2c_bulk<4096,3>, k_c2r_bulk<4096,3>)
set -x
mkdir -p gpurun_out/r02l
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02l/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c_bulk|k_c2r_bulk" -s 4 -c 2 -o gpurun_out/r02l/prof_rows python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02l/ncu.log 2>&1
ls -la gpurun_out/r02l; tail -3 gpurun_out/r02l/ncu.log
