# r02x: ncu --set full of cfg4's fused pass (k_cols_tma<1024,2>) and cfg5's row pairs on a CTA pair (k_rowpair_c<4096>)
set -x
D=gpurun_out/r02x
mkdir -p $D
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma" -s 2 -c 1 -o $D/prof_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rowpair_c" -s 1 -c 1 -o $D/prof_cfg5 python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu5.log 2>&1
ls -la $D
