# ncu --set full summaries of the cfg1 / cfg3 / cfg5 dominant kernels at HEAD
P=r01g
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowpair" -s 1 -c 1 -o gpurun_out/${P}_prof_cfg1 python bench.py --config cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused8192h" -s 1 -c 1 -o gpurun_out/${P}_prof_cfg3 python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rowpair" -s 1 -c 1 -o gpurun_out/${P}_prof_cfg5 python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1
for c in cfg1 cfg3 cfg5; do python scripts/ncu_summary.py gpurun_out/${P}_prof_$c.ncu-rep gpurun_out/${P}_ncu_full_${c}_summary.json "ncu --set full --clock-control none --import-source on, $c dominant kernel at HEAD (bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut)"; rm -f gpurun_out/${P}_prof_$c.ncu-rep; done
