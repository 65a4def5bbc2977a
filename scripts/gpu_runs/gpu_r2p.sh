# cfg4: ncu --set full of the fused pass (second k_cols_tma launch of a solve)
P=r01e
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma" -s 1 -c 1 -o gpurun_out/${P}_prof_cfg4f python bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/${P}_prof_cfg4f.ncu-rep gpurun_out/${P}_ncu_full_cfg4_summary.json "ncu --set full --clock-control none --import-source on, cfg4 fused pass (bench.py --config cfg4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut)"
rm -f gpurun_out/${P}_prof_cfg4f.ncu-rep
