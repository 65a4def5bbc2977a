# round-1 final evidence (r01g): tests, smoke, bench lines (fp64 all configs, fp32 cfg2),
# reference arm, cfg2 launch list and ncu --set full summary of the three cfg2 kernels
P=r01g
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${P}_pytest.log 2>&1; tail -2 gpurun_out/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P}_smoke.log 2>&1; tail -1 gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${P}_bench_ref.log 2>&1
timeout 600 python bench.py --precision 32 --no-cpu --no-cut > gpurun_out/${P}_bench_cfg2_f32.log 2>&1
for c in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/${P}_bench_$c.log 2>&1; done
python scripts/summarize.py gpurun_out/${P}_bench*.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut > gpurun_out/${P}_ncu_l.log 2>&1
python scripts/launches.py gpurun_out/${P}_launches_cfg2.csv | tail -5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c|k_cols_tma|k_c2r" -s 3 -c 3 -o gpurun_out/${P}_prof_cfg2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-cut > gpurun_out/${P}_ncu_full.log 2>&1
python scripts/ncu_summary.py gpurun_out/${P}_prof_cfg2.ncu-rep gpurun_out/${P}_ncu_full_cfg2_summary.json "ncu --set full --clock-control none --import-source on, cfg2 (bench.py --steps 2 --warmup 3 --no-e2e --no-cpu), round-1 final kernels"
ls gpurun_out/${P}_*
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
for c in cfg1 cfg5; do timeout 900 ncu $M --log-file gpurun_out/${P}_dram_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > gpurun_out/${P}_ncu_$c.log 2>&1; python scripts/launches.py gpurun_out/${P}_dram_$c.csv | tail -4; done
F="--metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none --csv"
for c in cfg1 cfg3 cfg5; do timeout 900 ncu $F -k regex:"k_rowpair|k_fused8192h" --log-file gpurun_out/${P}_fp64_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu --no-cut > gpurun_out/${P}_fp64_$c.log 2>&1; done
ls gpurun_out/${P}_*
