# round-1 final evidence (second pass): tests, smoke, bench lines, reference arm, launch lists, ncu
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f2_pytest.log 2>&1; tail -2 gpurun_out/f2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f2_smoke.log 2>&1; tail -1 gpurun_out/f2_smoke.log
timeout 600 python bench.py > gpurun_out/f2_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f2_bench_ref.log 2>&1
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/f2_bench_$c.log 2>&1; done
python scripts/summarize.py gpurun_out/f2_bench*.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f2_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/f2_ncu_l.log 2>&1
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do timeout 900 ncu $M --log-file gpurun_out/f2_dram_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/f2_ncu_$c.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c|k_cols_tma|k_c2r" -s 3 -c 3 -o gpurun_out/f2_prof_cfg2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/f2_ncu_full.log 2>&1
python scripts/launches.py gpurun_out/f2_launches_cfg2.csv
ls gpurun_out/f2_*
