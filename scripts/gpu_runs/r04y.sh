# r04y (re-run as r04y after the ColumnCut change): final check of the built library at HEAD: smoke, the full GPU suite with -x, default bench line
set -x
D=gpurun_out/r04y
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; cat $D/smoke.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt; tail -3 $D/pytest.txt
timeout 900 python bench.py > $D/bench_cfg3.json 2> $D/bench_cfg3.err
python scripts/summarize.py $D/bench_cfg3.json
