# final check: full GPU suite, smoke, default bench line
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r_pytest.log 2>&1; tail -2 gpurun_out/r_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; tail -1 gpurun_out/r_smoke.log
timeout 900 python bench.py > gpurun_out/r_bench.log 2>&1; python scripts/summarize.py gpurun_out/r_bench.log
