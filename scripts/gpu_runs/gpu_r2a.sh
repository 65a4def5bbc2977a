# round-1 re-entry check: tests, smoke, default bench, cfg3/cfg5 bench
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/a_pytest.log 2>&1; tail -3 gpurun_out/a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; tail -1 gpurun_out/a_smoke.log
timeout 600 python bench.py > gpurun_out/a_bench.log 2>&1; tail -1 gpurun_out/a_bench.log
for c in cfg3 cfg5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/a_bench_$c.log 2>&1; tail -1 gpurun_out/a_bench_$c.log; done
