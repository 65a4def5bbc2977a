# r02e: baseline at HEAD after re-entry: full GPU suite, default bench (cfg3), launch list, ncu full of k_fused8192c
set -x
mkdir -p gpurun_out/r02e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02e/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/r02e/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e/pytest.txt
timeout 600 python bench.py > gpurun_out/r02e/bench.json 2> gpurun_out/r02e/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02e/bench_ref.json 2> gpurun_out/r02e/bench_ref.err
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02e/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02e/ncu_l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused8192c -s 2 -c 1 -o gpurun_out/r02e/prof_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02e/ncu3.log 2>&1
tail -5 gpurun_out/r02e/pytest.txt; tail -2 gpurun_out/r02e/bench.json
