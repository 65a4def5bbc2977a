# r02d: k_fused8192c with st.async/mbarrier exchanges; acceptance/io tests; cfg3 bench; ncu of the kernel
set -x
mkdir -p gpurun_out/r02d
python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_acceptance.py tests/test_gpu_concurrency.py -x -q -s > gpurun_out/r02d/pytest.txt 2>&1
python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "cfg3_full_size_vs_oracle" > gpurun_out/r02d/pytest_full.txt 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02d/bench_cfg3.json 2> gpurun_out/r02d/bench_cfg3.err
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02d/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused8192c -s 2 -c 1 -o gpurun_out/r02d/prof_cfg3 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02d/ncu3.log 2>&1
tail -3 gpurun_out/r02d/pytest.txt; tail -3 gpurun_out/r02d/pytest_full.txt
python -c "
import json; d=json.loads(open('gpurun_out/r02d/bench_cfg3.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline']['frac'])"
