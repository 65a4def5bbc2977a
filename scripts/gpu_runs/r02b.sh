# r02b: 8192-point CTA-pair fused kernel + spill fixes: parity, concurrency tests, cfg3/cfg2 bench
set -x
mkdir -p gpurun_out/r02b
python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_slab.py tests/test_gpu_cut.py -x -q > gpurun_out/r02b/pytest.txt 2>&1
python -m pytest tests/test_gpu_fullsize.py -x -q -s -k "cfg3_full_size_vs_oracle" > gpurun_out/r02b/pytest_full.txt 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02b/bench_cfg3.json 2> gpurun_out/r02b/bench_cfg3.err
FSX_F8192=h python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02b/bench_cfg3_h.json 2>&1
python bench.py --config cfg2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/r02b/bench_cfg2.json 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02b/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02b/launches_cfg3.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02b/ncu.log 2>&1
tail -3 gpurun_out/r02b/pytest.txt gpurun_out/r02b/pytest_full.txt
python - <<'P'
import json
for f in ["bench_cfg3","bench_cfg3_h","bench_cfg2"]:
    try:
        d=json.loads(open(f"gpurun_out/r02b/{f}.json").read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"]["kernel_ms"], d["roofline"]["frac"], d["pipeline"]["frac"], d.get("e2e",{}).get("value"))
    except Exception as e: print(f, "ERR", e)
P
