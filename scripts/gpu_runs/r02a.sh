# r02a: full-size parity (cfg3, cfg4), cfg3 headline bench, reference arm at full size
set -x
mkdir -p gpurun_out/r02a
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/r02a/host.txt 2>&1
python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/r02a/pytest_fullsize.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r02a/bench_cfg3.json 2> gpurun_out/r02a/bench_cfg3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02a/bench_ref_cfg3.json 2> gpurun_out/r02a/bench_ref.err
tail -5 gpurun_out/r02a/pytest_fullsize.txt; cat gpurun_out/r02a/bench_cfg3.json gpurun_out/r02a/bench_ref_cfg3.json
