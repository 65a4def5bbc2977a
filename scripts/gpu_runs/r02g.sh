# r02g: k_fused8192c with the tap terms off the FFT's critical path + relaxed peer arrive: parity + cfg3 bench
set -x
mkdir -p gpurun_out/r02g
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -s -k "cfg3 or halves or 8192 or plan" > gpurun_out/r02g/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02g/pytest.txt
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02g/bench_cfg3_$i.json 2>/dev/null; done
tail -5 gpurun_out/r02g/pytest.txt
for i in 1 2; do python -c "
import json; d=json.loads(open('gpurun_out/r02g/bench_cfg3_$i.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline']['frac'])"; done
