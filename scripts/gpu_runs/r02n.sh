# r02n: M = 2048 group rows (FSX_ROW_GROUPS=2) on cfg2: parity + A/B
set -x
mkdir -p gpurun_out/r02n
FSX_ROW_GROUPS=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py -x -q > gpurun_out/r02n/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02n/pytest.txt
tail -2 gpurun_out/r02n/pytest.txt
for i in 1 2; do
timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02n/g1_$i.json 2>/dev/null
FSX_ROW_GROUPS=2 timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02n/g2_$i.json 2>/dev/null
done
for f in gpurun_out/r02n/g*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline']['frac'])"; done
