# r02j: non-blocking prefetch state machine: parity + A/B vs k_fused8192c
set -x
mkdir -p gpurun_out/r02j
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_cut.py -x -q -k "cfg3 or 8192 or halves or plan or slab or cut" > gpurun_out/r02j/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02j/pytest.txt
tail -5 gpurun_out/r02j/pytest.txt
for i in 1 2; do
FSX_F8192=c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02j/c_$i.json 2>/dev/null
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02j/p_$i.json 2>gpurun_out/r02j/p_$i.err
done
for f in gpurun_out/r02j/*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline']['frac'])"; done
