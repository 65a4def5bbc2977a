# r03c: 4096-point fused pass with 8 values per thread (FSX_COLS_R8=1, 32 warps/SM): parity + A/B on cfg2
set -x
D=gpurun_out/r03c
mkdir -p $D
FSX_COLS_R8=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $D/pytest_default.txt 2>&1; echo "rc=$?" >> $D/pytest_default.txt
tail -2 $D/pytest.txt $D/pytest_default.txt
for i in 1 2 3; do
timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_r16_$i.json 2>/dev/null
FSX_COLS_R8=1 timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_r8_$i.json 2>/dev/null
done
for f in $D/c2*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
