# r02p: row pairs on a CTA pair (k_rowpair_c): 1D parity suites + A/B on cfg5 / cfg1
set -x
D=gpurun_out/r02p
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py tests/test_gpu_acceptance.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
for i in 1 2; do
FSX_ROWPAIR_C=0 timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c5_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c5_new_$i.json 2>$D/c5_new_$i.err
FSX_ROWPAIR_C=0 timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c1_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c1_new_$i.json 2>/dev/null
done
for f in $D/c*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
