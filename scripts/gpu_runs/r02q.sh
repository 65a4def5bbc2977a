# r02q: persistent two-group fused column pass (k_cols_grp): parity suites + A/B on cfg2 / cfg4
set -x
D=gpurun_out/r02q
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py tests/test_gpu_slab.py tests/test_gpu_multi.py tests/test_gpu_slabs.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
for i in 1 2; do
FSX_COLS_GRP=0 timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_new_$i.json 2>$D/c2_new_$i.err
FSX_COLS_GRP=0 timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c4_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c4_new_$i.json 2>/dev/null
done
for f in $D/c*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
