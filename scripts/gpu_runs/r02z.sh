# r02z: per-column thread groups (named barriers) in the multi-column TMA column kernels: parity + A/B on cfg4 / cfg1 / cfg2
set -x
D=gpurun_out/r02z
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_multi.py tests/test_gpu_slabs.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -2 $D/pytest.txt
for i in 1 2; do
FSX_LIB=ab/old/libfsx.so timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c4_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c4_new_$i.json 2>/dev/null
done
FSX_LIB=ab/old/libfsx.so timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c1_old.json 2>/dev/null
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c1_new.json 2>/dev/null
for f in $D/c*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
for L in "FSX_LIB=ab/old/libfsx.so" "X=1"; do env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cols_tma" -c 3 --csv python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu --no-e2e --no-cut 2>/dev/null | grep k_cols_tma | awk -F'","' '{print substr($5,1,36), $NF}'; done
