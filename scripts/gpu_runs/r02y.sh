# r02y: power-of-two phase indices in the 1D row-pair symbols (modp2): parity + A/B on cfg5 / cfg1; ncu of cfg4's fused pass
set -x
D=gpurun_out/r02y
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py tests/test_gpu_naive.py -x -q -k "1d or row or cfg5 or cfg1 or naive or pair or vector" > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -2 $D/pytest.txt
for i in 1 2; do
FSX_LIB=ab/old/libfsx.so timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c5_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/c5_new_$i.json 2>/dev/null
FSX_LIB=ab/old/libfsx.so timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c1_old_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c1_new_$i.json 2>/dev/null
done
for f in $D/c*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cols_tma" -s 1 -c 1 -o $D/prof_cfg4 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu4.log 2>&1
