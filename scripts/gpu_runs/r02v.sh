# r02v: light twiddle prefetch (LPF: next pass's 4 base twiddles loaded before the exchange barrier) A/B on cfg3 / cfg2
set -x
D=gpurun_out/r02v
mkdir -p $D
FSX_LIB=ab/lpf/libfsx.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -2 $D/pytest.txt
for i in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c3_base_$i.json 2>/dev/null
FSX_LIB=ab/lpf/libfsx.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c3_lpf_$i.json 2>/dev/null
timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_base_$i.json 2>/dev/null
FSX_LIB=ab/lpf/libfsx.so timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-cut > $D/c2_lpf_$i.json 2>/dev/null
done
for f in $D/c*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
for L in "" "FSX_LIB=ab/lpf/libfsx.so"; do env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_r2c|k_c2r|k_fused" -c 9 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut 2>/dev/null | grep -E "k_r2c|k_c2r|k_fused" | awk -F'","' '{print substr($5,1,30), $NF}'; done
