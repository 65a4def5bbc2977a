# r02t: group rows with bulk-store epilogues (FSX_ROW_BS=1): parity + A/B on cfg3
set -x
D=gpurun_out/r02t
mkdir -p $D
FSX_ROW_BS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py tests/test_gpu_slabs.py -x -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -2 $D/pytest.txt
for i in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > $D/bs0_$i.json 2>/dev/null
FSX_ROW_BS=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > $D/bs1_$i.json 2>/dev/null
done
for f in $D/bs*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
FSX_ROW_BS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_r2c|k_c2r" -c 6 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut 2>/dev/null | grep -E "k_r2c|k_c2r" | awk -F'","' '{print $5, $NF}' | cut -c1-60,200-240
