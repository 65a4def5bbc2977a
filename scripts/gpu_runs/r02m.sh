# r02m: two-group row kernels at M = 4096 (k_r2c_grp / k_c2r_grp): full GPU suite + A/B on cfg3
set -x
mkdir -p gpurun_out/r02m
for i in 1 2; do
FSX_ROW_GROUPS=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02m/g0_$i.json 2>/dev/null
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02m/g1_$i.json 2>gpurun_out/r02m/g1_$i.err
done
for f in gpurun_out/r02m/g*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'], d['pipeline']['frac'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_r2c|k_c2r" -c 6 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/r02m/launch_rows.csv 2>/dev/null
grep -E "k_r2c|k_c2r" gpurun_out/r02m/launch_rows.csv | cut -c1-40,200-300 | head
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02m/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02m/pytest.txt
tail -3 gpurun_out/r02m/pytest.txt
