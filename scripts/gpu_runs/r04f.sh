# r04f: L2 strip prefetch (128-byte lines, FSX_F8192_PFD columns ahead) in k_fused8192c: distance sweep on cfg3
set -x
D=gpurun_out/r04f
mkdir -p $D
for rep in 1 2; do
for pfd in 0 152 304 608 1216; do
  FSX_F8192_PFD=$pfd timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/pfd_${pfd}_$rep.json 2>/dev/null
done
done
for f in $D/pfd_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
FSX_F8192_PFD=304 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cut.py -q -k "cfg3 or plans or cut" > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
FSX_F8192_PFD=304 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fused8192c -c 3 --csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_pfd304.csv 2>/dev/null
FSX_F8192_PFD=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_fused8192c -c 3 --csv python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_pfd0.csv 2>/dev/null
grep k_fused $D/ncu_pfd304.csv | tail -5 | cut -d, -f 5,13- ; grep k_fused $D/ncu_pfd0.csv | tail -5 | cut -d, -f 5,13-
