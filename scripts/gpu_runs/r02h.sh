# r02h: TMEM cp/ld self-test; A/B of k_fused8192c (HEAD vs relaxed peer arrive)
set -x
mkdir -p gpurun_out/r02h
timeout 60 ./scripts/micro/tmem_cp > gpurun_out/r02h/tmem_cp.txt 2>&1; echo "rc=$?" >> gpurun_out/r02h/tmem_cp.txt
for i in 1 2; do
FSX_LIB=ab/orig/libfsx.so timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02h/orig_$i.json 2>/dev/null
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-cut > gpurun_out/r02h/new_$i.json 2>/dev/null
done
cat gpurun_out/r02h/tmem_cp.txt
for f in gpurun_out/r02h/*_?.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
