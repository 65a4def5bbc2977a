# fused-pass multiplier power: 4 / 8 / 16 elements per warp-skip chunk
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for v in ch4 ch8 ch16 ch4 ch8 ch16; do cp ab/libfsx_$v.so paper_2105_06676_b200/libfsx.so; for c in cfg2; do echo -n "$v "; timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/l3_$v.log 2>&1; python -c "$S" < gpurun_out/l3_$v.log; done; done
cp ab/libfsx_ch8.so paper_2105_06676_b200/libfsx.so; echo -n "ch8 cfg4 "; timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut 2>&1 | tail -1 | python -c "$S"
cp ab/libfsx_ch4.so paper_2105_06676_b200/libfsx.so; echo -n "ch4 cfg4 "; timeout 300 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut 2>&1 | tail -1 | python -c "$S"
