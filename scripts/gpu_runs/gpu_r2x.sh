# full twiddle tables per pass in the 4096-point fused pass (FSX_FT4096 mask), A/B on one box
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for v in ft0 ft2 ft4 ft6 ft0; do cp ab/libfsx_$v.so paper_2105_06676_b200/libfsx.so; echo -n "$v "; timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > gpurun_out/x_$v.log 2>&1; python -c "$S" < gpurun_out/x_$v.log; done
