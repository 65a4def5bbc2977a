# rows: one stage x 3 or 4 CTAs/SM vs the default two stages x 3 CTAs/SM
S="import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['config']['workload'][:5],round(d['ms_per_step'],4),round(d['roofline']['kernel_ms'],4))"
for v in base m3 m4; do cp ab/libfsx_$v.so paper_2105_06676_b200/libfsx.so; for c in cfg2 cfg4; do
  if [ $v = base ]; then E=""; else E="FSX_ROW_STAGES=1"; fi
  echo -n "$v $c "; env $E timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/l_bench_${v}_$c.log 2>&1; python -c "$S" < gpurun_out/l_bench_${v}_$c.log; done; done
cp ab/libfsx_m4.so paper_2105_06676_b200/libfsx.so
FSX_ROW_STAGES=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launches_m4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python scripts/launches.py gpurun_out/l_launches_m4.csv | tail -3
