# full twiddle tables per pass for the 4096-point fused columns (FT mask)
for V in 0 2 4 6; do
  touch paper_2105_06676_b200/csrc/fsx_tma.cu; make -s EXTRA=-DFSX_FT4096=$V > /dev/null 2>&1
  timeout 300 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab35_ft$V.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab35_launch_ft$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
done
python scripts/summarize.py gpurun_out/ab35_ft*.log
python scripts/launches.py gpurun_out/ab35_launch_ft*.csv | grep -E "csv|cols"
