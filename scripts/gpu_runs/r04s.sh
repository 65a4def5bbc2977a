# r04s: ncu --set full of the cfg3 and cfg2 dominant kernels at HEAD (after their own commands exited 0
# without ncu in r04q), exported to csv on the box (the .ncu-rep files exceed the 64 MiB return limit)
set -x
D=gpurun_out/r04s
mkdir -p $D
for spec in "cfg3 k_fused8192c fused8192c" "cfg2 k_cols_tma cols_tma_cfg2" "cfg3 k_r2c_grp r2c_grp_cfg3" "cfg3 k_c2r_grp c2r_grp_cfg3"; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 -s 2 -c 1 -o /tmp/$3 -f python bench.py --config $1 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu_full_$3.log 2>&1
  ncu -i /tmp/$3.ncu-rep --page raw --csv > $D/$3_raw.csv 2>/dev/null
  ncu -i /tmp/$3.ncu-rep --page source --csv --print-source sass > $D/$3_src.csv 2>/dev/null
  rm -f /tmp/$3.ncu-rep
done
du -sh $D
