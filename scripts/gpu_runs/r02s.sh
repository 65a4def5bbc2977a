# r02s: smoke() at HEAD; ncu --set full of the two-group cfg3 row kernels; cluster placement micro
set -x
D=gpurun_out/r02s
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; echo "rc=$?" >> $D/smoke.txt
timeout 60 ./scripts/micro/cluster_place > $D/cluster_place.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > $D/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_r2c_grp|k_c2r_grp" -s 4 -c 2 -o $D/prof_rows python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cut > $D/ncu.log 2>&1
cat $D/smoke.txt $D/cluster_place.txt
