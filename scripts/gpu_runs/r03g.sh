# r03g: larger randomized parity sweeps at HEAD (seeds 31-33)
set -x
D=gpurun_out/r03g
mkdir -p $D
timeout 1500 python scripts/stress_parity.py 500 31 4000000 > $D/stress_s31.txt 2>&1
timeout 1500 python scripts/stress_parity.py 500 32 1000000 > $D/stress_s32.txt 2>&1
timeout 900 python scripts/stress_parity.py 200 33 40000000 > $D/stress_s33.txt 2>&1
for f in $D/stress_s31.txt $D/stress_s32.txt $D/stress_s33.txt; do tail -n 1 "$f"; done
