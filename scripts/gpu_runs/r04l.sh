# r04l: larger randomized parity sweeps at HEAD (seeds 61-63, zero-column shortcut on by default)
set -x
D=gpurun_out/r04l
mkdir -p $D
timeout 1500 python scripts/stress_parity.py 500 61 4000000 > $D/stress_s61.txt 2>&1
timeout 1500 python scripts/stress_parity.py 500 62 1000000 > $D/stress_s62.txt 2>&1
timeout 900 python scripts/stress_parity.py 200 63 40000000 > $D/stress_s63.txt 2>&1
for f in $D/stress_s61.txt $D/stress_s62.txt $D/stress_s63.txt; do tail -n 1 "$f"; done
