# r02r: full GPU suite + randomized stress sweep at HEAD (row groups, cfg5 row pairs on a CTA pair)
set -x
D=gpurun_out/r02r
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
timeout 900 python scripts/stress_parity.py 300 11 4000000 > $D/stress_s11.txt 2>&1
timeout 600 python scripts/stress_parity.py 150 12 40000000 > $D/stress_s12_large.txt 2>&1
tail -3 $D/pytest.txt; tail -8 $D/stress_s11.txt; tail -8 $D/stress_s12_large.txt
