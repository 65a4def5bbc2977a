# r04j: host-proved zero columns take multiplier 0 without evaluating the symbol (FusedSymbol::kzero):
# A/B (FSX_ZEROCOL=0 evaluates every column) on cfg3 / cfg2, bitwise test, cut and parity tests
set -x
D=gpurun_out/r04j
mkdir -p $D
for rep in 1 2; do
for c in cfg3 cfg2; do
for z in 0 1; do
  FSX_ZEROCOL=$z timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/zc${z}_${c}_$rep.json 2>/dev/null
done
done
done
for f in $D/zc*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
timeout 1200 python -m pytest tests/test_gpu_cut.py tests/test_gpu_parity.py tests/test_reference_outputs.py -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
