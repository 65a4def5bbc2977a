# r04c: folded cosine taps in the real row-pair symbol; cfg5 at full size against the exact answer
set -x
D=gpurun_out/r04c
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "rowpair or cfg5 or many_fields or plans or batch or semigroup" > $D/pytest_parity.txt 2>&1; echo "rc=$?" >> $D/pytest_parity.txt
timeout 900 python -m pytest tests/test_gpu_naive.py tests/test_gpu_determinism.py -q -s -k "cfg5 or rowpair or full" > $D/pytest_naive.txt 2>&1; echo "rc=$?" >> $D/pytest_naive.txt
timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu > $D/bench_cfg5.json 2> $D/bench_cfg5.err
grep -h "cfg5 \|passed\|failed\|rc=" $D/pytest_parity.txt $D/pytest_naive.txt
python -c "
import json; d=json.loads(open('$D/bench_cfg5.json').read().strip().splitlines()[-1]); print('cfg5', round(d['ms_per_step'],4), '%.3e'%d['value'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), round(d['pipeline']['frac'],3))"
