# r04h: oracle/_ref (the reference's own sources against the Eigen stand-in) on the GPU box: the new
# GPU-vs-reference tests, the reference arm and cpu_baseline with kind "reference", then the full suite
set -x
D=gpurun_out/r04h
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $D/smi.txt 2>&1
nproc > $D/host.txt; free -g >> $D/host.txt
timeout 900 python -m pytest tests/test_reference_outputs.py tests/test_oracle_vs_ref_cpu.py -q -s > $D/pytest_ref.txt 2>&1; echo "rc=$?" >> $D/pytest_ref.txt
grep -h "GPU vs\|passed\|failed\|rc=" $D/pytest_ref.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_ref_cfg3.json 2> $D/bench_ref.err
tail -1 $D/bench_ref_cfg3.json | cut -c1-400
timeout 900 python bench.py > $D/bench_cfg3.json 2> $D/bench_cfg3.err
python -c "
import json; d=json.loads(open('$D/bench_cfg3.json').read().strip().splitlines()[-1]); print('cfg3', round(d['ms_per_step'],4), '%.3e'%d['value'], round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3), round(d['pipeline']['frac'],3), '%.3e'%d['e2e']['value'], d['cpu_baseline']['kind'], '%.3e'%d['cpu_baseline']['value'], d['cpu_baseline']['sample'][:120])"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; cat $D/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
