# r04m: k_fused8192c with the W^k O products formed by the joining CTA (balanced pair) against the
# previous build (ab/libfsx_old.so), cfg3; bitwise old-vs-new output check; 8192-column tests
set -x
D=gpurun_out/r04m
mkdir -p $D
for rep in 1 2 3; do
  FSX_LIB=$PWD/ab/libfsx_old.so timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/old_$rep.json 2>/dev/null
  timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/new_$rep.json 2>/dev/null
done
for f in $D/old_*.json $D/new_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
cat > /tmp/bitwise.py <<'PY'
import sys, numpy as np
import paper_2105_06676_b200 as fs
from paper_2105_06676_b200 import synthetic
cfg = synthetic.configs()['cfg3'].scaled([8192, 1024])
out = fs.solve_periodic(fs.FieldGrid(cfg.shape(), cfg.initial()), cfg.kernel(), 300).data
np.save(sys.argv[1], out)
PY
FSX_LIB=$PWD/ab/libfsx_old.so python /tmp/bitwise.py /tmp/old.npy; python /tmp/bitwise.py /tmp/new.npy
python -c "
import numpy as np; a=np.load('/tmp/old.npy'); b=np.load('/tmp/new.npy'); print('bitwise old==new:', np.array_equal(a.view(np.int64), b.view(np.int64)), float(np.abs(a-b).max()))"
timeout 1200 python -m pytest tests/test_gpu_cut.py tests/test_gpu_determinism.py tests/test_gpu_multi.py -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -s -k "cfg3_full_size_vs" >> $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
grep -h "cfg3 FULL\|passed\|failed\|rc=" $D/pytest.txt
