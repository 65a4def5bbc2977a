# r04n: where the CTAs of a pair land (cluster_place under the three scheduling policies) and the
# cluster scheduling policy preference A/B on cfg3 (k_fused8192c) and cfg5 (k_rowpair_c); bitwise
# check of the balanced-join build against the previous one
set -x
D=gpurun_out/r04n
mkdir -p $D
timeout 60 ./scripts/micro/cluster_place > $D/cluster_place.txt 2>&1; cat $D/cluster_place.txt
for rep in 1 2; do
for pol in 0 1 2; do
  FSX_CLUSTER_POLICY=$pol timeout 600 python bench.py --config cfg3 --steps 20 --warmup 3 --no-cpu --no-e2e --no-cut > $D/pol${pol}_cfg3_$rep.json 2>/dev/null
  FSX_CLUSTER_POLICY=$pol timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-cut > $D/pol${pol}_cfg5_$rep.json 2>/dev/null
done
done
for f in $D/pol*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done
cat > $D/bitwise.py <<'PY'
import sys, numpy as np
import paper_2105_06676_b200 as fs
from paper_2105_06676_b200 import synthetic
cfg = synthetic.configs()['cfg3'].scaled([8192, 1024])
out = fs.solve_periodic(fs.FieldGrid(cfg.shape(), cfg.initial()), cfg.kernel(), 300).data
np.save(sys.argv[1], out)
PY
FSX_LIB=$PWD/ab/libfsx_old.so PYTHONPATH=$PWD python $D/bitwise.py /tmp/old.npy; PYTHONPATH=$PWD python $D/bitwise.py /tmp/new.npy
python -c "
import numpy as np; a=np.load('/tmp/old.npy'); b=np.load('/tmp/new.npy'); print('bitwise old==new:', np.array_equal(a.view(np.int64), b.view(np.int64)), float(np.abs(a-b).max()))" | tee $D/bitwise.txt
