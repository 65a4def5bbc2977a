# r04u: zero-column shortcut in the 2D slab (multi-GPU) fused pass: slab / multi-GPU / determinism tests
# (emulated ranks: vs the oracle and bitwise = single GPU), large-T slab case with and without the shortcut
set -x
D=gpurun_out/r04u
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_slab.py tests/test_gpu_multi.py tests/test_gpu_determinism.py -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
cat > $D/slab_zero.py <<'PY'
import os, time, numpy as np
import paper_2105_06676_b200 as fs
from paper_2105_06676_b200 import synthetic
cfg = synthetic.configs()['cfg3'].scaled([8192, 2048])
g = fs.FieldGrid(cfg.shape(), cfg.initial())
single = fs.solve_periodic(g, cfg.kernel(), cfg.T).data
outs = {}
for z in ("1", "0"):
    os.environ["FSX_ZEROCOL"] = z
    for P in (2, 4):
        o = fs.solve_periodic(g, cfg.kernel(), cfg.T, devices=[0] * P).data
        t0 = time.perf_counter()
        for _ in range(3):
            o = fs.solve_periodic(g, cfg.kernel(), cfg.T, devices=[0] * P).data
        dt = (time.perf_counter() - t0) / 3
        outs[(z, P)] = o
        print(f"FSX_ZEROCOL={z} P={P}: bitwise == single GPU: {np.array_equal(o.view(np.int64), single.view(np.int64))}, host call {dt * 1e3:.1f} ms")
PY
PYTHONPATH=$PWD timeout 600 python $D/slab_zero.py 2>&1 | tee $D/slab_zero.txt
