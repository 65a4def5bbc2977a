# r04x: column bounds cached per taps, cut per T by a threshold scan (ColumnCut): cut / parity / slab tests,
# host cost of a solve with a NEW T on every call (device-resident cfg3), default bench line
set -x
D=gpurun_out/r04x
mkdir -p $D
timeout 1500 python -m pytest tests/test_gpu_cut.py tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_multi.py tests/test_gpu_slabs.py -q > $D/pytest.txt 2>&1; echo "rc=$?" >> $D/pytest.txt
tail -3 $D/pytest.txt
cat > $D/newT.py <<'PY'
import os, time, numpy as np, torch
import paper_2105_06676_b200 as fs
from paper_2105_06676_b200 import synthetic
cfg = synthetic.configs()['cfg3']
shape, kern = cfg.shape(), cfg.kernel()
a = torch.from_numpy(cfg.initial()).cuda(); out = torch.empty_like(a)
for z in ("1", "0"):
    os.environ["FSX_ZEROCOL"] = z
    fs.solve_periodic_device(shape, a.data_ptr(), kern, cfg.T, out.data_ptr(), device=0); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(50):
        fs.solve_periodic_device(shape, a.data_ptr(), kern, cfg.T + 1 + i, out.data_ptr(), device=0)
    torch.cuda.synchronize()
    print(f"FSX_ZEROCOL={z}: 50 device-resident cfg3 solves, a new T each: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per solve (wall)")
PY
PYTHONPATH=$PWD timeout 600 python $D/newT.py 2>&1 | tee $D/newT.txt
timeout 900 python bench.py --no-cpu > $D/bench_cfg3.json 2> $D/bench_cfg3.err
python scripts/summarize.py $D/bench_cfg3.json
