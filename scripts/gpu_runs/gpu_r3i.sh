# final check after the row-stage change: full GPU suite, smoke, a cut run on 4096-complex rows, cfg3 bench
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python -c "
import sys; sys.path.insert(0,'tests'); import numpy as np, refutil as R, paper_2105_06676_b200 as fs
from oracle import oracle as orc
k=R.kern_from({(0,0):0.2,(1,0):0.2,(-1,0):0.2,(0,1):0.2,(0,-1):0.2},2)
K=fs.StencilKernel(2)
[K.add_tap(o,float(b[0,0])) for o,b in sorted(k.taps.items())]
a=orc.splitmix_fill(3,512*8192,True); g=fs.FieldGrid(fs.GridShape([512,8192]),a)
f=fs.solve_periodic(g,K,20000).data; c=fs.solve_periodic(g,K,20000,spectral_cut=1).data
print('cut on 4096-complex rows equal:', np.array_equal(f,c), fs.spectral_cut_columns(fs.GridShape([512,8192]),K,20000))"
timeout 600 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > gpurun_out/i3_cfg3.log 2>&1; python scripts/summarize.py gpurun_out/i3_cfg3.log
