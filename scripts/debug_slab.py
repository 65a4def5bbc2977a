import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import refutil as R
import paper_2105_06676_b200 as fs
from paper_2105_06676_b200.distributed import slab_describe, GpuSlabStages
from test_distributed_cpu import NumpyStages
for dims, P in (([256, 512], 1), ([256, 512], 2), ([32, 64, 128], 1), ([32, 64, 128], 2)):
    kern = R.random_kernel(R.Rng(7), len(dims), 1, 1, 0.95)
    k = fs.StencilKernel(len(dims))
    for off, blk in sorted(kern.taps.items()): k.add_tap(off, float(blk[0, 0]))
    n = int(np.prod(dims)); a0 = np.random.default_rng(1).uniform(-1, 1, n)
    shape = fs.GridShape(dims)
    r = 0
    info = slab_describe(shape, P, r)
    npst = NumpyStages(dims, P, r, info, kern)
    g = GpuSlabStages(shape, P, r)
    n0l = dims[0] // P
    slab = a0.reshape(dims[0], -1)[:n0l].reshape(-1).copy()
    nx = info["xbuf_bytes"] // 8
    s_np = torch.zeros(nx, dtype=torch.float64); npst.forward(torch.from_numpy(slab), s_np)
    s_gp = torch.zeros(nx, dtype=torch.float64, device="cuda"); g.forward(torch.from_numpy(slab).cuda(), s_gp)
    torch.cuda.synchronize()
    a = s_np.numpy().view(np.complex128); b = s_gp.cpu().numpy().view(np.complex128)
    if len(dims) == 2:
        A = a.reshape(P, n0l, -1)[:, :, :]; B = b.reshape(P, n0l, -1)
        M = dims[-1] // 2
        mask = np.zeros(A.shape, bool)
        for d in range(P):
            for j in range(A.shape[2]):
                mask[d, :, j] = d * info["col_block"] + j <= M
        print(dims, P, "forward maxdiff", np.abs((A - B)[mask]).max(), "scale", np.abs(A[mask]).max())
    else:
        print(dims, P, "forward maxdiff (incl padding)", np.abs(a - b).max())
    # spectral on identical input (numpy forward output as recv; P=1 -> recv == send)
    if P == 1:
        r_np = s_np.clone(); npst.spectral(r_np, None, 20)
        r_gp = s_np.clone().cuda(); g.spectral(r_gp, k, 20); torch.cuda.synchronize()
        a = r_np.numpy().view(np.complex128); b = r_gp.cpu().numpy().view(np.complex128)
        print(dims, "spectral maxdiff", np.abs(a - b).max(), "scale", np.abs(a).max(), "nan", np.isnan(b).sum())
        o_np = torch.zeros(slab.size, dtype=torch.float64); npst.inverse(r_np, o_np)
        o_gp = torch.zeros(slab.size, dtype=torch.float64, device="cuda"); g.inverse(r_np.clone().cuda(), o_gp); torch.cuda.synchronize()
        print(dims, "inverse maxdiff", np.abs(o_np.numpy() - o_gp.cpu().numpy()).max(), "scale", np.abs(o_np.numpy()).max())
