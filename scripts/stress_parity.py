"""Randomized parity sweep on the GPU (not part of the test suite): random
shapes (rank 1-3, pow2 and not, length-1 axes), random kernels (m = 1, 2,
symmetric or not), random T, each solved through the fp64 host API, the fp32
mode and the spectral cut, checked against the CPU oracle; then random
implicit (Crank-Nicolson-like) solves against the oracle and batches against
single calls (bitwise).
    python scripts/stress_parity.py [cases] [seed] [max cells]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2105_06676_b200 as fs  # noqa: E402
import refutil as R  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def K(k):
    out = fs.StencilKernel(k.rank, k.fields)
    for off in sorted(k.taps):
        out.add_tap(off, k.taps[off] if k.fields > 1 else float(k.taps[off][0, 0]))
    return out


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / (nb if nb > 0 else 1.0))


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    pow2 = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]
    other = [3, 5, 6, 7, 12, 15, 24, 100, 255, 300]
    worst = {"f64": 0.0, "f32": 0.0, "cut": 0.0}
    fails = 0
    for i in range(cases):
        rank = int(rng.integers(1, 4))
        m = 2 if (rank == 1 and rng.random() < 0.25) else (int(rng.integers(2, 4)) if rng.random() < 0.1 else 1)
        dims = []
        budget = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 18
        for a in range(rank):
            choices = pow2 if rng.random() < 0.8 else other
            if rng.random() < 0.1:
                choices = [1]
            d = int(rng.choice([c for c in choices if c <= budget] or [1]))
            dims.append(d)
            budget = max(1, budget // max(d, 1))
        if rank == 1 and dims[0] < 2:
            dims = [64]
        k = R.random_kernel(R.Rng(1000 + i), rank, int(rng.integers(1, 3)), m, 0.95)
        # symmetric half the time (real symbols: the fused multiplier / fp32 paths)
        if rng.random() < 0.5:
            sym = R.Kern(rank, m)
            for off, b in k.taps.items():
                if all(abs(o) < max(d, 1) for o, d in zip(off, dims)):
                    sym.add(off, b / 2)
                    sym.add(tuple(-o for o in off), b / 2)
            k = sym
        if not k.taps or any(any(abs(o) >= d for o, d in zip(off, dims)) for off in k.taps):
            continue
        T = int(rng.choice([1, 2, 7, 100, 1000, 10000]))
        n = int(np.prod(dims)) * m
        a0 = orc.splitmix_fill(5000 + i, n, True)
        try:
            want = orc.solve_periodic(a0, dims, m, *k.arrays(), T)
        except Exception as e:  # the reference raises too (NumericError): ours must as well
            try:
                fs.solve_periodic(fs.FieldGrid(fs.GridShape(dims, m), a0), K(k), T)
                print("MISSING ERROR", dims, m, T, e)
                fails += 1
            except fs.Error:
                pass
            continue
        g = fs.FieldGrid(fs.GridShape(dims, m), a0)
        tag = f"{dims} m={m} T={T} taps={len(k.taps)}"
        try:
            e64 = rel(fs.solve_periodic(g, K(k), T).data, want)
            ecut = rel(fs.solve_periodic(g, K(k), T, spectral_cut=1).data, want)
            e32 = rel(fs.solve_periodic_f32(fs.GridShape(dims, m), a0.astype(np.float32), K(k), T),
                      orc.solve_periodic(a0.astype(np.float32).astype(np.float64), dims, m, *k.arrays(), T))
        except fs.NumericError as e:
            # residue / non-finite limits can trip where the oracle's stricter-typed path did not
            print("numeric", tag, e)
            continue
        worst["f64"] = max(worst["f64"], e64)
        worst["cut"] = max(worst["cut"], ecut)
        # the fp32 mode cannot represent results below the float range (they round to 0 or to
        # subnormals): judge it only where the result is comfortably inside that range
        f32_ok_range = np.max(np.abs(want)) > 1e-30
        if not f32_ok_range:
            e32 = 0.0
        bad = e64 > 1e-10 or ecut > 1e-10 or e32 > 1e-4
        worst["f32"] = max(worst["f32"], e32)
        if bad:
            fails += 1
            print("FAIL", tag, f"f64 {e64:.2e} cut {ecut:.2e} f32 {e32:.2e} max|want| {np.max(np.abs(want)):.2e}")
    # implicit solves (Crank-Nicolson-like q = (1 + b) I - b S', s = I + ...) and batches
    worst_i = worst_b = 0.0
    for i in range(cases // 4):
        rank = int(rng.integers(1, 4))
        dims = [int(rng.choice([8, 16, 32, 64, 128, 256, 12, 100])) for _ in range(rank)]
        while int(np.prod(dims)) > (1 << 18):
            dims[0] //= 2
        b = float(rng.uniform(0.05, 0.4))
        qd, sd = {(0,) * rank: 1.0 + b * rank}, {(0,) * rank: 1.0 - b * rank}
        for a in range(rank):
            for sg in (-1, 1):
                off = tuple(sg if j == a else 0 for j in range(rank))
                if dims[a] > 1:
                    qd[off] = qd.get(off, 0.0) - b / 2
                    sd[off] = sd.get(off, 0.0) + b / 2
        q, sk = R.kern_from(qd, rank), R.kern_from(sd, rank)
        T = int(rng.choice([1, 10, 100, 1000]))
        n = int(np.prod(dims))
        a0 = orc.splitmix_fill(9000 + i, n, True)
        want = orc.solve_periodic_implicit(a0, dims, q.arrays(), sk.arrays(), T)
        got = fs.solve_periodic_implicit(K(q), K(sk), fs.FieldGrid(fs.GridShape(dims), a0), T).data
        e = rel(got, want)
        worst_i = max(worst_i, e)
        if e > 1e-10:
            fails += 1
            print("FAIL implicit", dims, T, f"{e:.2e}")
        g = fs.FieldGrid(fs.GridShape(dims), a0)
        outs = fs.solve_periodic_batch([g, g], K(sk), T)
        one = fs.solve_periodic(g, K(sk), T).data
        eb = max(rel(o, one) for o in outs)
        worst_b = max(worst_b, eb)
        if eb != 0.0:
            fails += 1
            print("FAIL batch", dims, T, f"{eb:.2e}")
    # slab decomposition emulated on one GPU (P ranks' stages in turn; nccl-layout and p2p
    # exchanges), random 2D / 3D power-of-two shapes
    import torch
    from paper_2105_06676_b200.distributed import slab_solve_emulated, slab_solve_emulated_p2p
    worst_s = 0.0
    for i in range(cases // 6):
        rank = int(rng.integers(2, 4))
        P = int(rng.choice([2, 4, 8]))
        dims = [int(rng.choice([64, 128, 256, 512, 1024]))] + \
               [int(rng.choice([16, 32, 64, 128, 256, 512, 1024])) for _ in range(rank - 1)]
        while int(np.prod(dims)) > (1 << 20):
            dims[-1] //= 2
        k = R.random_kernel(R.Rng(7000 + i), rank, 1, 1, 0.95)
        T = int(rng.choice([1, 10, 1000]))
        n = int(np.prod(dims))
        a0 = orc.splitmix_fill(8000 + i, n, True)
        try:
            want = orc.solve_periodic(a0, dims, 1, *k.arrays(), T)
        except orc.OracleSpecError as ex:  # the shrunken last axis is shorter than the kernel's reach
            print("slab skip", dims, P, ex)
            continue
        da = torch.from_numpy(a0).cuda()
        try:
            got = slab_solve_emulated(fs.GridShape(dims), da, K(k), T, P).cpu().numpy()
            e = rel(got, want)
            if rank == 2:
                e = max(e, rel(slab_solve_emulated_p2p(fs.GridShape(dims), da, K(k), T, P).cpu().numpy(), want))
        except fs.Error as ex:  # shapes the slab geometry rejects
            print("slab skip", dims, P, ex)
            continue
        worst_s = max(worst_s, e)
        if e > 1e-10:
            fails += 1
            print("FAIL slab", dims, P, T, f"{e:.2e}")
    worst["slab"] = worst_s
    worst["implicit"] = worst_i
    worst["batch_vs_single"] = worst_b
    print(f"{cases} + {cases // 4} cases, {fails} failures, worst: " + ", ".join(f"{k} {v:.2e}" for k, v in worst.items()))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
