"""Generates tests/golden/reference_outputs.npz: outputs of the REFERENCE's own
solve_periodic / solve_periodic_vector / solve_periodic_implicit code
(oracle/_ref/libfftstencil_ref.so = /root/reference/proj/src compiled unmodified
by `make -C oracle ref`, Eigen3 replaced by oracle/eigen_shim) on seeded inputs.

Run in the development container (needs /root/reference):

    python tests/golden/make_reference_outputs.py

The inputs are not stored: tests regenerate them from the seeds with
tests/refutil.py (the reference's test generators restated draw for draw).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ref as refmod  # noqa: E402
from refutil import Rng, random_grid, random_kernel  # noqa: E402

# (dims, fields, T, seed): explicit solves
CASES = [
    ([1024], 1, 1000, 1), ([1000], 1, 77, 2), ([4096], 2, 5000, 3), ([64, 64], 1, 10000, 4),
    ([48, 40], 1, 123, 5), ([128, 32], 1, 100000, 6), ([16, 16, 16], 1, 1000, 7), ([12, 10, 14], 1, 50, 8),
    ([32, 24], 2, 300, 9), ([8, 8, 8, 8], 1, 9, 10), ([256, 1], 1, 64, 11), ([4096], 1, 0, 12),
]
# (dims, T, seed): Crank-Nicolson-like implicit solves
IMPLICIT = [([512], 40, 21), ([32, 32], 25, 22), ([16, 8, 8], 10, 23)]


def explicit_inputs(dims, m, seed):
    rng = Rng(seed)
    sigma = max(0, min(2, (min(dims) - 1) // 2))
    k = random_kernel(rng, len(dims), sigma, m)
    a0 = random_grid(rng, int(np.prod(dims)) * m)
    off, blk = k.arrays()
    return a0, off, blk


def implicit_inputs(dims, seed):
    rng = Rng(seed)
    r = len(dims)
    a = 0.05 + 0.2 * rng.uniform()
    zero = tuple([0] * r)
    q, s = {zero: 1.0 + 2 * a * r}, {zero: 1.0 - 2 * a * r}
    for ax in range(r):
        for sg in (-1, 1):
            o = [0] * r
            o[ax] = sg
            q[tuple(o)], s[tuple(o)] = -a, a
    keys = sorted(q)
    off = np.array(keys, dtype=np.int64).reshape(len(keys), r)
    qa = (off, np.array([q[k] for k in keys]).reshape(-1, 1, 1))
    sa = (off, np.array([s[k] for k in keys]).reshape(-1, 1, 1))
    return random_grid(rng, int(np.prod(dims))), qa, sa


def main():
    assert refmod.build(), "oracle/_ref not buildable here"
    ref = refmod.module()
    out, meta = {}, {"explicit": [], "implicit": []}
    for i, (dims, m, T, seed) in enumerate(CASES):
        a0, off, blk = explicit_inputs(dims, m, seed)
        out[f"explicit_{i}"] = ref.solve_periodic(a0, dims, m, off, blk, T, vector=m > 1)
        meta["explicit"].append({"dims": dims, "fields": m, "T": T, "seed": seed})
    for i, (dims, T, seed) in enumerate(IMPLICIT):
        a0, q, s = implicit_inputs(dims, seed)
        out[f"implicit_{i}"] = ref.solve_periodic_implicit(a0, dims, q, s, T)
        meta["implicit"].append({"dims": dims, "T": T, "seed": seed})
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(ROOT, "tests", "golden", "reference_outputs.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(CASES) + len(IMPLICIT), "cases")


if __name__ == "__main__":
    main()
