"""Soak test of the grouped kernels' stage-release ordering: repeats the numeric phase of a banded
bs 16 (leaf 128, groups) and bs 32 (leaf 32, quads) product and compares every result bitwise with
the first one (as scripts/race_check.py does for k_numeric_tma)."""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2011_11762_b200 import MatrixSession, spgemm, _ffi

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
ses = MatrixSession(device="cuda:0")
lib = _ffi.load()
for bs, leaf, n, hb in ((16, 128, 65536, 256), (32, 32, 131072, 512), (16, 256, 32768, 128)):
    d = np.arange(-hb, hb + 1)
    rows = np.repeat(np.arange(n), d.size)
    cols = rows + np.tile(d, n)
    keep = (cols >= 0) & (cols < n)
    rows, cols = rows[keep], cols[keep]
    vals = np.random.default_rng(bs).uniform(-1, 1, rows.size)
    a = ses.matrix_from_triplets(n, rows, cols, vals, leaf_dim=leaf, block_size=bs)
    del rows, cols, vals
    x = a.root.require()
    lay = _ffi.make_layout(a.params, bs)
    plan = spgemm.symbolic(lay, x, x)
    kern = lib.qm_numeric_kernel(ctypes.byref(lay), plan.n_c, plan.n_triples, 0, 0).decode()
    first, _, _ = spgemm.numeric(lay, x, x, plan)
    bad = 0
    for _ in range(reps):
        c, _, _ = spgemm.numeric(lay, x, x, plan)
        bad += int(not (torch.equal(c.blocks, first.blocks) and torch.equal(c.sumsq, first.sumsq)))
    torch.cuda.synchronize()
    print(f"bs {bs} leaf {leaf} n {n}: {kern}, {plan.n_triples} triples, {reps} repetitions, {bad} differing", flush=True)
    assert bad == 0
print("ok")
